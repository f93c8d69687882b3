// sw_common.cuh -- constants, alphabet tables and the per-lane value traits of
// the sm_100a Smith-Waterman path.  Product code: shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "sw.h"

namespace swb {

constexpr uint32_t FULL = 0xffffffffu;

// Reference code layout: every reference gets PADL pad codes before it and
// PADR after it, so the wavefront's fill/drain columns read pad codes without
// bounds checks (the paper's "padding instead of boundary
// checks" lesson, reused here).
constexpr int PADL = 32;
constexpr int PADR = 64;
// Pad codes finish_fwd writes right after each reversed prefix (<= PADR).
constexpr int REV_PAD = 16;
// Tail guard of the code buffers: a work item's shorter half keeps reading
// (frozen, harmless) codes up to the item's longest reference + fill/drain.
constexpr int64_t GUARD = SW_MAX_SEQ_LEN + 256;

constexpr int NC_DNA = 5;        // A C G T + pad
constexpr int NC_PROTEIN = 25;   // 24 BLOSUM62 symbols + pad
constexpr uint8_t CODE_BAD = 0xff;

// Kernel routes of a pair:
//   ROUTE_TAG  s16x2 lanes, column-in-block and row carried in the low 6 bits of the running max
//              (pairs whose largest possible score is <= TAG_MAX_SCORE)
//   ROUTE_S16  s16x2 lanes, improvement columns saved to shared memory
//   ROUTE_S32  int32 lanes (scorings / lengths that are not int16-safe)
constexpr int ROUTE_TAG = 0, ROUTE_S16 = 1, ROUTE_S32 = 2, N_ROUTES = 3;
// s16 lanes hold Hb = H - o; the int8 profile already forces -o <= 126 (s - o <= 127, s >= 1)
constexpr int S16_MAX_SCORE = 32000;  // Hb <= 32126 < 32768
// protein geometry (sw_api.cu): 8 rows per lane keep the 25-code int8 profile at 8 bytes per (code, lane)
#ifndef SW_KP
#define SW_KP 8
#endif
#ifndef SW_WP
#define SW_WP 16
#endif
constexpr int TAG_MAX_SCORE = 511;    // 511 * 64 + 63 < 32768 (6 tag bits: column-in-block, row)
#ifndef SW_PTAG
#define SW_PTAG 0
#endif
// protein forward TAG (sw_wavefront.cuh PT): 8191 * 8 + 7 <= 65535 (3 row-tag bits, unsigned running max)
constexpr int PTAG_MAX_SCORE = 8191;
// largest max_s * n of a pair on the forward TAG route of an alphabet (-1: no TAG route)
__host__ __device__ constexpr int tag_max_score(int alphabet) {
    return alphabet == SW_ALPHABET_DNA ? TAG_MAX_SCORE : (SW_PTAG ? PTAG_MAX_SCORE : -1);
}
// Work keys: [31:30] 3 - route (0 = trivial / invalid), [29:16] stripes, [15:0] columns
__host__ __device__ constexpr uint32_t route_key(int route) { return (uint32_t)(3 - route) << 30; }

// per-pair flags: bit 0 invalid, bits 2:1 route
constexpr uint8_t FLAG_BAD = 1;
__host__ __device__ constexpr uint8_t route_flag(int route) { return (uint8_t)(route << 1); }
__host__ __device__ constexpr int flag_route(uint8_t f) { return (f >> 1) & 3; }

// Product copy of NCBI BLOSUM62 (order ARNDCQEGHILKMFPSTWYVBZX*), R11.
__constant__ int8_t c_blosum62[24][24] = {
    { 4,-1,-2,-2, 0,-1,-1, 0,-2,-1,-1,-1,-1,-2,-1, 1, 0,-3,-2, 0,-2,-1, 0,-4},
    {-1, 5, 0,-2,-3, 1, 0,-2, 0,-3,-2, 2,-1,-3,-2,-1,-1,-3,-2,-3,-1, 0,-1,-4},
    {-2, 0, 6, 1,-3, 0, 0, 0, 1,-3,-3, 0,-2,-3,-2, 1, 0,-4,-2,-3, 3, 0,-1,-4},
    {-2,-2, 1, 6,-3, 0, 2,-1,-1,-3,-4,-1,-3,-3,-1, 0,-1,-4,-3,-3, 4, 1,-1,-4},
    { 0,-3,-3,-3, 9,-3,-4,-3,-3,-1,-1,-3,-1,-2,-3,-1,-1,-2,-2,-1,-3,-3,-2,-4},
    {-1, 1, 0, 0,-3, 5, 2,-2, 0,-3,-2, 1, 0,-3,-1, 0,-1,-2,-1,-2, 0, 3,-1,-4},
    {-1, 0, 0, 2,-4, 2, 5,-2, 0,-3,-3, 1,-2,-3,-1, 0,-1,-3,-2,-2, 1, 4,-1,-4},
    { 0,-2, 0,-1,-3,-2,-2, 6,-2,-4,-4,-2,-3,-3,-2, 0,-2,-2,-3,-3,-1,-2,-1,-4},
    {-2, 0, 1,-1,-3, 0, 0,-2, 8,-3,-3,-1,-2,-1,-2,-1,-2,-2, 2,-3, 0, 0,-1,-4},
    {-1,-3,-3,-3,-1,-3,-3,-4,-3, 4, 2,-3, 1, 0,-3,-2,-1,-3,-1, 3,-3,-3,-1,-4},
    {-1,-2,-3,-4,-1,-2,-3,-4,-3, 2, 4,-2, 2, 0,-3,-2,-1,-2,-1, 1,-4,-3,-1,-4},
    {-1, 2, 0,-1,-3, 1, 1,-2,-1,-3,-2, 5,-1,-3,-1, 0,-1,-3,-2,-2, 0, 1,-1,-4},
    {-1,-1,-2,-3,-1, 0,-2,-3,-2, 1, 2,-1, 5, 0,-2,-1,-1,-1,-1, 1,-3,-1,-1,-4},
    {-2,-3,-3,-3,-2,-3,-3,-3,-1, 0, 0,-3, 0, 6,-4,-2,-2, 1, 3,-1,-3,-3,-1,-4},
    {-1,-2,-2,-1,-3,-1,-1,-2,-2,-3,-3,-1,-2,-4, 7,-1,-1,-4,-3,-2,-2,-1,-2,-4},
    { 1,-1, 1, 0,-1, 0, 0, 0,-1,-2,-2, 0,-1,-2,-1, 4, 1,-3,-2,-2, 0, 0, 0,-4},
    { 0,-1, 0,-1,-1,-1,-1,-2,-2,-1,-1,-1,-1,-2,-1, 1, 5,-2,-2, 0,-1,-1, 0,-4},
    {-3,-3,-4,-4,-2,-2,-3,-2,-2,-3,-2,-3,-1, 1,-4,-3,-2,11, 2,-3,-4,-3,-2,-4},
    {-2,-2,-2,-3,-2,-1,-2,-3, 2,-1,-1,-2,-1, 3,-3,-2,-2, 2, 7,-1,-3,-2,-1,-4},
    { 0,-3,-3,-3,-1,-2,-2,-3,-3, 3, 1,-2, 1,-1,-2,-2, 0,-3,-1, 4,-3,-2,-1,-4},
    {-2,-1, 3, 4,-3, 0, 1,-1, 0,-3,-4, 0,-3,-3,-2, 0,-1,-4,-3,-3, 4, 1,-1,-4},
    {-1, 0, 0, 1,-3, 3, 4,-2, 0,-3,-3, 1,-1,-3,-1, 0,-1,-3,-2,-2, 1, 4,-1,-4},
    { 0,-1,-1,-1,-2,-1,-1,-1,-1,-1,-1,-1,-1,-1,-2, 0, 0,-2,-1,-1,-1,-1,-1,-4},
    {-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4,-4, 1},
};

// Host-side max / min of BLOSUM62 (for routing decisions).
constexpr int BLOSUM62_MAX = 11;
constexpr int BLOSUM62_MIN = -4;

struct Scoring {
    int alphabet;
    int match, mismatch;
    int gap_open, gap_extend;
    int nc;        // codes incl. pad
    int max_sigma; // largest s(a,b)
};

// Gap-aware diagonal band of the reverse pass (reading R6).  Every score-S
// path of the reversed rectangle (n2 x m2) starts at its origin with an aligned pair; a cell of it on
// diagonal d = j' - i' > 0 needs >= d deletion columns, d < 0 needs >= -d insertion rows (each of
// which also forgoes its aligned pair), and any gap run costs |o| + (k-1)|e|.  With M <= n2 - I and
// M <= m2 - D aligned pairs scoring <= ms each:
//   -DI <= d <= DD,  DI = (ms n2 - S - (|o| - |e|)) / (ms + |e|),
//   DD = min((ms n2 - S - (|o| - |e|)) / |e|, (ms m2 - S - (|o| - |e|)) / (ms + |e|)).
// (go = -gap_open, ge = -gap_extend; clamped at 0: no gap fits -> the path is one diagonal.)
__host__ __device__ inline void rev_band(int ms, int go, int ge, int S, int n2, int m2, int& DI, int& DD) {
    const long long g0 = (long long)go - ge;
    long long slack = (long long)ms * n2 - S - g0, slack_m = (long long)ms * m2 - S - g0;
    slack = slack < 0 ? 0 : slack;
    slack_m = slack_m < 0 ? 0 : slack_m;
    long long di = slack / (ms + ge), dd = slack_m / (ms + ge);
    if (ge > 0 && slack / ge < dd) dd = slack / ge;
    DI = (int)(di < 0x3fffffffLL ? di : 0x3fffffffLL);
    DD = (int)(dd < 0x3fffffffLL ? dd : 0x3fffffffLL);
}

__device__ __forceinline__ int sigma_of(const Scoring& sc, int a, int b) {
    if (sc.alphabet == SW_ALPHABET_DNA) return a == b ? sc.match : sc.mismatch;
    return c_blosum62[a][b];
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// ---------------------------------------------------------------------------
// Per-lane value traits.  S16x2: every 32-bit register carries the same cell
// of TWO different pairs (low / high 16-bit half), so one DPX instruction
// advances two alignments.  S32: one pair per lane, int32 values (routing
// fallback for scorings / lengths that are not int16-safe).
// ---------------------------------------------------------------------------
struct TS16 {
    using V = uint32_t;
    static constexpr int NH = 2;
    static __device__ __forceinline__ V splat(int x) { return (uint32_t)(x & 0xffff) * 0x10001u; }
    // 32-bit addend that adds x to both halves of a word whose low half + x stays >= 0
    static __device__ __forceinline__ V lift(int x) { return (uint32_t)(x * 65537); }
    static __device__ __forceinline__ V add(V a, V b) { return __vadd2(a, b); }
    // max(a + b, c)
    static __device__ __forceinline__ V addmax(V a, V b, V c) { return __viaddmax_s16x2(a, b, c); }
    static __device__ __forceinline__ V max_relu(V a, V b) { return __vimax_s16x2_relu(a, b); }
    // max(a + b, c, 0)
    static __device__ __forceinline__ V addmax_relu(V a, V b, V c) { return __viaddmax_s16x2_relu(a, b, c); }
    static __device__ __forceinline__ V max3(V a, V b, V c) { return __vimax3_s16x2_relu(a, b, c); }
    static __device__ __forceinline__ V max2(V a, V b) { return __vimax_s16x2_relu(a, b); }
    // per-half all-ones mask where a != b (a >= b per half guaranteed)
    static __device__ __forceinline__ V changed_mask(V newv, V oldv) {
        uint32_t d = newv - oldv;                       // per-half >= 0: no borrow
        uint32_t nz = __vminu2(d, 0x00010001u);         // 0 or 1 per half
        return nz * 0xffffu;
    }
    static __device__ __forceinline__ int get(V v, int h) { return (int)(int16_t)(uint16_t)(v >> (16 * h)); }
    static __device__ __forceinline__ V set(V v, int h, int x) {
        return h ? ((v & 0x0000ffffu) | ((uint32_t)(x & 0xffff) << 16)) : ((v & 0xffff0000u) | (uint32_t)(x & 0xffff));
    }
    static constexpr int FROZEN = 0x7fff;
};

struct TS32 {
    using V = uint32_t;  // holds int32 bits
    static constexpr int NH = 1;
    static __device__ __forceinline__ V splat(int x) { return (uint32_t)x; }
    static __device__ __forceinline__ V lift(int x) { return (uint32_t)x; }
    static __device__ __forceinline__ V add(V a, V b) { return (uint32_t)((int)a + (int)b); }
    static __device__ __forceinline__ V addmax(V a, V b, V c) { return (uint32_t)__viaddmax_s32((int)a, (int)b, (int)c); }
    static __device__ __forceinline__ V max_relu(V a, V b) { return (uint32_t)__vimax_s32_relu((int)a, (int)b); }
    static __device__ __forceinline__ V addmax_relu(V a, V b, V c) { return (uint32_t)__viaddmax_s32_relu((int)a, (int)b, (int)c); }
    static __device__ __forceinline__ V max3(V a, V b, V c) { return (uint32_t)__vimax3_s32_relu((int)a, (int)b, (int)c); }
    static __device__ __forceinline__ V max2(V a, V b) { return (uint32_t)__vimax_s32_relu((int)a, (int)b); }
    static __device__ __forceinline__ V changed_mask(V newv, V oldv) { return newv != oldv ? 0xffffffffu : 0u; }
    static __device__ __forceinline__ int get(V v, int) { return (int)v; }
    static __device__ __forceinline__ V set(V, int, int x) { return (uint32_t)x; }
    static constexpr int FROZEN = 0x7fffffff;
};

}  // namespace swb
