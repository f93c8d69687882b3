// sw_wavefront.cuh -- steps a3 (forward: score + end) and a4 (reverse: start)
// of SURVEY.md sec. 8(a): the anti-diagonal Gotoh wavefront on sm_100a.
//
// Recurrence (affine state PAPER.md:507/713-714), in the
// clamped form the kernel runs (SW_XFORM, default).  With E^ = max(E, 0),
// F^ = max(F, 0), X = max(H[i-1][j-1] + s, E^) and R = H + o (o = gap_open):
//   E^[i][j] = max(E^[i][j-1] + e, R[i][j-1], 0)             VIADDMNMX.RELU
//   X[i][j]  = max(R[i-1][j-1] + (s - o), E^[i][j])          VIADDMNMX
//   F^[i][j] = max(F^[i-1][j] + e, X[i-1][j] + o, 0)         VIADDMNMX.RELU
//   R[i][j]  = max(F^[i][j] + o, X[i][j] + o)                VIADDMNMX (X + o: VIADD.16x2, FMA pipe)
// which is H = max(H[i-1][j-1] + s, E, F, 0), E = max(E[i][j-1] + e, H[i][j-1] + o),
// F = max(F[i-1][j] + e, H[i-1][j] + o) with E, F clamped at 0 (exact: e <= 0
// and o <= e, pin P13, readings R13/R21).  F^ of the next row needs
// only X + o of this one (H + o = max(X + o, F^ + o) and F^ + o <= F^ + e), so
// the dependency chain down a lane's rows is ONE operation per row; E^ and X
// depend only on the previous column.  The running max tracks X: an H = F^ > X
// lies strictly below an X of a row above, so max X = S and the cells holding S
// are the cells with X = S.  SW_XFORM=0 keeps the previous shifted-state update
// (E, F, H kept minus o; four dependent operations per row).
//
// Layout (B200-first, not ADEPT's block-per-pair / thread-per-residue):
// * a warp is split into 32/W segments of W lanes; a segment owns one (s32)
//   or two (s16x2: low / high halves) pairs;
// * lane L of a segment owns K consecutive query rows of the current stripe
//   (W*K rows per stripe) and sweeps the reference column by column, skewed by
//   one column per lane (anti-diagonal wavefront, PAPER.md:167-172 / Fig. 3);
// * the row above (H and F of the lane's neighbour) arrives by one full-mask
//   __shfl_up_sync per value per column -- no divergent shared-memory branch
//   and no block barrier per anti-diagonal (lessons of PAPER.md:530-560);
// * the substitution scores come from a per-stripe query profile in shared
//   memory: (s - o) as int8 per (code, lane, row); two LDS.128 per column
//   fetch all K rows of both halves, one PRMT per row interleaves and
//   sign-extends them into an s16x2 operand;
// * queries longer than W*K rows are processed as stripes; lane W-1 hands
//   the stripe's bottom row (HO, F) to lane 0 of the next stripe through a
//   per-warp global scratch row (L2-resident, no per-column conditions);
// * the argmax keeps, per lane and half, the first column where the lane's
//   running max improved (strict >) plus the HO values of that column, and
//   emits one 64-bit key (S, -j, -i) per lane with atomicMax -- the lexmin
//   (j, i) tie rule of reading R5 is associative, so lanes, halves and
//   stripes merge in any order;
// * REV mode runs the same kernel on the materialised reversed prefixes with
//   target S: a lane that reaches S emits immediately and the item stops one
//   segment-width after the first column holding S (reading R6).
#pragma once
#include "sw_common.cuh"
#include "sw_pack.cuh"

#define SV_QSTRIDE 512u  // bytes between quads of a saved column (32 lanes x 16 B), see Geometry::SVH
#define U_MAX_FILL 8     // >= the column unroll x loop-body blocks + the prefetch distance: the hand-off fill margin
#ifndef SW_CODE4
#define SW_CODE4 0         // 1 (measurement variant): DNA TAG forward reads 4-bit reference codes, 8 per word
#endif
#ifndef SW_COOP_STRIPES
#define SW_COOP_STRIPES 16 // reverse items with at least this many stripes are swept by all warps of a CTA (A/B 4-32: 16 best after the gap-aware band)
#endif
#ifndef SW_COOP_PUBLISH
#define SW_COOP_PUBLISH 32
#endif
#define COOP_PUBLISH SW_COOP_PUBLISH  // a cooperative producer publishes its hand-off progress every COOP_PUBLISH column steps

#ifndef SW_MIN_BLOCKS
#define SW_MIN_BLOCKS 4
#endif
#ifndef SW_MIN_BLOCKS_REV
#define SW_MIN_BLOCKS_REV SW_MIN_BLOCKS  // reverse-pass kernels (DNA / int32 geometry)
#endif
#ifndef SW_BODY_BLOCKS
#define SW_BODY_BLOCKS 2   // 4-column blocks per unrolled loop body (forward; chosen by tools/gevo_search.py)
#endif
#ifndef SW_XFORM
#define SW_XFORM 1         // 1: clamped-E/F update with a one-op row chain (four max operations, default);
                           // 2: three-max update, additions on the FMA pipe, a three-op row chain (measured
                           // slower: c2 forward 4.73 vs 4.90 TCUPS); 0: shifted-state update (see sweep<>)
#endif
#ifndef SW_IMPROVE_VOTE
#define SW_IMPROVE_VOTE 0  // 1: non-TAG forward with a warp-uniform improvement branch (vote) + predicated per-half
                           // stores (measured slower: c3 forward 3.14 vs 3.23 TCUPS, c5 3.63 vs 3.86)
#endif
#ifndef SW_IMERGE
#define SW_IMERGE 0        // 1: DNA TAG forward with a 32-bit-per-row profile, halves merged by one IMAD (FMA pipe)
#endif
#ifndef SW_PTAG
#define SW_PTAG 0          // 1 (measured slower): protein forward on the TAG route, 3-bit row tags, unsigned running max
#endif
#ifndef SW_PROT_T4
#define SW_PROT_T4 1       // protein profile build from a transposed (s - o) table with byte transposes
#endif
#ifndef SW_T4_ALL
#define SW_T4_ALL 0
#endif
#ifndef SW_TAG_LAZY
#define SW_TAG_LAZY 1      // TAG forward: branch-free block commit, column/row decode deferred to emit
#endif
#ifndef SW_SKEW2
#define SW_SKEW2 0         // 1: forward TAG sweep with a two-column skew per lane (sweep_skew2; measured slower)
#endif
#ifndef SW_PRED_IMPROVE
#define SW_PRED_IMPROVE 0     // non-TAG forward: record running-max improvements branch-free
#endif
#ifndef SW_REV_BODY_BLOCKS
#define SW_REV_BODY_BLOCKS 2  // reverse pass: the stop column is re-checked after every block either way (2 vs 1: c3 reverse 2.78 vs 2.94 ms, c4 8.75 vs 8.83, c5 47.6 vs 46.2)
#endif
// Launch bounds of the 8-row (protein) geometry: 3-warp blocks, 5 per SM by shared memory, so
// up to 136 registers per thread keep all 15 warps resident.
#ifndef SW_PROT_THREADS
#define SW_PROT_THREADS 96
#endif
#ifndef SW_PROT_BLOCKS
#define SW_PROT_BLOCKS 5
#endif
#ifndef SW_CODE_DIST
#define SW_CODE_DIST 4     // reference-code prefetch distance in columns
#endif
#ifndef SW_UNROLL
#define SW_UNROLL 4
#endif
#ifndef SW_ABLATE
#define SW_ABLATE 0        // timing experiments only (1: no improvement path, 2: no PRMT, 4: no stripe hand-off)
#endif
#ifndef SW_SINGLE_ONLY
#define SW_SINGLE_ONLY 0   // experiment: compile only the single-stripe sweep
#endif

namespace swb {

#ifndef SW_TRACE_ITEMS
#define SW_TRACE_ITEMS 0   // development builds only: per-item (route, pass, smid, start/end globaltimer, steps)
#endif
#if SW_TRACE_ITEMS
constexpr int TRACE_CAP = 1 << 21;
__device__ unsigned long long g_trace[TRACE_CAP][4];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

struct WaveParams {
    const uint8_t* qcode;       // query codes (positions qpos[p]; the reverse pass reads rows n-1 .. 0)
    const uint8_t* rcode;       // reference codes (padded positions rpos[p])
    const int64_t* qpos;        // query code position per pair
    const int64_t* rpos;        // reference code position per pair
    const int32_t* nlen;        // rows of each pair (forward: n, reverse: q_end+1)
    const int32_t* mlen;        // columns (forward: m, reverse: r_end+1)
    const int32_t* order;       // pair ids sorted by work key (routes in order TAG, S16, S32)
    const int32_t* counts;      // device: pairs per route for this pass
    const int32_t* pre;         // reverse pass: pairs ahead of the routes in the order (the banded ones), else null
    int route;                  // this launch's route
    const int32_t* target;      // reverse: forward score per pair
    unsigned long long* keys;   // per-pair atomicMax output
    int32_t* item_counter;      // work queue head (zeroed before launch)
    uint8_t* scratch;           // stripe hand-off rows
    int64_t scratch_seg_bytes;  // bytes of one segment x parity buffer
    unsigned long long* progress;  // per (warp, parity) hand-off row: CTA-cooperative reverse items (zeroed per call)
    unsigned long long* swept;  // cells swept (statistics)
    uint32_t tag_mul;           // = 64; a kernel parameter so the row tag is an IMAD (FMA pipe), not a LEA
    uint32_t one;               // = 1; a kernel parameter so H = Hb + o is an IMAD (FMA pipe), not an IADD3
    Scoring sc;
    const BatchStats* stats;    // whole-batch failure flags (batch_rejected)
    const uint32_t* rcode4;     // SW_CODE4 variant: the reference codes as nibbles (8 per word)
    uint32_t sixteen;           // = 16 (opaque: IMAD.HI extraction stays on the FMA pipe)
};

template <int W, int K, class T, bool IM = false>
struct Geometry {
    static constexpr int SEGS = 32 / W;
    static constexpr int SLOTS = SEGS * T::NH;
    static constexpr int ROWS = W * K;                       // rows per stripe
    // profile bytes per (slot, code, lane): int8 x K (s16x2) or int32 x K (s32), 16 B aligned
    // int8 profile: 4/8/16-byte entries (one LDS.32/.64/.128 per 4/8/16 rows); int32: 16-byte multiples
    // IM (SW_IMERGE, DNA TAG forward): one 32-bit word per row, the value in its half's 16 bits (8 B aligned:
    // LDS.64, conflict-free at a 40-byte lane stride)
    static constexpr int PB = IM ? 4 * K : (T::NH == 2) ? (K <= 4 ? 4 : K <= 8 ? 8 : 16 * ((K + 15) / 16)) : 16 * ((4 * K + 15) / 16);
    static constexpr int PWORDS = PB / 4;
    // saved improvement column per (lane, half); the lazy TAG commit keeps only (block start, raw max)
    static constexpr int SVB = IM ? 16 : 16 * ((4 * K + 15) / 16);
    // saved columns are stored quad-major across the warp's lanes: quad w of (half h, lane l) at
    // h * SVH + w * SV_QSTRIDE + l * 16, so a warp-wide STS.128 / LDS.128 touches 32 consecutive
    // 16-byte chunks (no bank conflicts; a lane-major 64-96 B stride conflicts 4-way)
    static constexpr int SVH = 32 * SVB;
    static __host__ __device__ int prof_bytes(int nc) { return SLOTS * nc * W * PB; }
    static constexpr int STOP_BYTES = 16 * ((SLOTS * 4 + 15) / 16);
    // shared memory per warp: profile + REV stop steps + saved improvement columns
    static __host__ __device__ int warp_smem(int nc) { return prof_bytes(nc) + STOP_BYTES + 32 * T::NH * SVB; }
};

// K 32-bit values kept as uint4 quads (so the improvement-column save can be
// vector stores straight from the registers).
template <int K>
struct Quads {
    uint4 q[(K + 3) / 4];
    __device__ __forceinline__ uint32_t& operator[](int r) {
        switch (r & 3) {
            case 0: return q[r >> 2].x;
            case 1: return q[r >> 2].y;
            case 2: return q[r >> 2].z;
            default: return q[r >> 2].w;
        }
    }
};
// Opaque copy of a value (keeps ptxas from turning `x * flag + b` back into a
// SEL on the ALU pipe: the multiply-add then issues on the FMA pipe).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

// Reference code byte into a full 32-bit register (read-only path).  An asm
// load keeps ptxas from packing the prefetched codes into shared registers
// with PRMT (ALU-pipe work on every column).
__device__ __forceinline__ uint32_t ld_code(const uint8_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// Saved HO words of an improvement column, kept in shared memory (one slot
// per lane and half; the full 32-bit words are stored, the half is picked at
// read time).  Predicated STS.128 instead of per-row LOP3 merges keeps this
// off the ALU pipe.
template <int K>
__device__ __forceinline__ void sv_store(uint32_t addr, const Quads<K>& HO) {
#pragma unroll
    for (int w = 0; w < K / 4; ++w)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(addr + SV_QSTRIDE * w), "r"(HO.q[w].x), "r"(HO.q[w].y),
                     "r"(HO.q[w].z), "r"(HO.q[w].w) : "memory");
    if (K % 4 >= 2)
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" :: "r"(addr + SV_QSTRIDE * (K / 4)), "r"(HO.q[K / 4].x),
                     "r"(HO.q[K / 4].y) : "memory");
    if (K % 4 == 1 || K % 4 == 3)
        asm volatile("st.shared.u32 [%0], %1;" :: "r"(addr + SV_QSTRIDE * (K / 4) + (K % 4 == 3 ? 8u : 0u)),
                     "r"(K % 4 == 1 ? HO.q[K / 4].x : HO.q[K / 4].z) : "memory");
}

template <int K>
__device__ __forceinline__ void sv_store_arr(uint32_t addr, const uint32_t (&v)[K]) {
    Quads<K> q;
#pragma unroll
    for (int r = 0; r < K; ++r) q[r] = v[r];
    sv_store<K>(addr, q);
}

// sv_store under a predicate (no branch): the stores issue always, write only where `cond` != 0.
template <int K>
__device__ __forceinline__ void sv_store_if(uint32_t addr, const uint32_t (&v)[K], uint32_t cond) {
#pragma unroll
    for (int w = 0; w < K / 4; ++w)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t@p st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}"
                     :: "r"(addr + SV_QSTRIDE * w), "r"(v[4 * w]), "r"(v[4 * w + 1]), "r"(v[4 * w + 2]), "r"(v[4 * w + 3]),
                     "r"(cond) : "memory");
    if (K % 4 >= 2)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p st.shared.v2.u32 [%0], {%1, %2};\n\t}"
                     :: "r"(addr + SV_QSTRIDE * (K / 4)), "r"(v[4 * (K / 4)]), "r"(v[4 * (K / 4) + 1]), "r"(cond) : "memory");
    if (K % 4 == 1 || K % 4 == 3)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}"
                     :: "r"(addr + SV_QSTRIDE * (K / 4) + (K % 4 == 3 ? 8u : 0u)), "r"(v[K - 1]), "r"(cond) : "memory");
}

// First row r of the saved column whose half h equals `target` (an HO value).
template <class T, int K>
__device__ __forceinline__ int sv_first_row(uint32_t addr, int h, int target) {
    int rr = 0;
#pragma unroll
    for (int w = (K + 3) / 4 - 1; w >= 0; --w) {
        const uint4 v = lds128(addr + SV_QSTRIDE * w);
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int b = 3; b >= 0; --b)
            if (4 * w + b < K && T::get(x[b], h) == target) rr = 4 * w + b;
    }
    return rr;
}

__device__ __forceinline__ unsigned long long pack_key(int S, int j, int i) {
    return ((unsigned long long)(uint32_t)S << 32) | ((unsigned long long)(0xffff - j) << 16) |
           (unsigned long long)(0xffff - i);
}

template <int R>
__device__ __forceinline__ uint4 lds_rem(uint32_t addr) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (R == 1) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v.x) : "r"(addr));
    if (R == 2) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}

// One stripe of one work item: the column sweep of the anti-diagonal
// wavefront for this lane's K rows of both halves.  MULTI adds the stripe
// hand-off (boundary row in from scratch, bottom row out to scratch).  EV
// (forward only) emits each half's result at its own last column; without EV
// every half emits after the sweep, which is exact when the item's
// references differ by at most the pad margin (the columns past a shorter
// reference are pad codes, whose cells stay below S).
template <class T, int W, int K, bool REV, bool MULTI, bool EV, bool TAG, bool LIN>
__device__ __forceinline__ int sweep(const WaveParams& P, const uint8_t* prof, volatile int* stop, const uint32_t sv_base,
                                      const int seg, const int L, const int s_lim, const int (&h_pid)[T::NH],
                                      const int (&h_m)[T::NH], const int (&h_tgt)[T::NH], const int64_t (&h_rpos)[T::NH],
                                      const int mmax, const int row0, const uint32_t o2, const uint32_t e2, const int o,
                                      const uint2* scr_in, uint2* scr_out, const bool from_scratch, const bool to_scratch,
                                      const int scr_cols, const int c_lo,
                                      const volatile unsigned long long* flag_in = nullptr, unsigned long long need_base = 0,
                                      volatile unsigned long long* flag_out = nullptr, unsigned long long pub_base = 0) {
    constexpr bool IM = SW_IMERGE && SW_TAG_LAZY && TAG && !REV && T::NH == 2 && K == 10;
    using G = Geometry<W, K, T, IM>;
    constexpr int NH = T::NH;
    constexpr int SLOTS = G::SLOTS;
    constexpr int U = TAG ? (K <= 16 ? 4 : 2) : SW_UNROLL;  // column unroll (codes prefetched one block ahead)
    constexpr int CS = W * G::PB;        // profile bytes per code
    const int nc = P.sc.nc;

    Quads<K> HO;   // H of the lane's rows at the previous column (plain, >= 0)
    uint32_t E[K]; // Eb = E - o of the lane's rows at the previous column (>= 0)
    const uint32_t o2s = T::splat(o);      // gap_open in every half
    // XF: HO holds R = H + o (column -1: H = 0), E holds max(E, 0); else HO holds H, E holds E - o
    const uint32_t R0 = SW_XFORM ? o2s : 0u;
#pragma unroll
    for (int r = 0; r < K; ++r) { HO[r] = R0; E[r] = 0u; }
    const uint32_t floor2 = T::splat(-o);  // Hb floor: H >= 0  <=>  Hb >= -o
    const uint32_t one = P.one;
    // TAG: the running max holds H*64 + (3 - u)*16 + (15 - r) for the cell of row r in the
    // u-th column of the current 4-column block, so the max itself names the first column of
    // the block and the smallest row holding it (reading R5).  Bookkeeping happens once per
    // block; afterwards the 6 tag bits are set to ones so a later column with the same H never
    // counts as an improvement.  Valid while H <= 511 (route eligibility).
    // 6 tag bits: RB for the row (K <= 2^RB), the rest for the column within the block.
    // PT (protein forward, SW_PTAG): 3 row bits and a commit every column, the running max taken
    // unsigned: X * 8 + tag <= 65535 while X <= 8191 (route rule max_s * n <= PTAG_MAX_SCORE)
    constexpr bool PT = SW_PTAG && TAG && !REV && K == 8 && K == SW_KP && NH == 2;
    static_assert(!PT || SW_TAG_LAZY, "protein TAG needs the lazy commit");
    constexpr int RB = PT ? 3 : K <= 16 ? 4 : 5;
    constexpr int UB = PT ? 0 : 6 - RB;
    constexpr int UC = PT ? 1 : U;  // columns per tag commit
    static_assert(!TAG || ((UC <= (1 << UB)) && K <= (1 << RB) && NH == 2), "TAG route geometry");
    constexpr uint32_t TAGSET = ((1u << (RB + UB)) - 1u) * 0x10001u;
    // tagged value of a half (unsigned for PT)
    auto tget = [](uint32_t v, int h) -> int { return PT ? (int)((v >> (16 * h)) & 0xffffu) : T::get(v, h); };
    uint32_t best = TAG ? TAGSET : 0u;
    int brow[NH];                        // TAG: row of the half's last improvement
    int bc[NH];                          // column of the last strict improvement, per half
    // TAG (lazy commit): block start column and raw block maximum of the half's last improving
    // block; decoded into bc / brow only when the half emits
    int bt0[NH];
    uint32_t btag[NH];
    uint32_t sv[NH];                     // shared address of the half's saved column
    int ev[NH];
    int next_ev = 0x7fffffff;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        bc[h] = 0;
        brow[h] = 0;
        bt0[h] = 0;
        btag[h] = 0u;
        sv[h] = sv_base + (uint32_t)h * G::SVH;
        ev[h] = (EV && h_pid[h] >= 0) ? L + h_m[h] - 1 : 0x7fffffff;
        next_ev = min(next_ev, ev[h]);
    }
    uint32_t hoLast = R0, fLast = 0u, prevUpHO = R0;
    uint32_t prof_h[NH];  // shared-window address of this lane's profile entries, code 0
    const uint8_t* rp[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        prof_h[h] = (uint32_t)__cvta_generic_to_shared(prof + (size_t)(seg * NH + h) * nc * CS + (size_t)L * G::PB);
        rp[h] = P.rcode + h_rpos[h] - L + c_lo;  // this lane's first column c_lo (pad codes before column 0)
    }
    const uint32_t cs = opaque(CS);  // code stride as a runtime value: the address is one IMAD
    // lane 0 takes the row above from the stripe boundary: up = shfl * notL0 + b (IMAD)
    const uint32_t notL0 = opaque(L != 0 ? 1u : 0u);
    // lane 0's row above at the top of the query (H = 0, F = -inf clamped): XF (R = o, F = 0),
    // else (H = 0, Fb = 0); other lanes add 0 to the shuffled value
    const uint32_t b0 = (SW_XFORM && L == 0) ? o2s : 0u;

    auto emit = [&](int h) {  // forward result of half h for this lane and stripe
        const int b = TAG ? (tget(best, h) >> (RB + UB)) : T::get(best, h);
        if (TAG && SW_TAG_LAZY) {
            uint32_t t0s, raw;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t0s), "=r"(raw) : "r"(sv[h]) : "memory");
            bt0[h] = (int)t0s;
            btag[h] = raw;
            const int v = tget(btag[h], h);
            bc[h] = bt0[h] + (UC - 1 - ((v >> RB) & ((1 << UB) - 1))) - L;
            brow[h] = ((1 << RB) - 1) - (v & ((1 << RB) - 1));
        }
        if (h_pid[h] >= 0 && b > 0) {
            const int rr = TAG ? brow[h] : sv_first_row<T, K>(sv[h], h, b);
            atomicMax(P.keys + h_pid[h], pack_key(b, bc[h], row0 + L * K + rr));
        }
    };
    // TAG: fold the block's running max into the per-half records (block start column t0)
    auto tag_commit = [&](uint32_t nbt, int t0) {
        const uint32_t d = nbt ^ best;
        if (SW_TAG_LAZY) {
            // branch-free: two compares and predicated moves (FMA-pipe IMAD.MOV); the decode of
            // column and row from the raw maximum waits for emit()
            // per half: record (block start, raw maximum) in the half's shared slot when it changed
            // (predicated STS on the LSU pipe instead of SELs on the saturated ALU pipe)
            asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %3, 0;\n\tsetp.ge.u32 q, %4, 65536;\n\t"
                         "@p st.shared.v2.u32 [%0], {%2, %5};\n\t@q st.shared.v2.u32 [%1], {%2, %5};\n\t}"
                         :: "r"(sv[0]), "r"(sv[NH - 1]), "r"(t0), "r"(d << 16), "r"(d), "r"(nbt) : "memory");
            best = nbt | TAGSET;
            return;
        }
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            if ((d >> (16 * h)) & 0xffffu) {
                const int v = T::get(nbt, h);
                bc[h] = t0 + (U - 1 - ((v >> RB) & ((1 << UB) - 1))) - L;
                brow[h] = ((1 << RB) - 1) - (v & ((1 << RB) - 1));
            }
        }
        best = nbt | TAGSET;
    };

    // rotating prefetch of the next U columns' codes (and boundary rows)
    constexpr int CD = SW_CODE_DIST < U ? SW_CODE_DIST : U;  // code prefetch distance (columns)
    // the prefetch ring is indexed u % CD within a U-column block: CD must divide U (a distance of 3
    // with U = 4 reads wrong codes -- the variant search's parity gate rejected it)
    static_assert(U % CD == 0, "SW_CODE_DIST must divide the column unroll");
    uint32_t cd[CD][NH];
    uint2 bnd[U];
    // CTA-cooperative reverse item: the previous stripe's producer (another warp) publishes how many
    // columns of its hand-off row are written (absolute, exclusive) with release semantics; this
    // warp waits before loading columns it has not published (see the kernel)
    unsigned long long seen = 0;
    auto wait_cols = [&](int col_excl) {
        if (MULTI && flag_in) {
            const unsigned long long need = need_base | (unsigned long long)min(col_excl, 0x1fffff);
            if (seen < need) {
                do {
                    seen = *flag_in;
                } while (seen < need);
                __threadfence();  // acquire: the row is read after the flag
            }
        }
    };
    wait_cols(c_lo + U);
    // diagonal input of lane 0's first column: the left border, or -- for a reverse stripe that starts
    // at c_lo > 0 -- the previous stripe's bottom row at column c_lo - 1 (inside that row's band)
    if (MULTI && from_scratch && L == 0 && c_lo > 0) prevUpHO = __ldcg(scr_in - 1).x;
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int h = 0; h < NH; ++h)
            if (u < CD) cd[u][h] = ld_code(rp[h] + u);
        if (MULTI) bnd[u] = __ldcg(scr_in + u);
    }
    // Stripe hand-off without per-column conditions: every lane of a segment loads lane 0's
    // boundary word (one broadcast LDG), and an IMAD keeps it only where it applies -- lane 0 of
    // a stripe below the first -- else the constant border b0 (lane 0 of the first stripe) or 0
    // (the other lanes, which take the row above from the shuffle).  The producing stripe filled
    // every column it did not sweep with the border (see the kernel), so no stale value is ever
    // read; the store is predicated on a loop-invariant lane test into a row with W slots of slack
    // before column 0.
    const uint32_t useL0 = opaque((MULTI && from_scratch && L == 0) ? 1u : 0u);
    const uint32_t bconst = (MULTI && from_scratch) ? 0u : b0;
    const bool st_lane = MULTI && to_scratch && L == W - 1;

    // reverse pass: packed targets of both halves (the forward score S of each pair); the
    // TAG route compares block maxima against S*64 (0x7fff: half finished or empty)
    uint32_t tgt2 = 0, tgt64 = 0;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        tgt2 = T::set(tgt2, h, h_pid[h] >= 0 ? h_tgt[h] : -1);
        if (TAG && REV) tgt64 = T::set(tgt64, h, h_pid[h] >= 0 ? h_tgt[h] * 64 : 0x7fff);
    }
    int found_blk = 0;
    // TAG reverse pass: some half's block maximum reached S*64.  Every cell of the reversed
    // rectangle has H <= S, so the block's first cell holding S is named by the tag (reading R6);
    // a maximum above S can only come from the code bytes past the rectangle (past the pad run
    // finish_fwd writes after the reversed prefix), i.e. after the half's true first S column.
    auto rev_tag_find = [&](uint32_t nbt_, int t0) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            const int v = T::get(nbt_, h);
            if (v >= T::get(tgt64, h)) {
                const int col = t0 + (U - 1 - ((v >> RB) & ((1 << UB) - 1))) - L;
                if ((v >> 6) == h_tgt[h] && col + c_lo < h_m[h]) {
                    atomicMax(P.keys + h_pid[h], pack_key(h_tgt[h], col + c_lo, row0 + L * K + ((1 << RB) - 1) - (v & ((1 << RB) - 1))));
                    atomicMin((int*)stop + seg * NH + h, col + c_lo + W);
                }
                tgt64 = T::set(tgt64, h, 0x7fff);
                found_blk = 1;
            }
        }
    };
    int T_end = mmax + W - 1;
    if (REV) {
        // steps until every lane passed each slot's last needed column (its reversed reference, its
        // band, or its found start: stop), in steps from column c_lo
        int te = 0;
#pragma unroll
        for (int sl = 0; sl < SLOTS; ++sl) te = max(te, min(__shfl_sync(FULL, s_lim, sl), stop[sl]));
        T_end = te - c_lo;
    }
    // NB blocks of U columns per loop iteration (the longer body lets ptxas keep loop-carried
    // values in place); tag bookkeeping stays per U-column block
    constexpr int NB = REV ? SW_REV_BODY_BLOCKS : SW_BODY_BLOCKS;
    // SW_CODE4 (measurement variant, DNA TAG forward): the block's four codes per half come from two
    // words of 4-bit codes prefetched one block ahead and one funnel shift; a code is extracted on the
    // FMA pipe (shift left by IMAD, high word of a multiply by 16)
    constexpr bool C4 = SW_CODE4 && TAG && !REV && NH == 2 && U == 4;
    int64_t x4[NH];
    uint32_t wa[NH], wb[NH], v4[NH];
    if (C4) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            x4[h] = h_rpos[h] - L + c_lo;
            wa[h] = __ldg(P.rcode4 + (x4[h] >> 3));
            wb[h] = __ldg(P.rcode4 + (x4[h] >> 3) + 1);
        }
    }
    const uint32_t sixteen = C4 ? P.sixteen : 16u;
    int t00 = 0;
    for (; t00 < T_end; t00 += U * NB) {
      wait_cols(c_lo + t00 + U * NB + U);
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        const int t0 = t00 + bb * U;
        uint32_t nbt = REV ? 0u : best;  // TAG: running max of this block
        if (C4) {
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const int64_t x0 = x4[h] + t0;
                v4[h] = __funnelshift_r(wa[h], wb[h], (uint32_t)(x0 & 7) * 4u);
                const int64_t x1 = x0 + U;
                wa[h] = __ldg(P.rcode4 + (x1 >> 3));
                wb[h] = __ldg(P.rcode4 + (x1 >> 3) + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u;
            // query-profile words of this lane's column (all K rows, both halves)
            uint32_t pw[NH][G::PWORDS];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const uint32_t code = C4 ? __umulhi(v4[h] << (28 - 4 * u), sixteen) : cd[u % CD][h];
                if (IM) {
                    const uint32_t src = prof_h[h] + code * cs;
#pragma unroll
                    for (int q2 = 0; q2 < K / 2; ++q2) {
                        uint32_t a, b;
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(src + 8 * q2));
                        pw[h][2 * q2] = a;
                        pw[h][2 * q2 + 1] = b;
                    }
                    cd[u % CD][h] = ld_code(rp[h] + t + CD);
                    continue;
                }
#ifdef SW_BAND_CHECK
                if (SW_BAND_CHECK && code >= (uint32_t)nc) {
                    printf("wave code %u >= nc: REV %d route %d pid %d t %d L %d\n", code, (int)REV, P.route, h_pid[h], t, L);
                    __trap();
                }
#endif
                const uint32_t src = prof_h[h] + code * cs;
                if (G::PWORDS >= 4) {
#pragma unroll
                    for (int q4 = 0; q4 < G::PWORDS / 4; ++q4) {
                        const uint4 v = lds128(src + 16 * q4);
                        pw[h][q4 * 4 + 0] = v.x; pw[h][q4 * 4 + 1] = v.y;
                        pw[h][q4 * 4 + 2] = v.z; pw[h][q4 * 4 + 3] = v.w;
                    }
                } else {
                    const uint4 v = lds_rem<G::PWORDS>(src);
                    pw[h][0] = v.x;
                    if (G::PWORDS > 1) pw[h][G::PWORDS - 1] = v.y;
                }
                if (!C4) cd[u % CD][h] = ld_code(rp[h] + t + CD);
            }
            uint32_t bHO = b0, bF = 0u;
            if (MULTI) {
                bHO = bnd[u].x * useL0 + bconst;  // IMAD (FMA pipe)
                bF = bnd[u].y * useL0;
                if (!(SW_ABLATE & 4)) bnd[u] = __ldcg(scr_in + t + U);  // (ablation 4: timing only, no hand-off)
            }
            // row above: neighbour lane's last row at this column, or the stripe boundary (lane 0)
            const uint32_t upHO = __shfl_up_sync(FULL, hoLast, 1, W) * notL0 + bHO;
            const uint32_t upF = LIN ? 0u : __shfl_up_sync(FULL, fLast, 1, W) * notL0 + bF;
            uint32_t hd = prevUpHO;
            prevUpHO = upHO;
            uint32_t F = upF, hu = upHO;
            uint32_t H[K];  // per row: the value the running max tracks (XF: X, else H), TAG-tagged
#pragma unroll
            for (int r = 0; r < K; ++r) {
                uint32_t sc;
                if (NH == 2 && (SW_ABLATE & 2)) {
                    sc = pw[r & 1][r >> 2];  // timing ablation only: wrong scores
                } else if (IM) {
                    sc = pw[NH - 1][r] * one + pw[0][r];  // IMAD: halves' 16-bit values, no carry
                } else if (NH == 2) {
                    constexpr uint32_t SEL[4] = {0xC480u, 0xD591u, 0xE6A2u, 0xF7B3u};
                    sc = prmt(pw[0][r >> 2], pw[NH - 1][r >> 2], SEL[r & 3]);
                } else {
                    sc = pw[0][r];
                }
                uint32_t xv;
                if (LIN) {
                    // linear gaps (gap_open == gap_extend = e): with R = H + e,
                    //   A[i][j] = max(R[i-1][j-1] + (s - e), R[i][j-1], 0)     VIADDMNMX.RELU
                    //   H[i][j] = max(A[i][j], R[i-1][j])                      VIMNMX
                    //   R[i][j] = H[i][j] + e                                  VIADD.16x2 (FMA pipe)
                    // (the affine recurrence with o = e: E[i][j] = H[i][j-1] + e since E <= H).
                    // The running max tracks A: H = R[i-1][j] > A lies below a larger H (e < 0).
                    xv = T::addmax_relu(hd, sc, HO[r]);
                    hd = HO[r];
                    HO[r] = T::add(T::max2(xv, hu), o2s);
                    hu = HO[r];
                } else if (SW_XFORM == 3) {
                    // Three-max form with a two-operation row chain: F of the row below is formed as
                    // soon as H of this row exists, max(H + o, F + e), with F + e added off the chain
                    //   t        = R[i-1][j-1] + (s - o)                           VIADD.16x2 (FMA pipe)
                    //   E[i][j]  = max(E[i][j-1] + e, R[i][j-1])                    VIADDMNMX
                    //   H[i][j]  = max(t, E, F[i][j], 0)                            VIMNMX3.RELU
                    //   F[i+1][j] = max(H[i][j] + o, F[i][j] + e)                   VIADDMNMX (+ VIADD, FMA)
                    //   R[i][j]  = H + o                                            VIADD.16x2 (FMA pipe)
                    // F of the lane's first row is max(F_up + e, R_up) as in the forms below; F keeps
                    // the last row's value for the hand-off (the next lane forms its first row's F).
                    const uint32_t tt = T::add(hd, sc);
                    E[r] = T::addmax(E[r], e2, HO[r]);
                    if (r == 0) F = T::addmax(F, e2, hu);
                    xv = T::max3(tt, E[r], F);
                    if (r + 1 < K) F = T::addmax(xv, o2s, T::add(F, e2));
                    hd = HO[r];
                    HO[r] = T::add(xv, o2s);
                    hu = HO[r];
                } else if (SW_XFORM == 2) {
                    // Three-max form (R = H + o kept per row, as below; E and F unclamped, bounded
                    // below by o since R >= o):
                    //   t        = R[i-1][j-1] + (s - o)                           VIADD.16x2 (FMA pipe)
                    //   E[i][j]  = max(E[i][j-1] + e, R[i][j-1])                    VIADDMNMX
                    //   F[i][j]  = max(F[i-1][j] + e, R[i-1][j])                    VIADDMNMX
                    //   H[i][j]  = max(t, E, F, 0)                                  VIMNMX3.RELU
                    //   R[i][j]  = H + o                                            VIADD.16x2 (FMA pipe)
                    // which is the Gotoh recurrence of the header with the borders E = F = o or 0
                    // (<= o - e, so they never win a max that matters: reading R13 / pin P13).  Three
                    // ALU max operations per cell pair instead of four (the additions ride the FMA
                    // pipe); the row chain is F -> H -> R (three operations).  The running max
                    // tracks H itself (>= 0; its cells equal to S are those of X in the form below).
                    const uint32_t tt = T::add(hd, sc);
                    E[r] = T::addmax(E[r], e2, HO[r]);
                    F = T::addmax(F, e2, hu);
                    xv = T::max3(tt, E[r], F);
                    hd = HO[r];
                    HO[r] = T::add(xv, o2s);
                    hu = HO[r];
                } else if (SW_XFORM) {
                    // E^ = max(E, 0), F^ = max(F, 0), X = max(H[i-1][j-1] + s, E^) (>= 0), R = H + o:
                    //   E^[i][j] = max(E^[i][j-1] + e, R[i][j-1], 0)          VIADDMNMX.RELU
                    //   X[i][j]  = max(R[i-1][j-1] + (s - o), E^[i][j])       VIADDMNMX
                    //   F^[i][j] = max(F^[i-1][j] + e, X[i-1][j] + o, 0)      VIADDMNMX.RELU (the row chain)
                    //   R[i][j]  = max(F^[i][j] + o, X[i][j] + o)             VIADDMNMX (+ VIADD.16x2, FMA pipe)
                    // H = max(X, F^); F^ feeds F^ of the next row through X + o only (o <= e), so the
                    // dependency chain down a lane's rows is one operation per row.  The running max
                    // tracks X: every H = F^ > X lies strictly below some X of a row above, so max X = S
                    // and the cells with H = S are exactly those with X = S.
                    E[r] = T::addmax_relu(E[r], e2, HO[r]);
                    xv = T::addmax(hd, sc, E[r]);
                    F = T::addmax_relu(F, e2, hu);
                    const uint32_t xo = T::add(xv, o2s);
                    hd = HO[r];
                    HO[r] = T::addmax(F, o2s, xo);
                    hu = xo;
                } else {
                    E[r] = T::addmax(E[r], e2, HO[r]);          // Eb[i][j] = max(Eb[i][j-1] + e, H[i][j-1])
                    F = T::addmax(F, e2, hu);                   // Fb[i][j] = max(Fb[i-1][j] + e, H[i-1][j])
                    const uint32_t tt = T::max3(E[r], F, floor2);  // max(E, F, 0) - o
                    const uint32_t hb = T::addmax(hd, sc, tt);  // max(H[i-1][j-1] + s, E, F, 0) - o
                    hd = HO[r];
                    HO[r] = hb * one + o2;                      // H = Hb + o: one IMAD, no borrow (Hb >= -o)
                    hu = HO[r];
                    xv = HO[r];
                }
                // TAG: value*64 + tag per half, one IMAD on the FMA pipe (value <= 511: no carry)
                H[r] = TAG ? xv * P.tag_mul + (uint32_t)((PT ? 0 : (U - 1 - u) * (1 << RB)) + (1 << RB) - 1 - r) * 0x10001u : xv;
            }
            hoLast = HO[K - 1];
            fLast = F;
            // running max over the lane's rows; strict improvement -> remember column + HO values
            if (PT) {
#pragma unroll
                for (int r = 0; r + 1 < K; r += 2) nbt = __vimax3_u16x2(nbt, H[r], H[r + 1]);
                tag_commit(nbt, t);  // every column (the tag names the row only)
                nbt = best;
            } else if (TAG) {
#pragma unroll
                for (int r = 0; r + 1 < K; r += 2) nbt = T::max3(nbt, H[r], H[r + 1]);
                if (K & 1) nbt = T::max2(nbt, H[K - 1]);
            } else {
                uint32_t nb = REV ? H[0] : best;
#pragma unroll
                for (int r = REV ? 1 : 0; r + 1 < K; r += 2) nb = T::max3(nb, H[r], H[r + 1]);
                if ((K & 1) != (REV ? 1 : 0)) nb = T::max2(nb, H[K - 1]);
                if (REV) {
                    // reverse pass: only cells equal to S matter (reading R6).  nb is this column's max;
                    // a half whose target was found gets the unreachable target -1.
                    const uint32_t x = nb ^ tgt2;
                    if (NH == 1 ? x == 0u : (((x & 0xffffu) == 0u) || ((x >> 16) == 0u))) {
#pragma unroll
                        for (int h = 0; h < NH; ++h) {
                            if (((x >> (16 * h)) & (NH == 1 ? 0xffffffffu : 0xffffu)) == 0u && h_pid[h] >= 0) {
                                int rr = 0;
                                // whole-word compare under the half's mask (no 16-bit extraction, which
                                // makes ptxas split the row values into 16-bit pieces in the hot path)
                                const uint32_t tw = T::splat(h_tgt[h]);
                                const uint32_t msk = NH == 1 ? 0xffffffffu : (h ? 0xffff0000u : 0x0000ffffu);
#pragma unroll
                                for (int r = K - 1; r >= 0; --r) if (((H[r] ^ tw) & msk) == 0u) rr = r;
                                atomicMax(P.keys + h_pid[h], pack_key(h_tgt[h], t - L + c_lo, row0 + L * K + rr));
                                atomicMin((int*)stop + seg * NH + h, t - L + c_lo + W);
                                tgt2 = T::set(tgt2, h, -1);
                                found_blk = 1;
                            }
                        }
                    }
                } else if (SW_ABLATE & 1) {
                    best = nb;  // timing ablation only: no improvement bookkeeping
                } else if (SW_PRED_IMPROVE && SW_XFORM) {
                    // branch-free: per half, predicated stores of the column's values and a
                    // predicated column update where the half's running max improved
                    const uint32_t d = nb ^ best;
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        const uint32_t dh = NH == 1 ? d : (h ? d >> 16 : d & 0xffffu);
                        sv_store_if<K>(sv[h], H, dh);
                        bc[h] = dh ? t - L : bc[h];
                    }
                    best = nb;
                } else if (SW_IMPROVE_VOTE && SW_XFORM) {
                    // warp-uniform branch (no divergence bookkeeping): when some lane's running max
                    // improved, every lane issues predicated stores of the column for the halves
                    // that improved and moves their column record
                    const uint32_t d = nb ^ best;
                    if (__any_sync(FULL, d != 0u)) {
#pragma unroll
                        for (int h = 0; h < NH; ++h) {
                            const uint32_t dh = NH == 1 ? d : (h ? d >> 16 : d & 0xffffu);
                            sv_store_if<K>(sv[h], H, dh);
                            bc[h] = dh ? t - L : bc[h];
                        }
                    }
                    best = nb;
                } else if (nb != best) {
                    const uint32_t d = nb ^ best;
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        if (NH == 1 || ((d >> (16 * h)) & 0xffffu)) {
                            bc[h] = t - L;
                            if (SW_XFORM) sv_store_arr<K>(sv[h], H); else sv_store<K>(sv[h], HO);
                        }
                    }
                    best = nb;
                }
            }
            if (EV && t == next_ev) {
                if (TAG && !PT) tag_commit(nbt, t0);  // make best / bc / brow current before emitting
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    if (ev[h] == t) {
                        emit(h);
                        best = T::set(best, h, PT ? 0xffff : T::FROZEN);
                        ev[h] = 0x7fffffff;
                    }
                }
                if (TAG) nbt = best;
                next_ev = ev[0];
                if (NH == 2) next_ev = min(next_ev, ev[NH - 1]);
            }
            if (st_lane && !(SW_ABLATE & 4)) scr_out[t - (W - 1)] = make_uint2(hoLast, fLast);
        }
        if (TAG && !PT && !REV && (SW_TAG_LAZY || nbt != best)) tag_commit(nbt, t0);
        if (TAG && REV) {
            const uint32_t x = T::max2(nbt, tgt64) ^ nbt;  // zero half: block max >= S*64
            if (((x - 0x00010001u) & ~x & 0x80008000u) != 0u) rev_tag_find(nbt, t0);
        }
        if (MULTI && flag_out && ((t0 + U) % COOP_PUBLISH) == 0) {
            // release: this stripe's row is written up to column c_lo + t0 + U - W + 1 (exclusive)
            __threadfence();
            __syncwarp();
            __threadfence();
            if (L == 0 && seg == 0) *flag_out = pub_base | (unsigned long long)max(0, c_lo + t0 + U - W + 1);
        }
        if (REV && __any_sync(FULL, found_blk)) {  // re-read the stop columns only after a find
            __syncwarp();
            int te = 0;
#pragma unroll
            for (int sl = 0; sl < SLOTS; ++sl) te = max(te, min(__shfl_sync(FULL, s_lim, sl), stop[sl]));
            T_end = te - c_lo;
            found_blk = 0;
        }
      }
    }
    if (!REV && !EV) {
#pragma unroll
        for (int h = 0; h < NH; ++h) emit(h);
    }
    if (MULTI && to_scratch) {
        // Columns this sweep did not hand off (it wrote [-(W-1), t00 - W + 1)): the border, so the
        // next stripe never reads a row left by an earlier item -- a reverse sweep stops early
        // (reading R6) while the next stripe may still sweep further for another half of the item
        // (the round-1 soak failure).  The border is a lower bound of the true
        // row (H is monotone in it); it only feeds columns the early stop already settled or cells
        // of a half's own rectangle / pad run, where H <= S.
        __syncwarp();
        for (int c = t00 - (W - 1) + L; c < scr_cols; c += W) scr_out[c] = make_uint2(R0, 0u);
        if (flag_out) {  // the whole row (swept and border-filled) is readable
            __threadfence();
            __syncwarp();
            __threadfence();
            if (L == 0 && seg == 0) *flag_out = pub_base | 0x1fffffull;
        }
    }
    return t00;  // column steps swept (statistics)
}

// Forward TAG sweep with a two-column skew per lane (single stripe, no end events): lane L's
// upper rows 0..4 work on column t - 2L while its lower rows 5..9 work on column t - 2L - 1.
// The lower rows need this lane's row 4 from the previous step and the row above (the previous
// lane's row 9) arrives from the previous step as before, so within a step the two 5-row chains
// are independent: half the dependent-chain length per column step for the same instruction
// count, at the price of W more fill/drain steps.  The tag of a cell orders lower rows before
// upper rows of the same step (their column is one smaller), so the block maximum still names
// the lexmin (j, i) cell (reading R5).
template <class T, int W, int K>
__device__ __forceinline__ int sweep_skew2(const WaveParams& P, const uint8_t* prof, const int seg, const int L,
                                           const int (&h_pid)[T::NH], const int64_t (&h_rpos)[T::NH], const int mmax,
                                           const int row0, const uint32_t o2, const uint32_t e2, const int o) {
    using G = Geometry<W, K, T>;
    constexpr int NH = T::NH;
    static_assert(NH == 2 && K == 10 && G::PWORDS == 4, "two-column skew: s16x2, 10 rows per lane");
    constexpr int KU = 5;                 // upper rows 0..4, lower rows 5..9
    constexpr int U = 4;                  // column steps per tag block
    constexpr int NB = SW_BODY_BLOCKS;
    constexpr int CS = W * G::PB;
    constexpr int CD = SW_CODE_DIST < U ? SW_CODE_DIST : U;
    static_assert(U % CD == 0, "SW_CODE_DIST must divide the column unroll");
    constexpr uint32_t TAGSET = 0x003f003fu;
    constexpr uint32_t SEL[4] = {0xC480u, 0xD591u, 0xE6A2u, 0xF7B3u};
    const int nc = P.sc.nc;

    Quads<K> HO;
    uint32_t E[K];
#pragma unroll
    for (int r = 0; r < K; ++r) { HO[r] = 0u; E[r] = 0u; }
    const uint32_t floor2 = T::splat(-o);
    const uint32_t one = P.one;
    uint32_t best = TAGSET;
    int brow[NH], bc[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) { brow[h] = 0; bc[h] = 0; }
    uint32_t prof_h[NH];
    const uint8_t* rp[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        prof_h[h] = (uint32_t)__cvta_generic_to_shared(prof + (size_t)(seg * NH + h) * nc * CS + (size_t)L * G::PB);
        rp[h] = P.rcode + h_rpos[h] - 2 * L;  // this lane's upper column 0 (pad codes before it)
    }
    const uint32_t cs = opaque(CS);
    const uint32_t notL0 = opaque(L != 0 ? 1u : 0u);
    uint32_t hoLast = 0u, fLast = 0u, prevUpHO = 0u;  // lower row 9 (previous step); row above's diagonal
    uint32_t f4 = 0u, ho4pp = 0u;                     // row 4's F (previous step), row 4's H two steps back
    uint32_t pwl[NH][2];                              // previous step's profile words 1, 2 (rows 4..11)
#pragma unroll
    for (int h = 0; h < NH; ++h) {                    // step 0's lower column is a pad column
        const uint4 v = lds128(prof_h[h] + (uint32_t)(nc - 1) * cs);
        pwl[h][0] = v.y; pwl[h][1] = v.z;
    }
    uint32_t cd[CD][NH];
#pragma unroll
    for (int u = 0; u < CD; ++u)
#pragma unroll
        for (int h = 0; h < NH; ++h) cd[u][h] = ld_code(rp[h] + u);

    // decode a block maximum v (one half): column and row of its cell
    auto decode = [&](int v, int t0, int& col, int& row) {
        const int step = t0 + (U - 1 - ((v >> 4) & 3));
        const int rho = 15 - (v & 15);
        if (rho < KU) { row = rho + KU; col = step - 2 * L - 1; }
        else { row = rho - KU; col = step - 2 * L; }
    };
    auto tag_commit = [&](uint32_t nbt, int t0) {
        const uint32_t d = nbt ^ best;
#pragma unroll
        for (int h = 0; h < NH; ++h)
            if ((d >> (16 * h)) & 0xffffu) decode(T::get(nbt, h), t0, bc[h], brow[h]);
        best = nbt | TAGSET;
    };

    const int T_end = mmax + 2 * W - 1;
    int t00 = 0;
    for (; t00 < T_end; t00 += U * NB) {
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
            const int t0 = t00 + bb * U;
            uint32_t nbt = best;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + u;
                uint32_t pw[NH][4];
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    const uint4 v = lds128(prof_h[h] + cd[u % CD][h] * cs);
                    pw[h][0] = v.x; pw[h][1] = v.y; pw[h][2] = v.z; pw[h][3] = v.w;
                    cd[u % CD][h] = ld_code(rp[h] + t + CD);
                }
                const uint32_t upHO = __shfl_up_sync(FULL, hoLast, 1, W) * notL0;
                const uint32_t upF = __shfl_up_sync(FULL, fLast, 1, W) * notL0;
                uint32_t H[K];
                // lower rows 5..9, column t - 2L - 1 (profile words of the previous step)
                {
                    uint32_t hd = ho4pp, hu = HO[4], F = f4;
#pragma unroll
                    for (int r = KU; r < K; ++r) {
                        const uint32_t sc = prmt(pwl[0][(r >> 2) - 1], pwl[NH - 1][(r >> 2) - 1], SEL[r & 3]);
                        E[r] = T::addmax(E[r], e2, HO[r]);
                        F = T::addmax(F, e2, hu);
                        const uint32_t tt = T::max3(E[r], F, floor2);
                        const uint32_t hb = T::addmax(hd, sc, tt);
                        hd = HO[r];
                        HO[r] = hb * one + o2;
                        hu = HO[r];
                        H[r] = HO[r] * P.tag_mul + (uint32_t)((U - 1 - u) * 16 + 15 - (r - KU)) * 0x10001u;
                    }
                    hoLast = HO[K - 1];
                    fLast = F;
                }
                ho4pp = HO[4];
                // upper rows 0..4, column t - 2L
                {
                    uint32_t hd = prevUpHO, hu = upHO, F = upF;
                    prevUpHO = upHO;
#pragma unroll
                    for (int r = 0; r < KU; ++r) {
                        const uint32_t sc = prmt(pw[0][r >> 2], pw[NH - 1][r >> 2], SEL[r & 3]);
                        E[r] = T::addmax(E[r], e2, HO[r]);
                        F = T::addmax(F, e2, hu);
                        const uint32_t tt = T::max3(E[r], F, floor2);
                        const uint32_t hb = T::addmax(hd, sc, tt);
                        hd = HO[r];
                        HO[r] = hb * one + o2;
                        hu = HO[r];
                        H[r] = HO[r] * P.tag_mul + (uint32_t)((U - 1 - u) * 16 + 15 - (r + KU)) * 0x10001u;
                    }
                    f4 = F;
                }
#pragma unroll
                for (int h = 0; h < NH; ++h) { pwl[h][0] = pw[h][1]; pwl[h][1] = pw[h][2]; }
#pragma unroll
                for (int r = 0; r + 1 < K; r += 2) nbt = T::max3(nbt, H[r], H[r + 1]);
            }
            if (nbt != best) tag_commit(nbt, t0);
        }
    }
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        const int b = T::get(best, h) >> 6;
        if (h_pid[h] >= 0 && b > 0) atomicMax(P.keys + h_pid[h], pack_key(b, bc[h], row0 + L * K + brow[h]));
    }
    return t00;
}

template <class T, int W, int K, bool REV, bool TAG, bool LIN>
__global__ void __launch_bounds__((K == SW_KP && W == SW_WP) ? SW_PROT_THREADS : 128, (K == SW_KP && W == SW_WP) ? SW_PROT_BLOCKS : REV ? SW_MIN_BLOCKS_REV : SW_MIN_BLOCKS)
    wavefront_kernel(const WaveParams P) {
    constexpr bool IMK = SW_IMERGE && SW_TAG_LAZY && TAG && !REV && T::NH == 2 && K == 10;
    using G = Geometry<W, K, T, IMK>;
    constexpr int NH = T::NH;
    constexpr int SLOTS = G::SLOTS;
    // Row/column tags (H*64 + tag) need H <= 511 in every computed cell, also past a half's
    // reference: the TAG route takes pairs with max_s * n <= 511 (pack), which bounds every
    // cell of the query's rows whatever the columns hold (end events, reverse pass alike).
    constexpr bool TAGF = TAG;
    extern __shared__ __align__(16) uint8_t smem[];
    if (batch_rejected(P.stats)) return;  // nothing of this call was packed (uniform over the grid)
    // substitution table for the profile builds, in shared memory: lanes index it with
    // divergent codes, which a constant-bank table would serialise
    __shared__ int8_t s_sigma[24 * 24];
    // protein s16x2 profiles: (s - o) bytes of query residue a against codes 4q..4q+3 in word
    // s_t4[a][q]; row a = 24 is the pad residue (-128 against every code), code 24 the pad code
    constexpr int TQ = (NC_PROTEIN + 3) / 4;
    __shared__ uint32_t s_t4[SW_T4_ALL || K == SW_KP ? 25 * TQ : 1];  // K == SW_KP: the protein geometry
    for (int k = threadIdx.x; k < 24 * 24; k += blockDim.x) {
        const int a = k / 24, b = k % 24;
        s_sigma[k] = (int8_t)(P.sc.alphabet == SW_ALPHABET_DNA ? 0 : c_blosum62[a][b]);
    }
    if (NH == 2 && (SW_T4_ALL || K == SW_KP) && P.sc.alphabet != SW_ALPHABET_DNA) {
        for (int k = threadIdx.x; k < 25 * TQ; k += blockDim.x) {
            const int a = k / TQ, q = k % TQ;
            uint32_t word = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int c = 4 * q + b;
                const int v = (a < 24 && c < 24) ? c_blosum62[a][c] - P.sc.gap_open : -128;
                word |= (uint32_t)(v & 0xff) << (8 * b);
            }
            s_t4[k] = word;
        }
    }
    __syncthreads();
    auto sigma = [&](int a, int b) -> int {
        return P.sc.alphabet == SW_ALPHABET_DNA ? (a == b ? P.sc.match : P.sc.mismatch) : (int)s_sigma[a * 24 + b];
    };

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int seg = lane / W;
    const int L = lane % W;
    const int nc = P.sc.nc;
    uint8_t* prof = smem + (size_t)warp * G::warp_smem(nc);
    volatile int* stop = reinterpret_cast<volatile int*>(prof + G::prof_bytes(nc));
    const uint32_t sv_base = (uint32_t)__cvta_generic_to_shared(prof + G::prof_bytes(nc) + G::STOP_BYTES) +
                             (uint32_t)(lane * 16);
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    const int n_path = P.counts[P.route];
    int first = P.pre ? P.pre[0] + P.pre[1] : 0;
    for (int r = 0; r < P.route; ++r) first += P.counts[r];
    const int items = (n_path + SLOTS - 1) / SLOTS;
    const uint32_t o2 = T::lift(P.sc.gap_open);  // H = Hb + o as one 32-bit add
    const uint32_t e2 = T::splat(P.sc.gap_extend);
    const int o = P.sc.gap_open;

    // One work item (SLOTS pairs) swept by `npart` warps of the CTA: warp `part` takes stripes part,
    // part + npart, ... (npart = 1: this warp alone).  stop_i: the item's per-slot stop columns.
    auto run_item = [&](const int item, const int part, const int npart, volatile int* stop_i) {
#if SW_TRACE_ITEMS
        const unsigned long long tr_t0 = gtimer();
#endif
        // ---- slot descriptors (lane s < SLOTS holds slot s) ----
        int s_pid = -1, s_n = 0, s_m = 0, s_tgt = 0;
        int64_t s_rpos = 0, s_qpos = 0;
        if (lane < SLOTS) {
            const int idx = item * SLOTS + lane;
            if (idx < n_path) {
                s_pid = P.order[first + idx];
                s_n = P.nlen[s_pid];
                s_m = P.mlen[s_pid];
                s_rpos = P.rpos[s_pid];
                s_qpos = P.qpos[s_pid];
                if (REV) s_tgt = P.target[s_pid];
            }
        }
        int mmax = s_m, nmax = s_n, mmin = s_pid >= 0 ? s_m : 0x7fffffff;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            mmax = max(mmax, __shfl_xor_sync(FULL, mmax, d));
            nmax = max(nmax, __shfl_xor_sync(FULL, nmax, d));
            mmin = min(mmin, __shfl_xor_sync(FULL, mmin, d));
        }
        // per-half end events are needed only when a shorter reference of the item runs
        // out of pad codes before the sweep ends (see sweep<>, EV)
        const bool need_ev = !REV && (mmax - mmin > PADR - W - 4 * SW_BODY_BLOCKS - 4);
        const int ns = (nmax + G::ROWS - 1) / G::ROWS;

        // this lane's halves
        int h_pid[NH], h_m[NH], h_tgt[NH];
        int64_t h_rpos[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            const int sl = seg * NH + h;
            h_pid[h] = __shfl_sync(FULL, s_pid, sl);
            h_m[h] = __shfl_sync(FULL, s_m, sl);
            h_tgt[h] = __shfl_sync(FULL, s_tgt, sl);
            h_rpos[h] = __shfl_sync(FULL, s_rpos, sl);
            if (h_pid[h] < 0) h_rpos[h] = PADL;  // empty slot: read pad region at buffer start
        }
        unsigned long long steps = 0;  // column steps over the item's stripes

        if (REV && npart == 1) {
            __syncwarp();
            if (lane < SLOTS) stop_i[lane] = 0x7fffffff;
        }
        // stripe hand-off rows: W slots of slack before column 0, scr_cols columns after it
        const int scr_cols = (int)(P.scratch_seg_bytes / (int64_t)sizeof(uint2)) - W;
        for (int s = part; s < ns; s += npart) {
            const int row0 = s * G::ROWS;
            // Reverse pass, stripes below the first: the exact band of the reversed rectangle.  A
            // reversed alignment ending in cell (i', j') scores <= max_s * min(i' + 1, j' + 1), and
            // from there to the start cell it can gain <= max_s * min(n2 - 1 - i', m2 - 1 - j'); every
            // cell of a score-S path from the origin (and every cell holding S) therefore has
            //   min(i' + 1, j' + 1) + min(n2 - 1 - i', m2 - 1 - j') >= B = ceil(S / max_s),
            // which in rows [row0, r1] bounds the columns to [B - n2 + row0, m2 + r1 - B].  Cells
            // outside are not swept: the stripe starts at the smallest such column of the item's
            // halves with the border (H = 0) on its left, and each half's sweep ends at its largest.
            // The swept cells then hold lower bounds of H' that are exact on every such path, so the
            // cells with H' = S -- and their lexmin -- are unchanged (reading R6).
            // A long, high-identity alignment (S close to max_s * n2, C5) sweeps a diagonal band of
            // ~(n2 - B) columns per side instead of the whole rectangle.
            int c_lo = 0, s_lim = s_m + W - 1;
            // columns the next stripe can read from this stripe's hand-off row (absolute, exclusive)
            int next_lim = mmax + W - 1;
            if (REV) {
                int lo = 0x7fffffff, nl = 0;
                if (lane < SLOTS && s_pid >= 0) {
                    const int ms = P.sc.max_sigma;
                    const int B = (s_tgt + ms - 1) / ms;
                    // gap-aware diagonal band (sw_common.cuh rev_band): rows [row0, r1] of a stripe
                    // need columns [row0 - DI, r1 + DD] only
                    int DI, DD;
                    rev_band(ms, -P.sc.gap_open, -P.sc.gap_extend, s_tgt, s_n, s_m, DI, DD);
                    if (row0 >= s_n) {
                        s_lim = 0;  // no row of this half in the stripe
                    } else {
                        const int r1 = min(row0 + G::ROWS, s_n) - 1;
                        lo = max(max(0, B - s_n + row0), row0 - DI);
                        s_lim = min(min(s_m, s_m + r1 - B + 1), (int)min((int64_t)0x3fffffff, (int64_t)r1 + DD + 1)) + W - 1;
                    }
                    if (row0 + G::ROWS < s_n) {
                        const int r1n = min(row0 + 2 * G::ROWS, s_n) - 1;
                        nl = min(min(s_m, s_m + r1n + 1 - B), (int)min((int64_t)0x3fffffff, (int64_t)r1n + DD + 1)) + W - 1;
                    }
                }
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) {
                    lo = min(lo, __shfl_xor_sync(FULL, lo, d));
                    nl = max(nl, __shfl_xor_sync(FULL, nl, d));
                }
                c_lo = lo == 0x7fffffff ? 0 : lo;
                next_lim = nl;
            }
            // ---- build the stripe's query profile: (s - o) per (slot, code, lane, row) ----
            __syncwarp();
            {
                constexpr int COMBOS = SLOTS * W * G::PWORDS;
                for (int cb = lane; cb < ((COMBOS + 31) / 32) * 32; cb += 32) {
                    const int sl = (cb / (W * G::PWORDS)) % SLOTS;
                    const int pid = __shfl_sync(FULL, s_pid, sl);
                    const int n = __shfl_sync(FULL, s_n, sl);
                    const int64_t qp = __shfl_sync(FULL, s_qpos, sl);
                    if (cb >= COMBOS) continue;
                    const int l = (cb / G::PWORDS) % W;
                    const int w = cb % G::PWORDS;
                    uint8_t* base = prof + (size_t)sl * nc * W * G::PB + (size_t)l * G::PB + w * 4;
                    if (IMK) {
                        // one word per row: (s - o) in the slot's half (low half: zero-extended; high half:
                        // low 16 bits zero), -128 for rows without a residue and for the pad code
                        const int i = row0 + l * K + w;
                        const int qc = (pid >= 0 && i < n) ? P.qcode[REV ? qp + n - 1 - i : qp + i] : -1;
                        const int sh = 16 * (sl % NH);
                        for (int c = 0; c < nc; ++c) {
                            const int v = (qc >= 0 && c < nc - 1) ? (qc == c ? P.sc.match : P.sc.mismatch) - o : -128;
                            *reinterpret_cast<uint32_t*>(base + (size_t)c * W * G::PB) = ((uint32_t)v & 0xffffu) << sh;
                        }
                    } else if (NH == 2 && P.sc.alphabet == SW_ALPHABET_DNA) {
                        // DNA: s(q, c) is match / mismatch, four rows per word with byte-SIMD
                        uint32_t q4 = 0u, inv = 0u;  // query codes; 0xff bytes for rows without a residue
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int r = w * 4 + b;
                            const int i = row0 + l * K + r;
                            if (pid >= 0 && r < K && i < n) q4 |= (uint32_t)P.qcode[REV ? qp + n - 1 - i : qp + i] << (8 * b);
                            else inv |= 0xffu << (8 * b);
                        }
                        const uint32_t mi = (uint32_t)((P.sc.mismatch - o) & 0xff) * 0x01010101u;
                        const uint32_t dm = ((uint32_t)((P.sc.match - o) & 0xff) * 0x01010101u) ^ mi;
                        const uint32_t padw = 0x80808080u;  // -128 per byte
                        for (int c = 0; c < nc - 1; ++c) {
                            const uint32_t x = q4 ^ ((uint32_t)c * 0x01010101u);
                            // 0x80 in every byte of x that is zero (exact: no carries across bytes)
                            const uint32_t z = ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
                            const uint32_t eq = (z >> 7) * 0xffu;
                            const uint32_t word = (((eq & dm) ^ mi) & ~inv) | (inv & padw);
                            *reinterpret_cast<uint32_t*>(base + (size_t)c * W * G::PB) = word;
                        }
                        *reinterpret_cast<uint32_t*>(base + (size_t)(nc - 1) * W * G::PB) = padw;
                    } else if (NH == 2 && SW_PROT_T4 && (SW_T4_ALL || K == SW_KP)) {
                        // protein: four rows' residues index the transposed table; a 4x4 byte
                        // transpose (8 PRMT) turns four table words into the words of four codes
                        uint32_t qa[4];
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int r = w * 4 + b;
                            const int i = row0 + l * K + r;
                            qa[b] = (pid >= 0 && r < K && i < n) ? (uint32_t)P.qcode[REV ? qp + n - 1 - i : qp + i] * TQ
                                                                 : 24u * TQ;
                        }
#pragma unroll
                        for (int q = 0; q < TQ; ++q) {
                            const uint32_t w0 = s_t4[qa[0] + q], w1 = s_t4[qa[1] + q];
                            const uint32_t w2 = s_t4[qa[2] + q], w3 = s_t4[qa[3] + q];
                            const uint32_t t0 = prmt(w0, w1, 0x5140u), t1 = prmt(w0, w1, 0x7362u);
                            const uint32_t t2 = prmt(w2, w3, 0x5140u), t3 = prmt(w2, w3, 0x7362u);
                            const uint32_t ow[4] = {prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u),
                                                    prmt(t1, t3, 0x5410u), prmt(t1, t3, 0x7632u)};
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                if (4 * q + k < NC_PROTEIN)
                                    *reinterpret_cast<uint32_t*>(base + (size_t)(4 * q + k) * W * G::PB) = ow[k];
                        }
                    } else if (NH == 2) {
                        int qc[4];
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int r = w * 4 + b;
                            const int i = row0 + l * K + r;
                            qc[b] = (pid >= 0 && r < K && i < n) ? P.qcode[REV ? qp + n - 1 - i : qp + i] : -1;
                        }
                        for (int c = 0; c < nc; ++c) {
                            uint32_t word = 0;
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                int v = -128;
                                if (qc[b] >= 0 && c < nc - 1) v = sigma(qc[b], c) - o;
                                word |= (uint32_t)(v & 0xff) << (8 * b);
                            }
                            *reinterpret_cast<uint32_t*>(base + (size_t)c * W * G::PB) = word;
                        }
                    } else {
                        const int r = w;
                        const int i = row0 + l * K + r;
                        const int qc = (pid >= 0 && r < K && i < n) ? P.qcode[REV ? qp + n - 1 - i : qp + i] : -1;
                        for (int c = 0; c < nc; ++c) {
                            int v = -(1 << 29);
                            if (qc >= 0 && c < nc - 1) v = sigma(qc, c) - o;
                            *reinterpret_cast<int32_t*>(base + (size_t)c * W * G::PB) = v;
                        }
                    }
                }
            }
            __syncwarp();

            // ---- the stripe's column sweep (single-stripe items skip all hand-off code) ----
            bool swept = false;
            if constexpr (SW_SKEW2 && TAGF && !REV && K == 10 && NH == 2 && G::PWORDS == 4) {
                if (!need_ev && ns == 1) {
                    steps += sweep_skew2<T, W, K>(P, prof, seg, L, h_pid, h_rpos, mmax, row0, o2, e2, o);
                    swept = true;
                }
            }
            if (swept) {
            } else if (SW_SINGLE_ONLY || ns == 1) {
                if (need_ev)
                    steps += sweep<T, W, K, REV, false, true, TAGF, LIN>(P, prof, stop_i, sv_base, seg, L, s_lim, h_pid, h_m, h_tgt, h_rpos, mmax,
                                                     row0, o2, e2, o, nullptr, nullptr, false, false, 0, 0);
                else
                    steps += sweep<T, W, K, REV, false, false, TAGF, LIN>(P, prof, stop_i, sv_base, seg, L, s_lim, h_pid, h_m, h_tgt, h_rpos, mmax,
                                                      row0, o2, e2, o, nullptr, nullptr, false, false, 0, 0);
            } else {
                // rows in absolute columns (W slots of slack before column 0), seen from column c_lo.
                // Stripe s writes the row of warp (s mod npart) of the CTA (this warp), parity
                // (s / npart) & 1, and reads its predecessor's; cooperative items (npart > 1) order
                // the two with a progress word per row (the producer is another warp)
                const int wbase = gwarp - warp;  // the CTA's first warp
                const int pw = (s + npart - 1) % npart, pp = ((s - 1) / npart) & 1;  // s >= 1 only
                const int ow = s % npart, op = (s / npart) & 1;
                const uint2* scr_in = reinterpret_cast<const uint2*>(
                    P.scratch + ((size_t)(npart > 1 ? wbase + pw : gwarp) * G::SEGS * 2 + seg * 2 + (npart > 1 ? pp : ((s + 1) & 1))) *
                                    P.scratch_seg_bytes) + W + c_lo;
                uint2* scr_out = reinterpret_cast<uint2*>(
                    P.scratch + ((size_t)(npart > 1 ? wbase + ow : gwarp) * G::SEGS * 2 + seg * 2 + (npart > 1 ? op : (s & 1))) *
                                    P.scratch_seg_bytes) + W + c_lo;
                const volatile unsigned long long* f_in =
                    (npart > 1 && s > 0) ? P.progress + (size_t)(wbase + pw) * 2 + pp : nullptr;
                volatile unsigned long long* f_out = (npart > 1 && s + 1 < ns) ? P.progress + (size_t)(wbase + ow) * 2 + op : nullptr;
                // progress words: (route, item + 1, stripe, columns): monotonic over the launches of a
                // call (routes in order) and the items a CTA takes; zeroed per call
                const unsigned long long tag_item = ((unsigned long long)P.route << 61) | ((unsigned long long)(item + 1) << 32);
                const unsigned long long nb_in = tag_item | ((unsigned long long)(s - 1) << 21);
                const unsigned long long nb_out = tag_item | ((unsigned long long)s << 21);
                if (need_ev)
                    steps += sweep<T, W, K, REV, true, true, TAGF, LIN>(P, prof, stop_i, sv_base, seg, L, s_lim, h_pid, h_m, h_tgt, h_rpos, mmax,
                                                    row0, o2, e2, o, scr_in, scr_out, s > 0, s + 1 < ns,
                                                    min(scr_cols, next_lim + 4 * U_MAX_FILL) - c_lo, c_lo, f_in, nb_in, f_out, nb_out);
                else
                    steps += sweep<T, W, K, REV, true, false, TAGF, LIN>(P, prof, stop_i, sv_base, seg, L, s_lim, h_pid, h_m, h_tgt, h_rpos, mmax,
                                                     row0, o2, e2, o, scr_in, scr_out, s > 0, s + 1 < ns,
                                                    min(scr_cols, next_lim + 4 * U_MAX_FILL) - c_lo, c_lo, f_in, nb_in, f_out, nb_out);
            }
        }
        if (lane == 0) atomicAdd(P.swept, steps * G::ROWS * SLOTS);
#if SW_TRACE_ITEMS
        if (lane == 0 && part == 0) {
            const unsigned k = atomicAdd(&g_trace_n, 1u);
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            if (k < (unsigned)TRACE_CAP) {
                g_trace[k][0] = ((unsigned long long)item << 32) | ((unsigned long long)smid << 16) | ((REV ? 1u : 0u) << 8) | (unsigned)P.route;
                g_trace[k][1] = tr_t0;
                g_trace[k][2] = gtimer();
                g_trace[k][3] = ((unsigned long long)ns << 48) | ((unsigned long long)(unsigned)mmax << 24) | (steps & 0xffffffull);
            }
        }
#endif
    };

    // stripes of an item (warp-uniform): the longest query of its slots
    auto item_stripes = [&](const int item) -> int {
        int n = 0;
        if (lane < SLOTS) {
            const int idx = item * SLOTS + lane;
            if (idx < n_path) n = P.nlen[P.order[first + idx]];
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) n = max(n, __shfl_xor_sync(FULL, n, d));
        return (n + G::ROWS - 1) / G::ROWS;
    };

    if constexpr (REV) {
        // Reverse pass: the longest items come first in the queue.  While they have at least
        // SW_COOP_STRIPES stripes, a CTA takes one item at a time and all its warps sweep it together,
        // consecutive stripes on consecutive warps, each stripe lagging its predecessor by a publish
        // interval -- one item no longer runs for the length of the whole pass on one warp (the
        // tail of long unrelated pairs, whose start lies far from the origin).
        // The first shorter item ends the phase: warp 0 sweeps it and every warp continues alone.
        __shared__ int s_item;
        const int nwarps = blockDim.x >> 5;
        if (nwarps > 1) {
            volatile int* stop0 = reinterpret_cast<volatile int*>(smem + G::prof_bytes(nc));  // warp 0's
            for (;;) {
                __syncthreads();
                if (threadIdx.x == 0) s_item = atomicAdd(P.item_counter, 1);
                if (warp == 0 && lane < SLOTS) stop0[lane] = 0x7fffffff;
                __syncthreads();
                const int item = s_item;
                if (item >= items) return;
                if (item_stripes(item) < SW_COOP_STRIPES) {
                    if (warp == 0) run_item(item, 0, 1, stop);
                    break;
                }
                run_item(item, warp, nwarps, stop0);
            }
        }
    }
    for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(P.item_counter, 1);
        item = __shfl_sync(FULL, item, 0);
        if (item >= items) break;
        run_item(item, 0, 1, stop);
    }
}

}  // namespace swb
