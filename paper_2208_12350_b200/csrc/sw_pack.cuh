// sw_pack.cuh -- step a1 of SURVEY.md sec. 8(a): validation, ASCII -> codes,
// per-pair lengths/flags/work keys and batch statistics, in one pass.
#pragma once
#include <cstddef>
#include "sw_common.cuh"
#include "sw_bin.cuh"

namespace swb {

// Batch statistics written by the pack / finish kernels (device), read back
// by the host once per batch to size grids and the stripe scratch.
struct BatchStats {
    // cumulative over a user call (sw_align_batch_host may run several chunks)
    int32_t n_bad;          // invalid pairs
    int32_t internal_err;   // self-check failures (reverse max != forward S)
    unsigned long long cells;        // sum n*m over valid pairs
    unsigned long long swept_fwd;    // cells swept by the forward wavefront (incl. padding)
    unsigned long long swept_rev;    // cells swept by the reverse wavefront
    // per batch (chunk)
    int32_t max_n;          // longest valid query
    int32_t max_m;          // longest valid reference
    int32_t malformed;      // offsets decrease somewhere -> whole batch invalid
    int32_t overflow;       // speculative extents: the payload did not fit the code buffers (nothing packed)
    int32_t rejected;       // reserved (asynchronous) call: the batch exceeds the reservation (sw_reserve)
    int32_t fwd_count[4];   // valid, non-trivial pairs per route (forward pass)
    int32_t rev_count[4];   // pairs with S > 0 per route (reverse pass)
    int32_t rev_band[2];    // of which on the banded reverse routes (32 / 64 diagonals, sw_band.cuh)
};
constexpr size_t STATS_PER_BATCH_OFFSET = offsetof(BatchStats, max_n);

// Whole-batch failure flags set by pack (malformed offsets, speculative extents that did not fit,
// a reserved call's batch beyond its reservation): every later kernel of the call checks them at
// entry and does nothing (finish_fwd then writes -1 to every output), so a call enqueued without a
// host round trip never reads per-pair state pack did not write.
static_assert(offsetof(BatchStats, overflow) == offsetof(BatchStats, malformed) + 4 &&
              offsetof(BatchStats, rejected) == offsetof(BatchStats, malformed) + 8,
              "bin_scatter_kernel reads the three flags from &malformed");
__device__ __forceinline__ bool batch_rejected(const BatchStats* st) {
    const volatile BatchStats* v = st;
    return (v->malformed | v->overflow | v->rejected) != 0;
}

struct PackParams {
    const uint8_t* queries;
    const int64_t* q_off;
    const uint8_t* refs;
    const int64_t* r_off;
    int64_t lo, hi;              // pairs to pack (positions in the code buffers are batch-global)
    int64_t q0, qN, r0, rN;      // payload extents of the whole batch (host-read, unless ext_dev)
    int64_t qshift, rshift;      // (payload + extent start) mod 16: code buffers keep the payload's alignment
    int ext_dev;                 // read the extents from q_off / r_off here (no host round trip) and check
    int64_t n_all;               //   they fit qcap / rcap (else stats->overflow, nothing written)
    int64_t qcap, rcap;
    int32_t cap_n, cap_m;        // reserved call (sw_reserve): longest query / reference it covers (0: none)
    int alphabet;
    int s16_ok;                  // scoring fits the s16x2 path (int8 profile, int16 range)
    int tag_ok;                  // the ROUTE_TAG kernel geometry supports row tags
    int max_sigma;
    int rows_s16, rows_s32;      // rows per stripe of each path
    uint8_t* qcode;              // [qN - q0]
    uint8_t* rcode;              // padded layout
    int32_t* nlen;
    int32_t* mlen;
    int64_t* qpos;
    int64_t* rpos;
    uint8_t* flags;
    uint32_t* key;               // work key per pair (sw_bin.cuh; 0: no forward work)
    int32_t* iota;               // 0..n-1 (values of the radix-sort path)
    uint32_t* hist;              // bin histogram (zero on entry)
    unsigned long long* keys_fwd;  // forward argmax keys: zeroed here
    BatchStats* stats;
};

// ASCII -> code table, case-insensitive; CODE_BAD outside the alphabet (reading R10).
__device__ __forceinline__ uint8_t ascii_code(int alphabet, int ch) {
    if (ch >= 'a' && ch <= 'z') ch -= 32;
    if (alphabet == SW_ALPHABET_DNA) {
        // A0 C1 T2 G3: bits 2:1 of the letter (dna4 below computes the same codes four at a time)
        switch (ch) {
            case 'A': return 0;
            case 'C': return 1;
            case 'T': return 2;
            case 'G': return 3;
            default: return CODE_BAD;
        }
    }
    // A R N D C Q E G H I L K M F P S T W Y V B Z X *
    switch (ch) {
        case 'A': return 0;  case 'R': return 1;  case 'N': return 2;  case 'D': return 3;
        case 'C': return 4;  case 'Q': return 5;  case 'E': return 6;  case 'G': return 7;
        case 'H': return 8;  case 'I': return 9;  case 'L': return 10; case 'K': return 11;
        case 'M': return 12; case 'F': return 13; case 'P': return 14; case 'S': return 15;
        case 'T': return 16; case 'W': return 17; case 'Y': return 18; case 'V': return 19;
        case 'B': return 20; case 'Z': return 21; case 'X': return 22; case '*': return 23;
        default: return CODE_BAD;
    }
}

__device__ __forceinline__ uint32_t conv4(uint32_t w, const uint8_t* lut, uint32_t& badmask) {
    const uint32_t c0 = lut[w & 0xff], c1 = lut[(w >> 8) & 0xff], c2 = lut[(w >> 16) & 0xff], c3 = lut[w >> 24];
    badmask |= c0 | c1 | c2 | c3;  // CODE_BAD has bit 7 set, valid codes do not
    return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}

// DNA, four ASCII bytes at a time: code = bits 2:1 of the upper-cased letter (A0 C1 T2 G3);
// a byte is valid iff the letter of its code equals it (one PRMT table lookup).  *nz gets
// 0x80 in every invalid byte.
__device__ __forceinline__ uint32_t dna4(uint32_t w, uint32_t& nz) {
    const uint32_t u = w & 0xdfdfdfdfu;
    const uint32_t c = (u >> 1) & 0x03030303u;
    const uint32_t t = c | (c >> 4);                      // bytes 0 / 2: two codes as nibbles
    const uint32_t sel = __byte_perm(t, 0u, 0x4420u);     // four 2-bit selectors
    const uint32_t diff = __byte_perm(0x47544341u, 0u, sel) ^ u;  // 'A' 'C' 'T' 'G'
    nz = (((diff & 0x7f7f7f7fu) + 0x7f7f7f7fu) | diff) & 0x80808080u;
    return c;
}

// DNA, four ASCII bytes at a time, without the invalid-byte markers: the codes and a word that is
// zero iff all four bytes are valid letters (dna4's diff).
__device__ __forceinline__ uint32_t dna4d(uint32_t w, uint32_t& diff) {
    const uint32_t u = w & 0xdfdfdfdfu;
    const uint32_t c = (u >> 1) & 0x03030303u;
    const uint32_t t = c | (c >> 4);
    const uint32_t sel = __byte_perm(t, 0u, 0x4420u);
    diff = __byte_perm(0x47544341u, 0u, sel) ^ u;
    return c;
}
__device__ __forceinline__ uint32_t nz_of_diff(uint32_t diff) {
    return (((diff & 0x7f7f7f7fu) + 0x7f7f7f7fu) | diff) & 0x80808080u;
}

// Codes of 16 ASCII bytes (DNA: arithmetic, protein: table) and their invalid-byte
// markers (0x80 per invalid byte).  Returns true when every byte is valid (the markers are then 0).
__device__ __forceinline__ bool conv16v(const uint4 v, bool dna, const uint8_t* lut, uint32_t (&c)[4], uint32_t (&nz)[4]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if (dna) {
        uint32_t d[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = dna4d(w[q], d[q]);
        if ((d[0] | d[1] | d[2] | d[3]) == 0u) {
#pragma unroll
            for (int q = 0; q < 4; ++q) nz[q] = 0u;
            return true;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) nz[q] = nz_of_diff(d[q]);
        return false;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t bm = 0;
        c[q] = conv4(w[q], lut, bm);
        nz[q] = c[q] & 0x80808080u;
    }
    return (nz[0] | nz[1] | nz[2] | nz[3]) == 0u;
}

__device__ __forceinline__ void conv16m(const uint4 v, bool dna, const uint8_t* lut, uint32_t (&c)[4], uint32_t (&nz)[4]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (dna) {
            c[q] = dna4(w[q], nz[q]);
        } else {
            uint32_t bm = 0;
            c[q] = conv4(w[q], lut, bm);
            nz[q] = c[q] & 0x80808080u;  // CODE_BAD = 0xff, valid codes < 25
        }
    }
}

// Byte mask of word q from a 16-bit per-byte mask.
__device__ __forceinline__ uint32_t expand_nibble(uint32_t m16, int q) {
    const uint32_t nib = (m16 >> (4 * q)) & 0xfu;
    return ((nib * 0x00204081u) & 0x01010101u) * 0xffu;
}

// Byte-wise conversion of one code position (partial vectors at span edges).
__device__ __forceinline__ uint8_t conv1(uint8_t ch, const uint8_t* lut, uint8_t bad_to, bool& bad) {
    const uint8_t c = lut[ch];
    if (c == CODE_BAD) { bad = true; return bad_to; }
    return c;
}

// Largest k in [0, cnt) with a[k] <= x (a non-decreasing; k = 0 if none).
__device__ __forceinline__ int owner_of32(const int32_t* a, int cnt, int x) {
    int lo = 0, hi = cnt - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ int owner_of(const int64_t* a, int cnt, int64_t x) {
    int lo = 0, hi = cnt - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void store16_within(uint8_t* dst, int64_t y0, uint4 v, int64_t lo, int64_t hi) {
    if (y0 >= lo && y0 + 16 <= hi) {
        *reinterpret_cast<uint4*>(dst + y0) = v;
    } else {  // span edge: only this warp's bytes (the neighbour warp writes the others)
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (y0 + b >= lo && y0 + b < hi) dst[y0 + b] = (uint8_t)(w[b >> 2] >> (8 * (b & 3)));
    }
}

#ifndef SW_PACK_PPW
#define SW_PACK_PPW 16
#endif
#ifndef SW_PACK_FB
#define SW_PACK_FB 2
#endif
#ifndef SW_PACK_MINB
#define SW_PACK_MINB 4
#endif
constexpr int PACK_WARPS = 8;  // warps per pack block (256 threads)
constexpr int PACK_PPW = SW_PACK_PPW;    // pairs per warp
constexpr int PACK_FB = SW_PACK_FB;      // 16-byte vectors per lane in flight

// One warp packs PACK_PPW consecutive pairs: lanes read the pairs' offsets,
// then the warp converts the pairs' reference and query payloads as flat
// lists of aligned 16-byte output vectors (the code buffers keep the payloads'
// 16-byte phase), PACK_FB vectors per lane loaded before any is stored.  The
// reference layout gives every pair the slot [rp - PADL, rp + m + PADR): pad
// codes around the converted reference; references are >= PADL + PADR apart,
// so a vector holds bytes of at most one reference plus pads (one load and a
// byte mask).  Vectors shared with the neighbouring warp's span are written
// byte-wise (only this warp's bytes).
__global__ void __launch_bounds__(256, SW_PACK_MINB) pack_kernel(PackParams P) {
    constexpr int PPW = PACK_PPW;
    __shared__ int s_bad, s_route[N_ROUTES], s_maxn, s_maxm, s_malformed, s_reject;
    __shared__ unsigned long long s_cells;
    __shared__ uint8_t lut[256];
    __shared__ int64_t s_slot[PACK_WARPS][PPW];   // rcode slot start rp - PADL
    __shared__ int64_t s_rdelta[PACK_WARPS][PPW]; // ra - rp: payload index of code position y is y + delta
    __shared__ int32_t s_m[PACK_WARPS][PPW];
    __shared__ int64_t s_qa[PACK_WARPS][PPW];     // query payload starts
    __shared__ uint32_t s_badbits[PACK_WARPS];
    __shared__ int32_t s_slot32[PACK_WARPS][PPW];        // slot start rp - PADL, relative to the warp's span base
    __shared__ int32_t s_ylo[PACK_WARPS][PPW], s_yhi[PACK_WARPS][PPW];  // relative vector starts whose 16 source
                                                                        // bytes lie inside the caller's payload
    __shared__ const uint8_t* s_srcb[PACK_WARPS][PPW];   // payload address of relative code position 0
    if (threadIdx.x == 0) {
        s_bad = s_maxn = s_maxm = s_malformed = s_reject = 0;
        for (int r = 0; r < N_ROUTES; ++r) s_route[r] = 0;
        s_cells = 0;
    }
    for (int c = threadIdx.x; c < 256; c += blockDim.x) lut[c] = ascii_code(P.alphabet, c);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t q0 = P.q0, qN = P.qN, r0 = P.r0, rN = P.rN, qshift = P.qshift, rshift = P.rshift;
    if (P.ext_dev) {
        // extents of the whole batch, read by every thread (one L2 line each): the host skips the
        // synchronous read-back and sized the code buffers from their current capacity
        q0 = P.q_off[0]; qN = P.q_off[P.n_all]; r0 = P.r_off[0]; rN = P.r_off[P.n_all];
        qshift = (int64_t)(((uintptr_t)(P.queries + q0)) & 15);
        rshift = (int64_t)(((uintptr_t)(P.refs + r0)) & 15);
        if (qN < q0 || rN < r0) {  // the host reports it after the statistics read-back
            if (blockIdx.x == 0 && threadIdx.x == 0) P.stats->malformed = 1;
            return;
        }
        if ((qN - q0) + 32 > P.qcap || (rN - r0) + P.n_all * (PADL + PADR) + GUARD + 16 > P.rcap) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                if (P.cap_n) P.stats->rejected = 1;  // reserved call: beyond the reservation
                else P.stats->overflow = 1;
            }
            return;  // uniform over the grid: nothing is written, the host grows and re-runs
        }
    }
    const uint8_t pad_code = (uint8_t)((P.alphabet == SW_ALPHABET_DNA ? NC_DNA : NC_PROTEIN) - 1);
    const uint32_t padw = (uint32_t)pad_code * 0x01010101u;
    const bool dna = P.alphabet == SW_ALPHABET_DNA;
    int l_bad = 0, l_route[N_ROUTES] = {0, 0, 0}, l_maxn = 0, l_maxm = 0, l_malf = 0, l_rej = 0;
    unsigned long long l_cells = 0;
    int64_t* slot = s_slot[wib];
    int64_t* rdelta = s_rdelta[wib];
    int32_t* sm = s_m[wib];
    int64_t* sqa = s_qa[wib];
    for (int64_t base = P.lo + gw * PPW; base < P.hi; base += nw * PPW) {
        const int cnt = (int)(P.hi - base < PPW ? P.hi - base : (int64_t)PPW);
        const int64_t p = base + lane;
        const bool act = lane < cnt;
        int64_t qa = 0, qb = 0, ra = 0, rb = 0;
        if (act) { qa = P.q_off[p]; qb = P.q_off[p + 1]; ra = P.r_off[p]; rb = P.r_off[p + 1]; }
        const int64_t n = qb - qa, m = rb - ra;
        const bool malf = act && (n < 0 || m < 0 || qa < q0 || qb > qN || ra < r0 || rb > rN);
        if (malf) l_malf = 1;
        const int64_t qp = (qa - q0) + qshift;
        const int64_t rp = (ra - r0) + (p + 1) * PADL + p * PADR + rshift;
        if (lane == 0) s_badbits[wib] = 0u;
        if (!__any_sync(FULL, malf)) {
            if (act) { slot[lane] = rp - PADL; rdelta[lane] = ra - rp; sm[lane] = (int32_t)m; sqa[lane] = qa; }
            __syncwarp();
            uint32_t badbits = 0;
            // ---- references: output vectors of [lo, hi) in rcode ----
            const int64_t lo = __shfl_sync(FULL, rp, 0) - PADL;
            const int64_t hi = __shfl_sync(FULL, rp + m + PADR, cnt - 1);
            // 32-bit offsets relative to the span's first 16-byte vector (a span is <= 8 references of
            // <= 65,535 codes plus pads)
            const int64_t base = lo & ~(int64_t)15;
            const int nvec = (int)(((hi - 1) >> 4) - (lo >> 4)) + 1;
            const int lo_r = (int)(lo - base), hi_r = (int)(hi - base);
            int32_t* slot32 = s_slot32[wib];
            int32_t* ylo = s_ylo[wib];
            int32_t* yhi = s_yhi[wib];
            const uint8_t** srcb = s_srcb[wib];
            if (act) {
                const int64_t d = (ra - rp) + base;  // payload index of relative position 0
                slot32[lane] = (int32_t)(rp - PADL - base);
                srcb[lane] = P.refs + d;
                const int64_t l0 = r0 - d, l1 = rN - 16 - d;
                ylo[lane] = (int32_t)max((int64_t)INT32_MIN, min((int64_t)INT32_MAX, l0));
                yhi[lane] = (int32_t)max((int64_t)INT32_MIN, min((int64_t)INT32_MAX, l1));
            }
            __syncwarp();
            uint8_t* rdst = P.rcode + base;
            for (int vr = 0; vr < nvec; vr += 32 * PACK_FB) {
                uint4 src[PACK_FB];
                int rs[PACK_FB], re[PACK_FB], kk[PACK_FB];
#pragma unroll
                for (int u = 0; u < PACK_FB; ++u) {
                    const int vi = vr + u * 32 + lane;
                    const int y0 = vi * 16;
                    src[u] = make_uint4(0, 0, 0, 0);
                    rs[u] = 0; re[u] = 0; kk[u] = 0;
                    if (vi >= nvec) continue;
                    const int k = owner_of32(slot32, cnt, y0);
                    const int rk = slot32[k] + PADL, ek = rk + sm[k];
                    const int a = max(y0, rk), b = min(y0 + 16, ek);
                    kk[u] = k;
                    if (a < b) {
                        rs[u] = a - y0; re[u] = b - y0;
                        if (y0 >= ylo[k] && y0 <= yhi[k]) {  // whole block inside the caller's payload
                            src[u] = __ldg(reinterpret_cast<const uint4*>(srcb[k] + y0));
                        } else {
                            uint32_t w[4] = {0, 0, 0, 0};
                            for (int bb = rs[u]; bb < re[u]; ++bb) w[bb >> 2] |= (uint32_t)srcb[k][y0 + bb] << (8 * (bb & 3));
                            src[u] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < PACK_FB; ++u) {
                    const int vi = vr + u * 32 + lane;
                    if (vi >= nvec) continue;
                    const int y0 = vi * 16;
                    uint4 o = make_uint4(padw, padw, padw, padw);
                    if (re[u] > rs[u]) {
                        // reference bytes [rs, re) of the vector converted, the rest (and invalid
                        // symbols) pad codes
                        uint32_t c[4], nz[4];
                        const bool allv = conv16v(src[u], dna, lut, c, nz);
                        if (rs[u] == 0 && re[u] == 16 && allv) {
                            o = make_uint4(c[0], c[1], c[2], c[3]);  // interior vector, all symbols valid
                        } else {
                            const uint32_t r16 = ((1u << re[u]) - 1u) ^ ((1u << rs[u]) - 1u);
                            uint32_t ow[4], badacc = 0;
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint32_t rm = expand_nibble(r16, q);
                                const uint32_t bb = ((nz[q] >> 7) * 0xffu) & rm;
                                badacc |= bb;
                                const uint32_t keep = rm & ~bb;
                                ow[q] = (c[q] & keep) | (padw & ~keep);
                            }
                            if (badacc) badbits |= 1u << kk[u];
                            o = make_uint4(ow[0], ow[1], ow[2], ow[3]);
                        }
                    }
                    if (y0 >= lo_r && y0 + 16 <= hi_r) {
                        *reinterpret_cast<uint4*>(rdst + y0) = o;
                    } else {  // span edge: only this warp's bytes (the neighbour warp writes the others)
                        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                        for (int bb = 0; bb < 16; ++bb)
                            if (y0 + bb >= lo_r && y0 + bb < hi_r) rdst[y0 + bb] = (uint8_t)(w[bb >> 2] >> (8 * (bb & 3)));
                    }
                }
            }
            // ---- queries: output vectors of [qlo, qhi) in qcode (no pads; shift qshift - q0) ----
            const int64_t qlo = __shfl_sync(FULL, qa, 0) - q0 + qshift;
            const int64_t qhi = __shfl_sync(FULL, qb, cnt - 1) - q0 + qshift;
            const int64_t qd = q0 - qshift;  // payload index of code position y is y + qd
            if (qhi > qlo) {
                // 32-bit offsets relative to the span's first 16-byte vector
                const int64_t qbase = qlo & ~(int64_t)15;
                const int qn = (int)(((qhi - 1) >> 4) - (qlo >> 4)) + 1;
                const int qlo_r = (int)(qlo - qbase), qhi_r = (int)(qhi - qbase);
                const uint8_t* qsrc = P.queries + qbase + qd;
                uint8_t* qdst = P.qcode + qbase;
                for (int vr = 0; vr < qn; vr += 32 * PACK_FB) {
                    uint4 src[PACK_FB];
#pragma unroll
                    for (int u = 0; u < PACK_FB; ++u) {
                        const int vi = vr + u * 32 + lane;
                        const int y0 = vi * 16;
                        src[u] = make_uint4(0, 0, 0, 0);
                        if (vi >= qn) continue;
                        if (y0 >= qlo_r && y0 + 16 <= qhi_r) {
                            src[u] = __ldg(reinterpret_cast<const uint4*>(qsrc + y0));
                        } else {  // span edge: only bytes inside [qlo, qhi)
                            uint32_t w[4] = {0, 0, 0, 0};
                            for (int bb = 0; bb < 16; ++bb)
                                if (y0 + bb >= qlo_r && y0 + bb < qhi_r) w[bb >> 2] |= (uint32_t)qsrc[y0 + bb] << (8 * (bb & 3));
                            src[u] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < PACK_FB; ++u) {
                        const int vi = vr + u * 32 + lane;
                        if (vi >= qn) continue;
                        const int y0 = vi * 16;
                        uint32_t cw[4], nz[4];
                        if (!conv16v(src[u], dna, lut, cw, nz)) {
                            const int lo16 = qlo_r - y0 > 0 ? qlo_r - y0 : 0, hi16 = qhi_r - y0 < 16 ? qhi_r - y0 : 16;
                            const uint32_t r16 = ((1u << hi16) - 1u) ^ ((1u << lo16) - 1u);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint32_t bb = ((nz[q] >> 7) * 0xffu) & expand_nibble(r16, q);
                                if (bb) {  // rare: attribute each bad byte to its pair, store pads instead
                                    for (int b = 0; b < 4; ++b)
                                        if ((bb >> (8 * b)) & 0xffu)
                                            badbits |= 1u << owner_of(sqa, cnt, qbase + y0 + qd + 4 * q + b);
                                }
                                cw[q] = (cw[q] & ~bb) | (padw & bb);
                            }
                        }
                        const uint4 o = make_uint4(cw[0], cw[1], cw[2], cw[3]);
                        if (y0 >= qlo_r && y0 + 16 <= qhi_r) {
                            *reinterpret_cast<uint4*>(qdst + y0) = o;
                        } else {  // span edge: only this warp's bytes
                            const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                            for (int bb = 0; bb < 16; ++bb)
                                if (y0 + bb >= qlo_r && y0 + bb < qhi_r) qdst[y0 + bb] = (uint8_t)(w[bb >> 2] >> (8 * (bb & 3)));
                        }
                    }
                }
            }
            if (badbits) atomicOr(&s_badbits[wib], badbits);
            __syncwarp();
        }
        // ---- per-pair metadata (lane = pair) ----
        if (act) {
            const bool bad = malf || n > SW_MAX_SEQ_LEN || m > SW_MAX_SEQ_LEN || ((s_badbits[wib] >> lane) & 1u);
            uint32_t key = 0;
            uint8_t fl = 0;
            int nn = 0, mm = 0;
            if (bad) {
                fl = FLAG_BAD;
                ++l_bad;
            } else {
                nn = (int)n; mm = (int)m;
                // largest score the pair can reach (reading R13): picks the lane width
                const int64_t smax = (int64_t)P.max_sigma * (int64_t)min(nn, mm);
                // TAG: every cell a sweep over this query can compute (also past the reference, in
                // the columns of a longer reference of the work item) has H <= max_s * n <= 511
                const int route = (P.s16_ok && P.tag_ok && (int64_t)P.max_sigma * nn <= tag_max_score(P.alphabet)) ? ROUTE_TAG
                                : (P.s16_ok && smax <= S16_MAX_SCORE) ? ROUTE_S16 : ROUTE_S32;
                fl = route_flag(route);
                if (nn > 0 && mm > 0) {
                    const int rows = route == ROUTE_S32 ? P.rows_s32 : P.rows_s16;
                    key = work_key(route, (uint32_t)((nn + rows - 1) / rows), (uint32_t)mm);
                    const uint32_t bin = key_bin(key);
                    if (bin) atomicAdd(P.hist + bin, 1u);
                    ++l_route[route];
                    l_cells += (unsigned long long)nn * (unsigned long long)mm;
                }
                l_maxn = max(l_maxn, nn);
                l_maxm = max(l_maxm, mm);
                if (P.cap_n && (nn > P.cap_n || mm > P.cap_m)) l_rej = 1;
            }
            P.nlen[p] = nn;
            P.mlen[p] = mm;
            P.qpos[p] = qp;
            P.rpos[p] = rp;
            P.flags[p] = fl;
            P.key[p] = key;
            P.iota[p] = (int32_t)p;
            P.keys_fwd[p] = 0ull;
        }
        __syncwarp();
    }
    // block reduction of the lanes' statistics
    if (l_bad) atomicAdd(&s_bad, l_bad);
    for (int r = 0; r < N_ROUTES; ++r)
        if (l_route[r]) atomicAdd(&s_route[r], l_route[r]);
    if (l_maxn) atomicMax(&s_maxn, l_maxn);
    if (l_maxm) atomicMax(&s_maxm, l_maxm);
    if (l_malf) atomicOr(&s_malformed, 1);
    if (l_rej) atomicOr(&s_reject, 1);
    if (l_cells) atomicAdd(&s_cells, l_cells);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_bad) atomicAdd(&P.stats->n_bad, s_bad);
        for (int r = 0; r < N_ROUTES; ++r)
            if (s_route[r]) atomicAdd(&P.stats->fwd_count[r], s_route[r]);
        if (s_maxn) atomicMax(&P.stats->max_n, s_maxn);
        if (s_maxm) atomicMax(&P.stats->max_m, s_maxm);
        if (s_malformed) atomicOr(&P.stats->malformed, 1);
        if (s_reject) atomicOr(&P.stats->rejected, 1);
        if (s_cells) atomicAdd(&P.stats->cells, s_cells);
    }
}

}  // namespace swb
