// sw_pack.cuh -- step a1 of SURVEY.md sec. 8(a): validation, ASCII -> codes,
// per-pair lengths/flags/work keys and batch statistics, in one pass.
#pragma once
#include <cstddef>
#include "sw_common.cuh"

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
    int32_t pad_;
    int32_t fwd_count[4];   // valid, non-trivial pairs per route (forward pass)
    int32_t rev_count[4];   // pairs with S > 0 per route (reverse pass)
};
constexpr size_t STATS_PER_BATCH_OFFSET = offsetof(BatchStats, max_n);

struct PackParams {
    const uint8_t* queries;
    const int64_t* q_off;
    const uint8_t* refs;
    const int64_t* r_off;
    int64_t n_pairs;
    int64_t q0, qN, r0, rN;      // payload extents (host-read)
    int64_t qshift, rshift;      // (payload + extent start) mod 16: code buffers keep the payload's alignment
    int alphabet;
    int s16_ok;                  // scoring fits the s16x2 path (int8 profile, int16 range)
    int tag_ok;                  // the ROUTE_TAG kernel geometry supports row tags
    int max_sigma;
    int rows_s16, rows_s32;      // rows per stripe of each path
    uint8_t* qcode;              // [qN - q0]
    uint8_t* rcode;              // padded layout
    uint8_t* rrev;               // padded layout (pads only here)
    int32_t* nlen;
    int32_t* mlen;
    int64_t* qpos;
    int64_t* rpos;
    uint8_t* flags;
    uint32_t* key;
    int32_t* iota;
    BatchStats* stats;
};

// ASCII -> code table, case-insensitive; CODE_BAD outside the alphabet (reading R10).
__device__ __forceinline__ uint8_t ascii_code(int alphabet, int ch) {
    if (ch >= 'a' && ch <= 'z') ch -= 32;
    if (alphabet == SW_ALPHABET_DNA) {
        switch (ch) {
            case 'A': return 0;
            case 'C': return 1;
            case 'G': return 2;
            case 'T': return 3;
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

// Convert one sequence: src and dst have the same address mod 16 (by construction of
// the code-buffer positions), so the body moves as aligned 16-byte vectors.
// Returns true if a symbol is outside the alphabet; such symbols become `bad_to`.
__device__ __forceinline__ bool convert_run(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t len,
                                            const uint8_t* lut, uint8_t bad_to, int lane) {
    uint32_t badmask = 0;
    bool bad = false;
    const int head = (int)(len < (int64_t)((16 - ((uintptr_t)src & 15)) & 15) ? len : (int64_t)((16 - ((uintptr_t)src & 15)) & 15));
    if (lane < head) {
        const uint8_t c = lut[src[lane]];
        bad |= c == CODE_BAD;
        dst[lane] = c == CODE_BAD ? bad_to : c;
    }
    const int64_t body = (len - head) >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    for (int64_t k = lane; k < body; k += 32) {
        const uint4 v = __ldg(s4 + k);
        uint32_t bm = 0;
        uint4 o;
        o.x = conv4(v.x, lut, bm); o.y = conv4(v.y, lut, bm); o.z = conv4(v.z, lut, bm); o.w = conv4(v.w, lut, bm);
        if (bm & 0x80u) {  // rare: replace bad bytes
            uint32_t* ow = &o.x;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (((ow[q] >> (8 * b)) & 0xff) == CODE_BAD) ow[q] = (ow[q] & ~(0xffu << (8 * b))) | ((uint32_t)bad_to << (8 * b));
        }
        badmask |= bm;
        d4[k] = o;
    }
    const int64_t t0 = head + body * 16;
    if (lane < len - t0) {
        const uint8_t c = lut[src[t0 + lane]];
        bad |= c == CODE_BAD;
        dst[t0 + lane] = c == CODE_BAD ? bad_to : c;
    }
    return bad || (badmask & 0x80u);
}

__global__ void __launch_bounds__(256) pack_kernel(PackParams P) {
    __shared__ int s_bad, s_route[N_ROUTES], s_maxn, s_maxm, s_malformed;
    __shared__ unsigned long long s_cells;
    __shared__ uint8_t lut[256];
    if (threadIdx.x == 0) {
        s_bad = s_maxn = s_maxm = s_malformed = 0;
        for (int r = 0; r < N_ROUTES; ++r) s_route[r] = 0;
        s_cells = 0;
    }
    for (int c = threadIdx.x; c < 256; c += blockDim.x) lut[c] = ascii_code(P.alphabet, c);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint8_t pad_code = (uint8_t)((P.alphabet == SW_ALPHABET_DNA ? NC_DNA : NC_PROTEIN) - 1);
    int l_bad = 0, l_route[N_ROUTES] = {0, 0, 0}, l_maxn = 0, l_maxm = 0, l_malf = 0;
    unsigned long long l_cells = 0;
    for (int64_t p = gw; p < P.n_pairs; p += nw) {
        const int64_t qa = P.q_off[p], qb = P.q_off[p + 1];
        const int64_t ra = P.r_off[p], rb = P.r_off[p + 1];
        const int64_t n = qb - qa, m = rb - ra;
        bool in_range = qa >= P.q0 && qb <= P.qN && ra >= P.r0 && rb <= P.rN && n >= 0 && m >= 0;
        if (n < 0 || m < 0) l_malf = 1;
        bool bad = !in_range || n > SW_MAX_SEQ_LEN || m > SW_MAX_SEQ_LEN;
        const int64_t qp = (qa - P.q0) + P.qshift;
        const int64_t rp = (ra - P.r0) + (p + 1) * PADL + p * PADR + P.rshift;
        if (in_range && !bad) {
            bad |= convert_run(P.queries + qa, P.qcode + qp, n, lut, pad_code, lane);
            bad |= convert_run(P.refs + ra, P.rcode + rp, m, lut, pad_code, lane);
            // pads around the reference, in both the forward and the reverse buffer
            for (int k = lane; k < PADL + PADR; k += 32) {
                const int64_t pos = k < PADL ? rp - PADL + k : rp + m + (k - PADL);
                P.rcode[pos] = pad_code;
                P.rrev[pos] = pad_code;
            }
        }
        bad = __any_sync(FULL, bad);
        if (lane == 0) {
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
                const int route = (P.s16_ok && P.tag_ok && smax <= TAG_MAX_SCORE) ? ROUTE_TAG
                                : (P.s16_ok && smax <= 32000) ? ROUTE_S16 : ROUTE_S32;
                fl = route_flag(route);
                if (nn > 0 && mm > 0) {
                    const int rows = route == ROUTE_S32 ? P.rows_s32 : P.rows_s16;
                    const uint32_t stripes = min((nn + rows - 1) / rows, 0x3fff);
                    key = route_key(route) | (stripes << 16) | (uint32_t)mm;
                    ++l_route[route];
                    l_cells += (unsigned long long)nn * (unsigned long long)mm;
                }
                l_maxn = max(l_maxn, nn);
                l_maxm = max(l_maxm, mm);
            }
            P.nlen[p] = nn;
            P.mlen[p] = mm;
            P.qpos[p] = qp;
            P.rpos[p] = rp;
            P.flags[p] = fl;
            P.key[p] = key;
            P.iota[p] = (int32_t)p;
        }
    }
    if (lane == 0) {
        if (l_bad) atomicAdd(&s_bad, l_bad);
        for (int r = 0; r < N_ROUTES; ++r)
            if (l_route[r]) atomicAdd(&s_route[r], l_route[r]);
        if (l_maxn) atomicMax(&s_maxn, l_maxn);
        if (l_maxm) atomicMax(&s_maxm, l_maxm);
        if (l_malf) atomicOr(&s_malformed, 1);
        if (l_cells) atomicAdd(&s_cells, l_cells);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_bad) atomicAdd(&P.stats->n_bad, s_bad);
        for (int r = 0; r < N_ROUTES; ++r)
            if (s_route[r]) atomicAdd(&P.stats->fwd_count[r], s_route[r]);
        if (s_maxn) atomicMax(&P.stats->max_n, s_maxn);
        if (s_maxm) atomicMax(&P.stats->max_m, s_maxm);
        if (s_malformed) atomicOr(&P.stats->malformed, 1);
        if (s_cells) atomicAdd(&P.stats->cells, s_cells);
    }
}

}  // namespace swb
