// sw_finish.cuh -- step a5 of SURVEY.md sec. 8(a) (decode the argmax keys
// into the caller's arrays) plus the reverse-pass preparation, and the DPX
// roofline probe of sec. 8(d).
#pragma once
#include "sw_common.cuh"
#include "sw_pack.cuh"

namespace swb {

struct FinishParams {
    int64_t n_pairs;
    const uint8_t* flags;
    const unsigned long long* keys_fwd;
    const unsigned long long* keys_rev;
    const uint8_t* qcode;
    uint8_t* qrev;
    const uint8_t* rcode;
    uint8_t* rrev;
    const int64_t* qpos;
    const int64_t* rpos;
    int32_t* nlen_rev;
    int32_t* mlen_rev;
    int32_t* target;
    uint32_t* key_rev;
    int32_t* iota;
    int rows_s16, rows_s32;
    int max_sigma, gap_extend;
    sw_result_t out;
    BatchStats* stats;
};

__device__ __forceinline__ void decode_key(unsigned long long key, int& S, int& j, int& i) {
    S = (int)(key >> 32);
    j = 0xffff - (int)((key >> 16) & 0xffff);
    i = 0xffff - (int)(key & 0xffff);
}

// After the forward pass: score / q_end / r_end into the caller's arrays,
// sentinels for invalid and S = 0 pairs, and the reversed prefixes
// reverse(q[0..q_end]) x reverse(r[0..r_end]) materialised for the reverse
// pass (reading R6).  One warp per pair.
__global__ void __launch_bounds__(256) finish_fwd_kernel(FinishParams P) {
    __shared__ int s_route[N_ROUTES];
    if (threadIdx.x < N_ROUTES) s_route[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int l_route[N_ROUTES] = {0, 0, 0};
    for (int64_t p = gw; p < P.n_pairs; p += nw) {
        const uint8_t fl = P.flags[p];
        const unsigned long long key = P.keys_fwd[p];
        int S = 0, j = -1, i = -1;
        if (key) decode_key(key, S, j, i);
        if (fl & FLAG_BAD) {
            if (lane == 0) {
                P.out.score[p] = -1; P.out.q_end[p] = -1; P.out.r_end[p] = -1;
                P.out.q_start[p] = -1; P.out.r_start[p] = -1;
                P.key_rev[p] = 0; P.iota[p] = (int32_t)p;
            }
            continue;
        }
        if (S == 0) {
            if (lane == 0) {
                P.out.score[p] = 0; P.out.q_end[p] = -1; P.out.r_end[p] = -1;
                P.out.q_start[p] = -1; P.out.r_start[p] = -1;
                P.key_rev[p] = 0; P.iota[p] = (int32_t)p;
            }
            continue;
        }
        const int64_t qp = P.qpos[p];
        const int64_t rp = P.rpos[p];
        for (int k = lane; k <= i; k += 32) P.qrev[qp + k] = P.qcode[qp + i - k];
        for (int k = lane; k <= j; k += 32) P.rrev[rp + k] = P.rcode[rp + j - k];
        if (lane == 0) {
            P.out.score[p] = S; P.out.q_end[p] = i; P.out.r_end[p] = j;
            const int n2 = i + 1;
            // Columns the reverse pass can need (reading R6): every score-S alignment in the
            // reversed rectangle starts at its origin (SURVEY.md 8(c) C-5 proof) and spans
            // M + I columns, M <= n2 aligned pairs and I gap columns each costing >= |e|, so
            // S <= max_s*M - |e|*I  =>  columns <= n2 + (max_s*n2 - S) / |e|.  Exact bound.
            int m2 = j + 1;
            if (P.gap_extend < 0) {
                const long long bound = (long long)n2 + ((long long)P.max_sigma * n2 - S) / (long long)(-P.gap_extend);
                if (bound < m2) m2 = (int)max(bound, 1LL);
            }
            const int route = flag_route(fl);
            const int rows = route == ROUTE_S32 ? P.rows_s32 : P.rows_s16;
            const uint32_t stripes = min((n2 + rows - 1) / rows, 0x3fff);
            P.nlen_rev[p] = n2;
            P.mlen_rev[p] = m2;
            P.target[p] = S;
            // reverse work items are grouped by S: the early-stopped sweep's length follows the
            // alignment's span, for which S is the available proxy
            P.key_rev[p] = route_key(route) | (stripes << 16) | (uint32_t)min(S, 0xffff);
            P.iota[p] = (int32_t)p;
            ++l_route[route];
        }
    }
    if (lane == 0)
        for (int r = 0; r < N_ROUTES; ++r)
            if (l_route[r]) atomicAdd(&s_route[r], l_route[r]);
    __syncthreads();
    if (threadIdx.x < N_ROUTES && s_route[threadIdx.x]) atomicAdd(&P.stats->rev_count[threadIdx.x], s_route[threadIdx.x]);
}

// After the reverse pass: q_start = q_end - i', r_start = r_end - j'.
// Self-check (pin P14 on the device): the reverse maximum must equal S.
__global__ void __launch_bounds__(256) finish_rev_kernel(FinishParams P) {
    int err = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P.n_pairs; p += (int64_t)gridDim.x * blockDim.x) {
        if (P.flags[p] & FLAG_BAD) continue;
        const unsigned long long kf = P.keys_fwd[p];
        if (!kf) continue;
        int S, j, i, S2, j2, i2;
        decode_key(kf, S, j, i);
        decode_key(P.keys_rev[p], S2, j2, i2);
        if (S2 != S || i2 > i || j2 > j) {
            ++err;
            P.out.q_start[p] = -2; P.out.r_start[p] = -2;
            continue;
        }
        P.out.q_start[p] = i - i2;
        P.out.r_start[p] = j - j2;
    }
    if (err) atomicAdd(&P.stats->internal_err, err);
}

// Whole-batch invalid (malformed offsets): every field -1.
__global__ void fill_invalid_kernel(sw_result_t out, int64_t n) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        out.score[p] = -1; out.q_end[p] = -1; out.r_end[p] = -1; out.q_start[p] = -1; out.r_start[p] = -1;
    }
}

// ---------------------------------------------------------------------------
// DPX roofline probe: the minimal s16x2
// Gotoh cell-pair mix -- per chain step 1 VIADD.16x2 (H + o), 2 VIADDMNMX
// (E, F), 1 VIMNMX.RELU (max(E, F, 0)), 1 VIADDMNMX (H), 1/2 VIMNMX3 (running
// max) = 5.5 instructions per two cells -- on 8 independent chains per thread.
// ---------------------------------------------------------------------------
constexpr int DPX_CHAINS = 8;

__global__ void __launch_bounds__(256) dpx_peak_kernel(uint32_t* sink, int iters, uint32_t seed, uint32_t o2, uint32_t e2) {
    uint32_t h[DPX_CHAINS], e[DPX_CHAINS], f[DPX_CHAINS], d[DPX_CHAINS];
    uint32_t best = 0;
#pragma unroll
    for (int c = 0; c < DPX_CHAINS; ++c) {
        h[c] = seed * (c + 1) + threadIdx.x; e[c] = h[c] ^ 0x5555u; f[c] = h[c] + 77u; d[c] = h[c] * 3u;
    }
    const uint32_t s = seed ^ 0x00030003u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < DPX_CHAINS; ++c) {
            const uint32_t ho = __vadd2(h[c], o2);
            e[c] = __viaddmax_s16x2(e[c], e2, ho);
            f[c] = __viaddmax_s16x2(f[c], e2, ho);
            const uint32_t t = __vimax_s16x2_relu(e[c], f[c]);
            const uint32_t hn = __viaddmax_s16x2(d[c], s, t);
            d[c] = h[c];
            h[c] = hn;
            if (c & 1) best = __vimax3_s16x2_relu(best, h[c], h[c - 1]);
        }
    }
    uint32_t acc = best;
#pragma unroll
    for (int c = 0; c < DPX_CHAINS; ++c) acc ^= h[c] ^ e[c] ^ f[c] ^ d[c];
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;  // keep the chains live
}

}  // namespace swb
