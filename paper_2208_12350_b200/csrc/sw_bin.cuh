// sw_bin.cuh -- step a2 of SURVEY.md sec. 8(a): length binning of the work
// items.  The wavefront kernels pull pairs in the order of a per-pass array:
// grouped by kernel route (TAG, S16, S32) and, inside a route, longest work
// first (the load balance of PAPER.md:574-590's length sorting, kept; the sort
// itself need not be exact).  A counting sort on a 14-bit bin replaces a full
// radix sort: the producing kernel (pack / finish_fwd) adds each pair to the
// bin histogram, one block scans the histogram (descending bins), one kernel
// scatters the pair ids.  Order within a bin is arbitrary; results do not
// depend on it (the per-pair argmax keys merge with atomicMax).
#pragma once
#include "sw_common.cuh"

namespace swb {

// Work keys (one 32-bit word per pair, larger = more work, taken first):
//   [31:30] 3 - route (0: no work)   [29:16] stripes   [15:0] columns
// (forward: columns = m; reverse: the score S, the proxy of the early-stopped
// sweep's length).  Batches whose keys all lie in the "small" region -- at
// most BIN_MAX_STRIPES stripes and fewer than BIN_COLS columns, the ADEPT
// regime -- are counting-sorted on an exact bin (below); others take a radix
// sort of the full keys (sw_api.cu).  Exact bins keep a work item's four pairs
// on identical (stripes, columns): no padded rows or columns.
constexpr int BIN_MAX_STRIPES = 8;
constexpr int BIN_COLS = 1040;   // columns 0..1039 (references up to 1,024 plus slack)
constexpr int BIN_PER_ROUTE = BIN_MAX_STRIPES * BIN_COLS;
constexpr int NBINS = N_ROUTES * BIN_PER_ROUTE;     // bin 0 never holds work (columns >= 1)
constexpr int BIN_SCAN_THREADS = 1024;

__host__ __device__ __forceinline__ uint32_t work_key(int route, uint32_t stripes, uint32_t cols) {
    return route_key(route) | ((stripes < 0x3fffu ? stripes : 0x3fffu) << 16) | (cols < 0xffffu ? cols : 0xffffu);
}

// Exact bin of a key in the small region (0 if the key has no work or lies outside).
__host__ __device__ __forceinline__ uint32_t key_bin(uint32_t key) {
    const uint32_t rank = key >> 30, stripes = (key >> 16) & 0x3fffu, cols = key & 0xffffu;
    if (rank == 0 || stripes < 1 || stripes > (uint32_t)BIN_MAX_STRIPES || cols >= (uint32_t)BIN_COLS) return 0;
    return (rank - 1) * BIN_PER_ROUTE + (stripes - 1) * BIN_COLS + cols;
}
constexpr int BIN_SCAN_SMEM = (NBINS + NBINS / 32) * 4;  // the whole histogram in shared memory (padded)
__device__ __forceinline__ int bin_pad(int i) { return i + (i >> 5); }  // no bank conflicts per thread chunk

// hist[NBINS] -> base[NBINS] = number of pairs in higher bins (descending
// order); hist is reset for the next pass.  One block; the histogram is
// staged in shared memory with coalesced loads.
__global__ void __launch_bounds__(BIN_SCAN_THREADS) bin_scan_kernel(uint32_t* hist, uint32_t* base) {
    constexpr int PER = (NBINS + BIN_SCAN_THREADS - 1) / BIN_SCAN_THREADS;
    extern __shared__ uint32_t s_h[];  // [bin_pad(NBINS)]
    __shared__ uint32_t s_warp[BIN_SCAN_THREADS / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int k = t; k < NBINS; k += BIN_SCAN_THREADS) {
        s_h[bin_pad(k)] = hist[k];
        hist[k] = 0u;
    }
    __syncthreads();
    // thread t owns the descending chunk of bins [NBINS - (t+1)*PER, NBINS - t*PER)
    const int hi_bin = NBINS - t * PER;
    uint32_t sum = 0;
#pragma unroll 8
    for (int k = 0; k < PER; ++k)
        if (hi_bin - 1 - k >= 0) sum += s_h[bin_pad(hi_bin - 1 - k)];
    // exclusive scan of the thread sums: warp shuffles, then the warp totals
    uint32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += x;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_warp[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t x = __shfl_up_sync(FULL, w, d);
            if (lane >= d) w += x;
        }
        s_warp[lane] = w;
    }
    __syncthreads();
    uint32_t run = incl - sum + (warp ? s_warp[warp - 1] : 0u);
#pragma unroll 8
    for (int k = 0; k < PER; ++k) {
        if (hi_bin - 1 - k < 0) break;
        const uint32_t v = s_h[bin_pad(hi_bin - 1 - k)];
        s_h[bin_pad(hi_bin - 1 - k)] = run;
        run += v;
    }
    __syncthreads();
    for (int k = t; k < NBINS; k += BIN_SCAN_THREADS) base[k] = s_h[bin_pad(k)];
}

// order[base[bin(key[p])]++] = p for every pair with work (small-region batches only).  `reject`
// (optional) points at BatchStats::malformed, overflow, rejected: a rejected batch scatters nothing.
// Warp-aggregated: lanes holding the same bin (reverse keys cluster on a few scores) take
// their slots with one atomic per distinct bin of the warp.
__global__ void __launch_bounds__(256) bin_scatter_kernel(const uint32_t* key, uint32_t* base, int32_t* order, int64_t lo,
                                                         int64_t hi, const int32_t* reject) {
    if (reject && (((const volatile int32_t*)reject)[0] | ((const volatile int32_t*)reject)[1] |
                   ((const volatile int32_t*)reject)[2])) return;  // batch_rejected (sw_pack.cuh)
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p0 = lo + (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); p0 < hi; p0 += stride) {
        const int64_t p = p0 + lane;
        const uint32_t b = p < hi ? key_bin(key[p]) : 0u;
        const uint32_t peers = __match_any_sync(FULL, b);
        const int leader = __ffs(peers) - 1;
        uint32_t off = 0;
        if (b && lane == leader) off = atomicAdd(base + b, (uint32_t)__popc(peers));
        off = __shfl_sync(FULL, off, leader);
        if (b) order[off + __popc(peers & ((1u << lane) - 1u))] = (int32_t)p;
    }
}

}  // namespace swb
