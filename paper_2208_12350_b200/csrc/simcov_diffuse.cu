// simcov_diffuse.cu -- SURVEY.md sec. 8(f) row f4: the SIMCoV diffusion stencil on a
// zero-padded grid (PAPER.md:197 task 4; sec. VI-D "padding the grid
// borders with extra points of value 0"), behind the C ABI of include/simcov.h.
//
// Step rule (reading R22): share(v) = floor(v * a / 2^32) = __umulhi(v, a);
//   v'[y][x] = v - 4 share(v) + share(up) + share(down) + share(left) + share(right),
// a neighbour outside the grid being a zero padding point.
//
// The paper's lesson, kept on sm_100a: neighbour reads never branch on the grid
// boundary -- the padded layout (include/simcov.h) puts a zero ring (one row above
// and below, >= 4 words left and right, 16-byte aligned rows) around every field,
// so every read of an edge point's neighbour is an ordinary in-bounds load of 0.
// What is B200-specific is the rest:
// * HBM-bound (8 B of algorithmic traffic per cell and step, one read + one
//   write): 16-byte vector loads and stores, one warp per 128-column strip that
//   marches down R = 4 rows keeping the rows above and below in registers (short
//   chunks: many warps in flight beat the re-read of the chunk's boundary rows,
//   which L2 serves), left/right neighbour shares by __shfl (only the two
//   strip-edge lanes load a scalar from the padding or the next strip);
// * temporal blocking (k <= 8 steps per launch, the default schedule): a CTA of 8 warps
//   loads a 128-word x 160-row tile straight into registers (20 rows per warp), runs k
//   steps there -- only the first/last-row shares of each warp cross through shared
//   memory, one barrier per step -- and writes its core (the tile shrunk by k rows and a
//   4- or 8-word halo), so HBM traffic is 8 B per cell per k steps plus the halo re-reads.
//   Tiles reaching outside the grid force the cells outside it back to 0 after every step
//   -- the same padding points, held at 0 by one AND per cell (a per-thread column mask
//   computed once, a per-row bit); interior tiles skip the mask.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "simcov.h"

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;
int32_t g_schedule = 0;

constexpr int64_t kColPad = 4;   // interior starts at word 4 of a padded row
constexpr int kStripCols = 128;  // one warp: 32 lanes x 4 cells
#ifndef SIMCOV_TB_WARPS
#define SIMCOV_TB_WARPS 8
#endif
#ifndef SIMCOV_TB_RPW
#define SIMCOV_TB_RPW 20
#endif
#ifndef SIMCOV_TB_MINB
#define SIMCOV_TB_MINB 2
#endif
#ifndef SIMCOV_TB_KMAX
#define SIMCOV_TB_KMAX 8
#endif
constexpr int kTbMaxK = SIMCOV_TB_KMAX;  // default steps per launch (halo 4 words for k <= 4, else 8)
constexpr int kTbWarps = SIMCOV_TB_WARPS;
constexpr int kTbRowsPerWarp = SIMCOV_TB_RPW;

struct Rates {
    uint32_t a[SIMCOV_MAX_FIELDS];
};

__device__ __forceinline__ uint4 ldg4(const uint32_t* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ uint4 share4(uint4 v, uint32_t a) {
    return make_uint4(__umulhi(v.x, a), __umulhi(v.y, a), __umulhi(v.z, a), __umulhi(v.w, a));
}

// v - 4 s + up + down + left + right, for the 4 cells of a lane (sl / sr: the shares
// of the cells left of .x and right of .w)
__device__ __forceinline__ uint4 update4(uint4 v, uint4 s, uint4 su, uint4 sd, uint32_t sl, uint32_t sr) {
    uint4 o;
    o.x = v.x - 4u * s.x + su.x + sd.x + sl + s.y;
    o.y = v.y - 4u * s.y + su.y + sd.y + s.x + s.z;
    o.z = v.z - 4u * s.z + su.z + sd.z + s.y + s.w;
    o.w = v.w - 4u * s.w + su.w + sd.w + s.z + sr;
    return o;
}

// Store the first `nvalid` (0..4) cells of a lane's 4: a vector store unless the
// lane straddles the right edge of the grid (the padding words must stay 0).
__device__ __forceinline__ void store4(uint32_t* p, uint4 o, int nvalid) {
    if (nvalid >= 4) {
        *reinterpret_cast<uint4*>(p) = o;
    } else {
        if (nvalid > 0) p[0] = o.x;
        if (nvalid > 1) p[1] = o.y;
        if (nvalid > 2) p[2] = o.z;
    }
}

// ---------------------------------------------------------------------------------------
// One step per launch.  Warp w -> (field, row chunk, strip), strips fastest so that the
// warps of a CTA read adjacent 512-byte row segments.  The warp owns interior rows
// [chunk*R, chunk*R + R) of columns [strip*128, strip*128 + 128).
template <int R>
__global__ void __launch_bounds__(256) diffuse_step_kernel(const uint32_t* __restrict__ src,
                                                           uint32_t* __restrict__ dst, int64_t pitch,
                                                           int64_t fstride, int H, int W, int n_strips,
                                                           int n_chunks, int n_fields, const __grid_constant__ Rates rates) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int strip = (int)(warp % n_strips);
    const int64_t t = warp / n_strips;
    const int chunk = (int)(t % n_chunks);
    const int field = (int)(t / n_chunks);
    if (field >= n_fields) return;  // whole warps only
    const uint32_t a = rates.a[field];
    const int x0 = strip * kStripCols + lane * 4;
    const int nvalid = W - x0;
    const int64_t off = (int64_t)field * fstride + kColPad + x0;
    const uint32_t* s = src + off;
    uint32_t* d = dst + off;
    const int y0 = chunk * R;
    // padded row of interior row y is y + 1; rows 0 and H + 1 are the zero ring
    uint4 vc = ldg4(s + (int64_t)(y0 + 1) * pitch);
    uint4 su = share4(ldg4(s + (int64_t)y0 * pitch), a);
    uint4 sc = share4(vc, a);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        const int64_t prow = min(y + 2, H + 1);
        const uint4 vd = ldg4(s + prow * pitch);
        uint32_t el = 0, er = 0;
        const uint32_t* rowc = s + (int64_t)(y + 1) * pitch;
        if (lane == 0) el = __ldg(rowc - 1);  // padding (strip 0) or the previous strip
        if (lane == 31) er = __ldg(rowc + 4); // padding or the next strip
        const uint4 sd = share4(vd, a);
        uint32_t sl = __shfl_up_sync(0xffffffffu, sc.w, 1);
        uint32_t sr = __shfl_down_sync(0xffffffffu, sc.x, 1);
        if (lane == 0) sl = __umulhi(el, a);
        if (lane == 31) sr = __umulhi(er, a);
        const uint4 o = update4(vc, sc, su, sd, sl, sr);
        if (y < H) store4(d + (int64_t)(y + 1) * pitch, o, nvalid);
        su = sc;
        sc = sd;
        vc = vd;
    }
}

// ---------------------------------------------------------------------------------------
// K steps per launch, the tile held in registers (temporal blocking).  CTA (tile_x, tile_y,
// field) loads padded words [tx0, tx0 + 128) (tx0 = tile_x * (128 - 2 HALO) + 4 - HALO) of the
// NW * RPW interior rows starting at ty0 - K; warp w keeps rows [RPW w, RPW w + RPW) of the
// tile in registers, lane l words [4l, 4l + 4).  Per step a warp publishes the shares of its
// first and last row in shared memory (double-buffered by step parity: one barrier per
// step), reads its neighbours' and updates its RPW rows in place; left/right shares come by
// __shfl (the tile's outermost lanes read their own share instead: those words are halo,
// invalid after one step and never written).  After K steps the valid region is the tile
// shrunk by K rows and K words on each side; the CTA writes rows [K, NW*RPW - K) of words
// [HALO, 128 - HALO).  Tiles that touch the grid edge (or the padding) force the cells
// outside the grid back to 0 after every step (the padding points of PAPER.md:570, held at
// 0 by one AND per cell); the other tiles skip the mask.
template <int K, int NW, int RPW, bool MASK>
__device__ __forceinline__ void tblock_run(uint4 (&v)[RPW], uint4* pub, int w, int lane, uint32_t a,
                                           uint4 cm, uint32_t rmask) {
#pragma unroll 1
    for (int step = 0; step < K; ++step) {
        // shares are formed on the fly (three rows live), so the tile itself is most of
        // the register budget; only the first and last row's shares are formed up front
        const uint4 sfirst = share4(v[0], a), slast = share4(v[RPW - 1], a);
        uint4* top = pub + (step & 1) * (2 * NW * 32);  // [NW][32] first-row shares
        uint4* bot = top + NW * 32;                     // [NW][32] last-row shares
        top[w * 32 + lane] = sfirst;
        bot[w * 32 + lane] = slast;
        __syncthreads();
        const uint4 zero = make_uint4(0, 0, 0, 0);
        uint4 su = w > 0 ? bot[(w - 1) * 32 + lane] : zero;
        const uint4 ed = w < NW - 1 ? top[(w + 1) * 32 + lane] : zero;
        uint4 sc = sfirst;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            // v[r + 1] still holds the previous step's value here
            const uint4 sd = r == RPW - 1 ? ed : (r == RPW - 2 ? slast : share4(v[r + 1], a));
            const uint32_t sl = __shfl_up_sync(0xffffffffu, sc.w, 1);
            const uint32_t sr = __shfl_down_sync(0xffffffffu, sc.x, 1);
            uint4 o = update4(v[r], sc, su, sd, sl, sr);
            if (MASK) {
                const uint32_t rm = (rmask >> r) & 1u ? 0xffffffffu : 0u;
                o.x &= cm.x & rm;
                o.y &= cm.y & rm;
                o.z &= cm.z & rm;
                o.w &= cm.w & rm;
            }
            v[r] = o;
            su = sc;
            sc = sd;
        }
    }
}

template <int K, int NW, int RPW>
__global__ void __launch_bounds__(NW * 32, SIMCOV_TB_MINB) diffuse_tblock_kernel(const uint32_t* __restrict__ src,
                                                                 uint32_t* __restrict__ dst, int64_t pitch,
                                                                 int64_t fstride, int H, int W,
                                                                 const __grid_constant__ Rates rates) {
    constexpr int HALO = K <= 4 ? 4 : 8;        // words on each side (whole lanes)
    constexpr int OUTC = 128 - 2 * HALO;         // written words per row
    constexpr int TH = NW * RPW - 2 * K;         // written rows per tile
    __shared__ uint4 pub[2 * 2 * NW * 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int field = blockIdx.z;
    const uint32_t a = rates.a[field];
    // padded column of the tile's word 0: word HALO is interior column blockIdx.x * OUTC
    const int64_t tx0 = (int64_t)blockIdx.x * OUTC + kColPad - HALO;
    const int ty0 = blockIdx.y * TH;                     // first written interior row
    const int gx = (int)tx0 - (int)kColPad + lane * 4;   // interior column of the lane's .x
    const int64_t pc = tx0 + lane * 4;                   // padded column of the lane's .x
    const bool col_in_alloc = pc >= 0 && pc + 4 <= pitch; // pc, pitch: multiples of 4
    const int gy0 = ty0 - K + w * RPW;                   // interior row of the warp's row 0
    const uint32_t* s = src + (int64_t)field * fstride + pc;
    uint4 v[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const int pr = gy0 + r + 1;
        v[r] = (pr >= 0 && pr < H + 2 && col_in_alloc) ? ldg4(s + (int64_t)pr * pitch) : make_uint4(0, 0, 0, 0);
    }
    // does the tile (with its halo) reach outside the grid?  CTA-uniform.
    const bool edge = ty0 - K < 0 || ty0 - K + NW * RPW > H || (int)tx0 - (int)kColPad < 0 ||
                      (int)tx0 - (int)kColPad + 128 > W;
    if (edge) {
        const uint4 cm = make_uint4(gx >= 0 && gx < W ? ~0u : 0u, gx + 1 >= 0 && gx + 1 < W ? ~0u : 0u,
                                    gx + 2 >= 0 && gx + 2 < W ? ~0u : 0u, gx + 3 >= 0 && gx + 3 < W ? ~0u : 0u);
        uint32_t rmask = 0;
#pragma unroll
        for (int r = 0; r < RPW; ++r) rmask |= (gy0 + r >= 0 && gy0 + r < H) ? (1u << r) : 0u;
        tblock_run<K, NW, RPW, true>(v, pub, w, lane, a, cm, rmask);
    } else {
        tblock_run<K, NW, RPW, false>(v, pub, w, lane, a, make_uint4(0, 0, 0, 0), 0u);
    }
    if (lane < HALO / 4 || lane >= 32 - HALO / 4 || gx >= W) return;
    uint32_t* d = dst + (int64_t)field * fstride + pc;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const int row = w * RPW + r, gy = gy0 + r;
        if (row >= K && row < K + TH && gy < H) store4(d + (int64_t)(gy + 1) * pitch, v[r], W - gx);
    }
}

// The same K-step tile computation as a persistent kernel: each CTA walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ...; while it computes one tile in registers, cp.async copies the next
// tile's rows (each thread its own 16-byte words) into a shared staging area, so HBM latency is
// paid once per CTA instead of once per tile.
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gptr, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(saddr), "l"(gptr), "r"(valid ? 16 : 0) : "memory");
}

template <int K, int NW, int RPW>
__global__ void __launch_bounds__(NW * 32, SIMCOV_TB_MINB) diffuse_tblock_pipe_kernel(
    const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int64_t pitch, int64_t fstride, int H, int W,
    int n_fields, int ntx, int nty, const __grid_constant__ Rates rates) {
    constexpr int HALO = K <= 4 ? 4 : 8;
    constexpr int OUTC = 128 - 2 * HALO;
    constexpr int TH = NW * RPW - 2 * K;
    constexpr int NT = NW * 32;
    extern __shared__ uint4 stage[];           // [RPW][NT]: thread-contiguous per row
    __shared__ uint4 pub[2 * 2 * NW * 32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t total = (int64_t)ntx * nty * n_fields;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(stage);
    auto prefetch = [&](int64_t tile) {
        const int tx = (int)(tile % ntx);
        const int64_t rest = tile / ntx;
        const int ty = (int)(rest % nty), field = (int)(rest / nty);
        const int64_t tx0 = (int64_t)tx * OUTC + kColPad - HALO;
        const int64_t pc = tx0 + lane * 4;
        const bool cin = pc >= 0 && pc + 4 <= pitch;
        const int gy0 = ty * TH - K + w * RPW;
        const uint32_t* s = src + (int64_t)field * fstride + (cin ? pc : 0);
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int pr = gy0 + r + 1;
            const bool ok = cin && pr >= 0 && pr < H + 2;
            cp_async16(sbase + (uint32_t)((r * NT + tid) * 16), ok ? s + (int64_t)pr * pitch : src, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int64_t tile = blockIdx.x;
    if (tile >= total) return;
    prefetch(tile);
    for (; tile < total; tile += gridDim.x) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        uint4 v[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) v[r] = stage[r * NT + tid];
        __syncthreads();  // every thread's staged words are in registers before the next copy lands
        if (tile + gridDim.x < total) prefetch(tile + gridDim.x);
        const int tx = (int)(tile % ntx);
        const int64_t rest = tile / ntx;
        const int ty = (int)(rest % nty), field = (int)(rest / nty);
        const uint32_t a = rates.a[field];
        const int64_t tx0 = (int64_t)tx * OUTC + kColPad - HALO;
        const int ty0 = ty * TH;
        const int gx = (int)tx0 - (int)kColPad + lane * 4;
        const int64_t pc = tx0 + lane * 4;
        const int gy0 = ty0 - K + w * RPW;
        const bool edge = ty0 - K < 0 || ty0 - K + NW * RPW > H || (int)tx0 - (int)kColPad < 0 ||
                          (int)tx0 - (int)kColPad + 128 > W;
        if (edge) {
            const uint4 cm = make_uint4(gx >= 0 && gx < W ? ~0u : 0u, gx + 1 >= 0 && gx + 1 < W ? ~0u : 0u,
                                        gx + 2 >= 0 && gx + 2 < W ? ~0u : 0u, gx + 3 >= 0 && gx + 3 < W ? ~0u : 0u);
            uint32_t rmask = 0;
#pragma unroll
            for (int r = 0; r < RPW; ++r) rmask |= (gy0 + r >= 0 && gy0 + r < H) ? (1u << r) : 0u;
            tblock_run<K, NW, RPW, true>(v, pub, w, lane, a, cm, rmask);
        } else {
            tblock_run<K, NW, RPW, false>(v, pub, w, lane, a, make_uint4(0, 0, 0, 0), 0u);
        }
        if (!(lane < HALO / 4 || lane >= 32 - HALO / 4 || gx >= W)) {
            uint32_t* d = dst + (int64_t)field * fstride + pc;
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const int row = w * RPW + r, gy = gy0 + r;
                if (row >= K && row < K + TH && gy < H) store4(d + (int64_t)(gy + 1) * pitch, v[r], W - gx);
            }
        }
        __syncthreads();  // the exchange buffer `pub` is reused by the next tile's first step
    }
}

// ---------------------------------------------------------------------------------------
// Zero every padding word of n_fields padded fields: warp per padded row.
__global__ void zero_ring_kernel(uint32_t* __restrict__ g, int64_t pitch, int64_t fstride, int H, int W,
                                 int n_fields) {
    const int lane = threadIdx.x & 31;
    const int64_t nrows = (int64_t)n_fields * (H + 2);
    for (int64_t wr = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wr < nrows;
         wr += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int field = (int)(wr / (H + 2));
        const int pr = (int)(wr % (H + 2));
        uint32_t* row = g + (int64_t)field * fstride + (int64_t)pr * pitch;
        if (pr == 0 || pr == H + 1) {
            for (int64_t c = lane * 4; c < pitch; c += 128)
                *reinterpret_cast<uint4*>(row + c) = make_uint4(0, 0, 0, 0);
        } else {
            if (lane == 0) *reinterpret_cast<uint4*>(row) = make_uint4(0, 0, 0, 0);
            for (int64_t c = kColPad + W + lane; c < pitch; c += 32) row[c] = 0u;
        }
    }
}

// dense <-> padded, warp per (field, interior row); dense rows are not 16-byte aligned
template <bool TO_PADDED>
__global__ void convert_kernel(const uint32_t* __restrict__ from, uint32_t* __restrict__ to, int64_t pitch,
                               int64_t fstride, int H, int W, int n_fields) {
    const int lane = threadIdx.x & 31;
    const int64_t nrows = (int64_t)n_fields * H;
    for (int64_t wr = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wr < nrows;
         wr += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int field = (int)(wr / H);
        const int y = (int)(wr % H);
        const int64_t dense = ((int64_t)field * H + y) * W;
        const int64_t padded = (int64_t)field * fstride + (int64_t)(y + 1) * pitch + kColPad;
        for (int x = lane; x < W; x += 32) {
            if (TO_PADDED) to[padded + x] = from[dense + x];
            else to[dense + x] = from[padded + x];
        }
    }
}

int grid_stride_blocks(int64_t work_warps) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (work_warps + 7) / 8;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

sw_status_t fail(sw_status_t st, const std::string& msg) {
    g_err = msg;
    return st;
}

sw_status_t check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return SW_OK;
}

sw_status_t check_layout(const void* p, int64_t H, int64_t W, int32_t n_fields, int64_t fstride) {
    if (!p) return fail(SW_ERR_INVALID_ARGUMENT, "null pointer");
    if (H < 0 || W < 0 || H > (1 << 30) || W > (1 << 30)) return fail(SW_ERR_INVALID_ARGUMENT, "bad H or W");
    if (n_fields < 1 || n_fields > SIMCOV_MAX_FIELDS) return fail(SW_ERR_INVALID_ARGUMENT, "n_fields out of range");
    const int64_t words = simcov_grid_words(H, W);
    if (words < 0 || fstride < words || (fstride & 3)) return fail(SW_ERR_INVALID_ARGUMENT, "bad field_stride");
    if (reinterpret_cast<uintptr_t>(p) & 15) return fail(SW_ERR_INVALID_ARGUMENT, "pointer not 16-byte aligned");
    return SW_OK;
}

#ifndef SIMCOV_STEP_ROWS
#define SIMCOV_STEP_ROWS 4
#endif
constexpr int kStepRows = SIMCOV_STEP_ROWS;  // rows per warp of the one-step kernel

sw_status_t launch_step(const uint32_t* src, uint32_t* dst, int64_t pitch, int64_t fstride, int H, int W,
                        int n_fields, const Rates& rates, cudaStream_t st) {
    const int n_strips = (W + kStripCols - 1) / kStripCols;
    const int n_chunks = (H + kStepRows - 1) / kStepRows;
    const int64_t warps = (int64_t)n_strips * n_chunks * n_fields;
    const int64_t blocks = (warps + 7) / 8;
    diffuse_step_kernel<kStepRows><<<(unsigned)blocks, 256, 0, st>>>(src, dst, pitch, fstride, H, W, n_strips,
                                                                     n_chunks, n_fields, rates);
    ++g_launches;
    return check_launch("diffuse_step_kernel");
}

#ifndef SIMCOV_TB_PIPE
#define SIMCOV_TB_PIPE 0  // persistent CTAs with a cp.async-prefetched next tile: measured slower
#endif

template <int K>
sw_status_t launch_tblock_pipe_k(const uint32_t* src, uint32_t* dst, int64_t pitch, int64_t fstride, int H, int W,
                                 int n_fields, const Rates& rates, cudaStream_t st) {
    constexpr int HALO = K <= 4 ? 4 : 8, TH = kTbWarps * kTbRowsPerWarp - 2 * K;
    const int ntx = (W + 128 - 2 * HALO - 1) / (128 - 2 * HALO), nty = (H + TH - 1) / TH;
    const size_t smem = (size_t)kTbRowsPerWarp * kTbWarps * 32 * 16;
    auto kern = diffuse_tblock_pipe_kernel<K, kTbWarps, kTbRowsPerWarp>;
    static int occ = -1;  // per process: CTAs per SM of this instantiation
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (occ < 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTbWarps * 32, smem) != cudaSuccess || occ < 1) occ = 1;
    }
    const int64_t total = (int64_t)ntx * nty * n_fields;
    const int blocks = (int)std::min<int64_t>(total, (int64_t)sms * occ);
    kern<<<blocks, kTbWarps * 32, smem, st>>>(src, dst, pitch, fstride, H, W, n_fields, ntx, nty, rates);
    ++g_launches;
    return check_launch("diffuse_tblock_pipe_kernel");
}

template <int K>
sw_status_t launch_tblock_k(const uint32_t* src, uint32_t* dst, int64_t pitch, int64_t fstride, int H, int W,
                            int n_fields, const Rates& rates, cudaStream_t st) {
    constexpr int HALO = K <= 4 ? 4 : 8, TH = kTbWarps * kTbRowsPerWarp - 2 * K;
    dim3 grid((unsigned)((W + 128 - 2 * HALO - 1) / (128 - 2 * HALO)), (unsigned)((H + TH - 1) / TH),
              (unsigned)n_fields);
    if (SIMCOV_TB_PIPE) return launch_tblock_pipe_k<K>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
    if (grid.y > 65535u) return fail(SW_ERR_INVALID_ARGUMENT, "grid too tall for the temporal-blocking schedule");
    diffuse_tblock_kernel<K, kTbWarps, kTbRowsPerWarp><<<grid, kTbWarps * 32, 0, st>>>(src, dst, pitch, fstride, H,
                                                                                        W, rates);
    ++g_launches;
    return check_launch("diffuse_tblock_kernel");
}

sw_status_t launch_k(int k, const uint32_t* src, uint32_t* dst, int64_t pitch, int64_t fstride, int H, int W,
                     int n_fields, const Rates& rates, cudaStream_t st) {
    switch (k) {
        case 1: return launch_tblock_k<1>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 2: return launch_tblock_k<2>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 3: return launch_tblock_k<3>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 4: return launch_tblock_k<4>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 5: return launch_tblock_k<5>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 6: return launch_tblock_k<6>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 7: return launch_tblock_k<7>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        case 8: return launch_tblock_k<8>(src, dst, pitch, fstride, H, W, n_fields, rates, st);
        default: return fail(SW_ERR_INTERNAL, "bad steps per launch");
    }
}

}  // namespace

extern "C" {

int64_t simcov_grid_pitch(int64_t W) {
    if (W < 0 || W > (1 << 30)) return -1;
    const int64_t strips = (W + kStripCols - 1) / kStripCols * kStripCols;
    // strips * 128 interior words + 4 left + >= 4 right (lane 31's right neighbour), rows on 128 B
    return (strips + 2 * kColPad + 31) / 32 * 32;
}

int64_t simcov_grid_words(int64_t H, int64_t W) {
    if (H < 0 || H > (1 << 30)) return -1;
    const int64_t p = simcov_grid_pitch(W);
    return p < 0 ? -1 : (H + 2) * p;
}

sw_status_t simcov_pad(const uint32_t* dense, uint32_t* padded, int64_t H, int64_t W, int32_t n_fields,
                       int64_t field_stride, void* stream) {
    sw_status_t st = check_layout(padded, H, W, n_fields, field_stride);
    if (st != SW_OK) return st;
    if (!dense && H * W > 0) return fail(SW_ERR_INVALID_ARGUMENT, "null dense pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t pitch = simcov_grid_pitch(W);
    zero_ring_kernel<<<grid_stride_blocks((int64_t)n_fields * (H + 2)), 256, 0, s>>>(padded, pitch, field_stride,
                                                                                     (int)H, (int)W, n_fields);
    if ((st = check_launch("zero_ring_kernel")) != SW_OK) return st;
    if (H * W == 0) return SW_OK;
    convert_kernel<true><<<grid_stride_blocks((int64_t)n_fields * H), 256, 0, s>>>(dense, padded, pitch, field_stride,
                                                                                   (int)H, (int)W, n_fields);
    return check_launch("convert_kernel<pad>");
}

sw_status_t simcov_unpad(const uint32_t* padded, uint32_t* dense, int64_t H, int64_t W, int32_t n_fields,
                         int64_t field_stride, void* stream) {
    sw_status_t st = check_layout(padded, H, W, n_fields, field_stride);
    if (st != SW_OK) return st;
    if (H * W == 0) return SW_OK;
    if (!dense) return fail(SW_ERR_INVALID_ARGUMENT, "null dense pointer");
    convert_kernel<false><<<grid_stride_blocks((int64_t)n_fields * H), 256, 0, (cudaStream_t)stream>>>(
        padded, dense, simcov_grid_pitch(W), field_stride, (int)H, (int)W, n_fields);
    return check_launch("convert_kernel<unpad>");
}

sw_status_t simcov_diffuse(uint32_t* grid, uint32_t* scratch, int64_t H, int64_t W, int32_t n_fields,
                           int64_t field_stride, const uint32_t* rates, int32_t steps, void* stream) {
    g_launches = 0;
    sw_status_t st = check_layout(grid, H, W, n_fields, field_stride);
    if (st != SW_OK) return st;
    if ((st = check_layout(scratch, H, W, n_fields, field_stride)) != SW_OK) return st;
    if (!rates) return fail(SW_ERR_INVALID_ARGUMENT, "null rates");
    if (steps < 0) return fail(SW_ERR_INVALID_ARGUMENT, "steps < 0");
    const int64_t bytes = (int64_t)n_fields * field_stride * 4;
    const char *g0 = (const char*)grid, *s0 = (const char*)scratch;
    if (g0 < s0 + bytes && s0 < g0 + bytes) return fail(SW_ERR_INVALID_ARGUMENT, "grid and scratch overlap");
    Rates r{};
    for (int f = 0; f < n_fields; ++f) {
        if (rates[f] > SIMCOV_MAX_RATE) return fail(SW_ERR_INVALID_ARGUMENT, "rate > 2^30");
        r.a[f] = rates[f];
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t pitch = simcov_grid_pitch(W);
    const int h = (int)H, w = (int)W;
    // both ping-pong buffers need a zero ring: the kernels write interior words only
    for (uint32_t* g : {grid, scratch}) {
        zero_ring_kernel<<<grid_stride_blocks((int64_t)n_fields * (H + 2)), 256, 0, s>>>(g, pitch, field_stride, h, w,
                                                                                         n_fields);
        ++g_launches;
        if ((st = check_launch("zero_ring_kernel")) != SW_OK) return st;
    }
    if (steps == 0 || H * W == 0) return SW_OK;

    // the launch plan: steps per launch, an even number of launches so the result lands in grid
    int kmax = g_schedule;
    if (kmax == 0) kmax = kTbMaxK;
    if (kmax > SIMCOV_MAX_TBLOCK) kmax = SIMCOV_MAX_TBLOCK;
    if ((H + kTbWarps * kTbRowsPerWarp - 2 * 8 - 1) / (kTbWarps * kTbRowsPerWarp - 2 * 8) > 65535) kmax = 1;  // grid.y limit
    if (kmax == 1 || steps == 1) {
        // one step per launch (marching kernel); odd counts end with a copy back
        uint32_t *a = grid, *b = scratch;
        for (int i = 0; i < steps; ++i) {
            if ((st = launch_step(a, b, pitch, field_stride, h, w, n_fields, r, s)) != SW_OK) return st;
            std::swap(a, b);
        }
        if (a != grid) {
            if (cudaMemcpyAsync(grid, scratch, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                return fail(SW_ERR_CUDA, "copy back");
        }
        return SW_OK;
    }
    int64_t left = steps;
    std::vector<int> ks;
    while (left > 0) {
        const int k = (int)std::min<int64_t>(kmax, left);
        ks.push_back(k);
        left -= k;
    }
    if (ks.size() & 1) {  // split the last launch with k >= 2 into two
        for (size_t i = ks.size(); i-- > 0;) {
            if (ks[i] >= 2) {
                const int k = ks[i];
                ks[i] = k / 2;
                ks.insert(ks.begin() + i + 1, k - k / 2);
                break;
            }
        }
    }
    uint32_t *a = grid, *b = scratch;
    for (int k : ks) {
        if ((st = launch_k(k, a, b, pitch, field_stride, h, w, n_fields, r, s)) != SW_OK) return st;
        std::swap(a, b);
    }
    if (a != grid) {  // only when every launch has k = 1 (not reached: steps >= 2 and kmax >= 2)
        if (cudaMemcpyAsync(grid, scratch, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return fail(SW_ERR_CUDA, "copy back");
    }
    return SW_OK;
}

sw_status_t simcov_set_schedule(int32_t steps_per_launch) {
    if (steps_per_launch < 0 || steps_per_launch > SIMCOV_MAX_TBLOCK)
        return fail(SW_ERR_INVALID_ARGUMENT, "steps_per_launch out of range");
    g_schedule = steps_per_launch;
    return SW_OK;
}

int32_t simcov_last_launch_count(void) { return g_launches; }

const char* simcov_last_error_message(void) { return g_err.c_str(); }

}  // extern "C"
