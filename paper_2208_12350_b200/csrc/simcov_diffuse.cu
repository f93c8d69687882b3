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
//   marches down R rows keeping the rows above and below in registers (each
//   word is loaded once), left/right neighbour shares by __shfl (only the two
//   strip-edge lanes load a scalar from the padding or the next strip);
// * temporal blocking (k <= 4 steps per launch): a CTA stages a 128-word x
//   (64 + 2k)-row tile in shared memory, runs k steps there (the valid region
//   shrinks by one cell per step) and writes only its 120 x 64 core, so HBM
//   traffic is 8 B per cell per k steps plus the halo re-reads.  Inside the tile
//   the cells outside the grid are forced back to 0 after every step -- the same
//   padding points, now held at 0 in shared memory by one select per cell
//   (a per-thread column mask computed once, a row compare per row).

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
constexpr int kTbMaxK = 4;       // temporal blocking: halo of 4 words covers k <= 4
constexpr int kTbWarps = 8;
constexpr int kTbRowsPerWarp = 9;
constexpr int kTbRows = kTbWarps * kTbRowsPerWarp;  // 72 staged rows
constexpr int kTbCols = 128;                        // staged words per row (32 lanes x 4)
constexpr int kTbOutCols = kTbCols - 2 * 4;         // 120 written columns

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
// K steps per launch through shared memory (temporal blocking).  CTA (tile_x, tile_y,
// field) stages padded words [tx0, tx0 + 128) of interior rows [ty0 - K, ty0 - K + 72)
// (tx0 = tile_x * 120: interior columns tx0 - 4 .. tx0 + 123), runs K steps and writes
// interior rows [ty0, ty0 + 72 - 2K) x columns [tx0, tx0 + 120).  Warp w marches rows
// [9w, 9w + 9) of the tile; lane l owns words [4l, 4l + 4).
template <int K>
__global__ void __launch_bounds__(kTbWarps * 32) diffuse_tblock_kernel(const uint32_t* __restrict__ src,
                                                                       uint32_t* __restrict__ dst,
                                                                       int64_t pitch, int64_t fstride, int H,
                                                                       int W, const __grid_constant__ Rates rates) {
    extern __shared__ uint4 smem[];
    uint4* buf0 = smem;                       // [kTbRows][32]
    uint4* buf1 = smem + kTbRows * 32;
    constexpr int TH = kTbRows - 2 * K;       // written rows per tile
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int field = blockIdx.z;
    const uint32_t a = rates.a[field];
    const int64_t tx0 = (int64_t)blockIdx.x * kTbOutCols;  // padded column of the tile's word 0
    const int ty0 = blockIdx.y * TH;                       // first written interior row
    const int gx = (int)tx0 - (int)kColPad + lane * 4;     // interior column of the lane's .x
    const int64_t pc = tx0 + lane * 4;                     // padded column of the lane's .x
    const uint32_t* s = src + (int64_t)field * fstride + pc;
    const bool col_in_alloc = pc + 4 <= pitch;
    // per-cell interior column mask, fixed for the whole launch
    const bool c0 = gx >= 0 && gx < W, c1 = gx + 1 >= 0 && gx + 1 < W;
    const bool c2 = gx + 2 >= 0 && gx + 2 < W, c3 = gx + 3 >= 0 && gx + 3 < W;
    const int row0 = w * kTbRowsPerWarp;

    // stage: tile row r <-> interior row ty0 - K + r <-> padded row ty0 - K + r + 1
#pragma unroll
    for (int r = 0; r < kTbRowsPerWarp; ++r) {
        const int pr = ty0 - K + row0 + r + 1;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (pr >= 0 && pr < H + 2 && col_in_alloc) v = ldg4(s + (int64_t)pr * pitch);
        buf0[(row0 + r) * 32 + lane] = v;
    }
    __syncthreads();

#pragma unroll 1
    for (int step = 1; step <= K; ++step) {
        const uint4* cur = (step & 1) ? buf0 : buf1;
        uint4* nxt = (step & 1) ? buf1 : buf0;
        const bool last = step == K;
        // rows outside [step, kTbRows - step) are no longer valid after this step
        const int lo = max(row0, last ? K : step);
        const int hi = min(row0 + kTbRowsPerWarp, last ? K + TH : kTbRows - step);
        if (lo < hi) {  // warp-uniform
            uint4 sc = share4(cur[lo * 32 + lane], a);
            uint4 vc = cur[lo * 32 + lane];
            uint4 su = share4(cur[(lo - 1) * 32 + lane], a);  // lo >= 1
            for (int row = lo; row < hi; ++row) {
                const uint4 vd = cur[(row + 1) * 32 + lane];   // row + 1 <= kTbRows - 1
                const uint4 sd = share4(vd, a);
                uint32_t sl = __shfl_up_sync(0xffffffffu, sc.w, 1);
                uint32_t sr = __shfl_down_sync(0xffffffffu, sc.x, 1);
                if (lane == 0) sl = 0;   // beyond the tile: garbage halo, never read back
                if (lane == 31) sr = 0;
                uint4 o = update4(vc, sc, su, sd, sl, sr);
                const int gy = ty0 - K + row;
                const bool rin = gy >= 0 && gy < H;
                o.x = (rin && c0) ? o.x : 0u;  // padding points stay 0
                o.y = (rin && c1) ? o.y : 0u;
                o.z = (rin && c2) ? o.z : 0u;
                o.w = (rin && c3) ? o.w : 0u;
                if (!last) {
                    nxt[row * 32 + lane] = o;
                } else if (rin && lane >= 1 && lane <= 30 && gx < W) {
                    store4(dst + (int64_t)field * fstride + (int64_t)(gy + 1) * pitch + pc, o, W - gx);
                }
                su = sc;
                sc = sd;
                vc = vd;
            }
        }
        if (!last) __syncthreads();
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

constexpr int kStepRows = 16;

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

template <int K>
sw_status_t launch_tblock_k(const uint32_t* src, uint32_t* dst, int64_t pitch, int64_t fstride, int H, int W,
                            int n_fields, const Rates& rates, cudaStream_t st) {
    constexpr int TH = kTbRows - 2 * K;
    const size_t smem = 2 * (size_t)kTbRows * kTbCols * sizeof(uint32_t);
    static bool attr = false;  // per process; the attribute is per device function
    if (!attr) {
        cudaFuncSetAttribute(diffuse_tblock_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid((unsigned)((W + kTbOutCols - 1) / kTbOutCols), (unsigned)((H + TH - 1) / TH), (unsigned)n_fields);
    if (grid.y > 65535u) return fail(SW_ERR_INVALID_ARGUMENT, "grid too tall for the temporal-blocking schedule");
    diffuse_tblock_kernel<K><<<grid, kTbWarps * 32, smem, st>>>(src, dst, pitch, fstride, H, W, rates);
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
    if (kmax > kTbMaxK) kmax = kTbMaxK;
    if ((H + kTbRows - 2 * kTbMaxK - 1) / (kTbRows - 2 * kTbMaxK) > 65535) kmax = 1;  // grid.y limit
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
