// sw_api.cu -- host side of the C ABI declared in include/sw.h: argument and
// scoring validation, workspace management, the launch sequence
//   pack -> sort -> forward wavefront -> finish_fwd -> sort -> reverse
//   wavefront -> finish_rev
// and the instrumentation entry points.  No exceptions cross the ABI.

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "sw.h"
#include <cub/device/device_radix_sort.cuh>
#include "sw_common.cuh"
#include "sw_pack.cuh"
#include "sw_wavefront.cuh"
#include "sw_finish.cuh"
#include "sw_band.cuh"
#include "sw_traceback.cuh"

using namespace swb;

namespace {

// Kernel geometry of this build: 16-lane segments, 10 rows
// per lane -> 160-row stripes (one stripe covers the ADEPT-shaped 150 bp reads).
#ifndef SW_W16
#define SW_W16 16
#endif
#ifndef SW_K16
#define SW_K16 10
#endif
constexpr int W16 = SW_W16, K16 = SW_K16;
// protein: 8 rows per lane keep the 25-code int8 profile at 8 bytes per (code, lane) -> 12.8 KB per
// warp, so shared memory allows 16 resident warps per SM (10 rows would need 16-byte entries)
constexpr int WP = SW_WP, KP = SW_KP;
constexpr int W32 = 16, K32 = 10;
constexpr int WARPS_PER_BLOCK = 4;
using G16 = Geometry<W16, K16, TS16>;
using G16F = Geometry<W16, K16, TS16, SW_IMERGE && SW_TAG_LAZY && K16 == 10>;  // DNA TAG forward kernels
using GP = Geometry<WP, KP, TS16>;
using G32 = Geometry<W32, K32, TS32>;

// The wavefront kernel of a pass (REV), gap model (LIN: gap_open == gap_extend), alphabet and
// route.  The int32 route keeps the affine kernel for linear gaps (same results, o = e).
template <bool REV, bool LIN>
const void* wave_kernel_ptr(bool protein, int route) {
    if (route == ROUTE_S32) return (const void*)wavefront_kernel<TS32, W32, K32, REV, false, false>;
    const bool tag = route == ROUTE_TAG;
    if (protein)
        return tag ? (const void*)wavefront_kernel<TS16, WP, KP, REV, true, LIN>
                   : (const void*)wavefront_kernel<TS16, WP, KP, REV, false, LIN>;
    return tag ? (const void*)wavefront_kernel<TS16, W16, K16, REV, true, LIN>
               : (const void*)wavefront_kernel<TS16, W16, K16, REV, false, LIN>;
}

void wave_kernels(bool protein, bool lin, const void** kfwd, const void** krev) {
    for (int r = 0; r < N_ROUTES; ++r) {
        kfwd[r] = lin ? wave_kernel_ptr<false, true>(protein, r) : wave_kernel_ptr<false, false>(protein, r);
        krev[r] = lin ? wave_kernel_ptr<true, true>(protein, r) : wave_kernel_ptr<true, false>(protein, r);
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
};

}  // namespace

constexpr int MAX_CHUNKS = 8;
constexpr int N_SLOTS = 2;

struct sw_context {
    int device = 0;
    int sm_count = 0;
    int occ_s16_fwd = 1, occ_s16_rev = 1, occ_s32_fwd = 1, occ_s32_rev = 1;
    int max_occ_cached_nc = -1;
    cudaStream_t last_stream = nullptr;
    bool have_last = false;
    bool no_spec_ext = false;  // force the synchronous extent read (after a speculative overflow)
    std::string err;

    // per-pair
    DevBuf<int32_t> nlen, mlen, nlen_rev, mlen_rev, target, iota, order, order_rev;
    DevBuf<int64_t> qpos, rpos;
    DevBuf<uint8_t> flags;
    DevBuf<uint32_t> key, key_sorted;
    DevBuf<unsigned long long> keys_fwd, keys_rev;
    // codes
    DevBuf<uint8_t> qcode, rcode, rrev;
    DevBuf<uint8_t> bslots;   // banded reverse pass (sw_band.cuh): slot 0 pads, pair p's slot p + 1
    DevBuf<uint32_t> rcode4;  // SW_CODE4 measurement variant only
    // misc.  Per-slot state: the host-buffer entry point runs consecutive chunks of one batch
    // on two streams (slot k & 1), so their small kernels and tails overlap; slot 0 is the
    // device entry point's.
    DevBuf<uint8_t> scratch[N_SLOTS], cub_temp[N_SLOTS];
    DevBuf<unsigned long long> progress[N_SLOTS];  // cooperative reverse items: per (warp, parity) hand-off progress
    BatchStats* d_stats = nullptr;  // [N_SLOTS]
    BatchStats* h_stats = nullptr;  // [N_SLOTS] (pinned)
    int64_t* h_ext = nullptr;
    int32_t* d_counters = nullptr;  // [N_SLOTS][8] work-queue heads: 3 forward + 3 reverse routes
    uint32_t* d_sink = nullptr;
    uint32_t* d_hist = nullptr;     // [N_SLOTS][NBINS] work-bin histogram (kept zero between passes)
    uint32_t* d_binbase = nullptr;  // [N_SLOTS][NBINS] bin cursors
    cudaStream_t aux_stream = nullptr;  // slot 1's stream
    // host-buffer entry point staging
    DevBuf<uint8_t> st_q, st_r;
    DevBuf<int64_t> st_qo, st_ro;
    DevBuf<int32_t> st_out;
    // alignment paths (sw_traceback): per-warp direction words and stripe boundary rows
    DevBuf<uint32_t> tb_dir;
    DevBuf<int2> tb_bnd;
    int32_t* d_tb = nullptr;   // [0] max a, [1] max b, [2] queue head, [3] internal errors; int64 q0, r0; [8] s16x2 queue head; [9] bad intervals
    int32_t* h_tb = nullptr;   // pinned copy
    bool tb_pending = false;   // a traceback ran since the last sw_batch_status: read its error count
    // asynchronous host-buffer entry point: double-buffered staging, copy-in / copy-out streams
    DevBuf<uint8_t> as_q[2], as_r[2];
    DevBuf<int64_t> as_qo[2], as_ro[2];
    DevBuf<int32_t> as_out[2];
    DevBuf<uint8_t> db_q;     // sw_align_query_db: the broadcast query
    DevBuf<int64_t> db_qo;
    cudaEvent_t as_in[2] = {}, as_comp[2] = {}, as_done[2] = {}, as_start = nullptr;
    bool as_used[2] = {false, false};
    bool as_inflight = false;
    int as_next = 0;
    cudaStream_t out_stream = nullptr;   // device -> host result copies
    cudaStream_t as_stream = nullptr;    // the caller's stream of the submitted batches

    int codes_alphabet = -1;  // alphabet the code buffers were last cleared for
    // sw_reserve: bounds the workspace was sized for; device-buffer calls within them never
    // synchronise (enqueue and return, capturable in a CUDA graph)
    bool reserved = false;
    int64_t res_pairs = 0, res_qbytes = 0, res_rbytes = 0;
    int32_t res_n = 0, res_m = 0;
    cudaStream_t copy_stream = nullptr;  // host-buffer entry point: overlapped copies
    cudaEvent_t ev_in[MAX_CHUNKS] = {}, ev_out[MAX_CHUNKS] = {}, ev_prep = nullptr;
    bool timing = false;
    int mode = SW_MODE_FULL;
    cudaEvent_t ev[8] = {};
    bool ev_valid = false;
    int32_t own_launches = 0, lib_launches = 0;
};

namespace {

sw_status_t fail(sw_context* h, sw_status_t st, const std::string& msg) {
    if (h) h->err = msg;
    return st;
}

sw_status_t cuda_fail(sw_context* h, cudaError_t e, const char* what) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    if (h) h->err = m;
    return e == cudaErrorMemoryAllocation ? SW_ERR_OUT_OF_MEMORY : SW_ERR_CUDA;
}

#ifndef SW_DEBUG_SYNC
#define SW_DEBUG_SYNC 0  // development builds: synchronise after every launch of a call and name the failing one
#endif
#define SW_DBG(h, s, what)                                                                        \
    do {                                                                                          \
        if (SW_DEBUG_SYNC) {                                                                      \
            cudaError_t _e = cudaStreamSynchronize(s);                                            \
            if (_e != cudaSuccess) { fprintf(stderr, "sw debug: %s failed: %s\n", what, cudaGetErrorString(_e)); return cuda_fail((h), _e, what); } \
        }                                                                                         \
    } while (0)

#define SW_CUDA(h, call)                                          \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return cuda_fail((h), _e, #call);  \
    } while (0)

template <class T>
sw_status_t ensure(sw_context* h, DevBuf<T>& b, size_t n) {
    if (n == 0) n = 1;
    if (b.cap >= n) return SW_OK;
    size_t cap = std::max(n, (size_t)(b.cap * 5 / 4));
    if (b.p) {
        cudaError_t e = cudaFree(b.p);
        b.p = nullptr; b.cap = 0;
        if (e != cudaSuccess) return cuda_fail(h, e, "cudaFree");
    }
    cudaError_t e = cudaMalloc(&b.p, cap * sizeof(T));
    if (e != cudaSuccess) {
        // retry exact size
        cap = n;
        e = cudaMalloc(&b.p, cap * sizeof(T));
        if (e != cudaSuccess) { b.p = nullptr; return cuda_fail(h, e, "cudaMalloc(workspace)"); }
    }
    b.cap = cap;
    return SW_OK;
}

template <class T>
void release(DevBuf<T>& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr; b.cap = 0;
}

#if SW_CODE4
// measurement variant: byte codes -> 4-bit codes, 8 per word (nibble k of word w = byte 8w + k)
__global__ void nibble_kernel(const uint8_t* __restrict__ c, uint32_t* __restrict__ c4, size_t words) {
    for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (size_t)gridDim.x * blockDim.x) {
        const uint2 b = reinterpret_cast<const uint2*>(c)[w];
        uint32_t v = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) v |= ((b.x >> (8 * k)) & 15u) << (4 * k);
#pragma unroll
        for (int k = 0; k < 4; ++k) v |= ((b.y >> (8 * k)) & 15u) << (16 + 4 * k);
        c4[w] = v;
    }
}
#endif

// SW_MODE_POISON helper: p[0 .. n) = v.
__global__ void fill_u32_kernel(uint32_t* p, size_t n, uint32_t v) {
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) p[k] = v;
}

// Scoring preconditions (reading R3) and the s16x2 routing condition.
sw_status_t check_scoring(sw_context* h, const sw_scoring_t* s, Scoring& sc, bool& s16_ok) {
    if (!s) return fail(h, SW_ERR_INVALID_ARGUMENT, "scoring is NULL");
    if (s->alphabet != SW_ALPHABET_DNA && s->alphabet != SW_ALPHABET_PROTEIN)
        return fail(h, SW_ERR_INVALID_SCORING, "unknown alphabet");
    if (!(s->gap_open < 0) || s->gap_open < -32768)
        return fail(h, SW_ERR_INVALID_SCORING, "gap_open must be in [-32768, 0)");
    if (!(s->gap_open <= s->gap_extend && s->gap_extend <= 0))
        return fail(h, SW_ERR_INVALID_SCORING, "need gap_open <= gap_extend <= 0");
    int smax, smin;
    if (s->alphabet == SW_ALPHABET_DNA) {
        if (!(s->match > 0) || s->match > 32767) return fail(h, SW_ERR_INVALID_SCORING, "match must be in (0, 32767]");
        if (!(s->mismatch < s->match) || s->mismatch < -32768)
            return fail(h, SW_ERR_INVALID_SCORING, "mismatch must be in [-32768, match)");
        smax = s->match; smin = std::min(s->mismatch, s->match);
    } else {
        smax = BLOSUM62_MAX; smin = BLOSUM62_MIN;
    }
    sc.alphabet = s->alphabet;
    sc.match = s->match;
    sc.mismatch = s->mismatch;
    sc.gap_open = s->gap_open;
    sc.gap_extend = s->gap_extend;
    sc.nc = s->alphabet == SW_ALPHABET_DNA ? NC_DNA : NC_PROTEIN;
    sc.max_sigma = smax;
    // s16x2 path: int8 profile of (s - o) in [-127, 127], gap values whose
    // additions stay inside int16 (shifted values live in [e, 32000]).
    s16_ok = (smax - s->gap_open <= 127) && (smin - s->gap_open >= -127) &&
             s->gap_open >= -8000 && s->gap_extend >= -8000;
    return SW_OK;
}

template <class K>
void set_smem_attr(K kernel, int bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int occupancy_blocks(const void* kernel, int threads, int smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess) nb = 1;
    return std::max(nb, 1);
}

struct Launch {
    int blocks = 0;
    int smem = 0;
    int warps = WARPS_PER_BLOCK;  // warps per block
};

template <class G>
Launch plan_wave(const sw_context* h, const void* kernel, int nc, int64_t n_path, int warps = WARPS_PER_BLOCK) {
    Launch l;
    l.warps = warps;
    l.smem = warps * G::warp_smem(nc);
    const int64_t items = (n_path + G::SLOTS - 1) / G::SLOTS;
    const int64_t need = (items + warps - 1) / warps;
    const int64_t maxb = (int64_t)h->sm_count * occupancy_blocks(kernel, warps * 32, l.smem);
    l.blocks = (int)std::max<int64_t>(0, std::min(need, maxb));
    return l;
}

// Grids of the forward / reverse wavefront launches of every route (persistent, at most one
// resident wave; the kernels pull work items up to the device-side counts).
void plan_waves(const sw_context* h, const Scoring& sc, bool protein, const BatchStats& hs, const void* const* kfwd,
                const void* const* krev, Launch* lf, Launch* lr) {
    for (int r = 0; r < N_ROUTES; ++r) {
        // reverse-pass pairs are a subset of the forward ones (finish_fwd may move TAG pairs to
        // S16): forward counts bound the grids
        const bool demote = protein || (int64_t)sc.max_sigma * hs.max_n > TAG_MAX_SCORE;  // finish_fwd's TAG -> S16 rule
        const int64_t rev_upper = hs.fwd_count[r] + (r == ROUTE_S16 && demote ? hs.fwd_count[ROUTE_TAG] : 0);
        if (r == ROUTE_S32) {
            lf[r] = plan_wave<G32>(h, kfwd[r], sc.nc, hs.fwd_count[r]);
            lr[r] = plan_wave<G32>(h, krev[r], sc.nc, rev_upper);
        } else if (protein) {
            // 3-warp blocks: 5 blocks x 3 warps fit the SM's shared memory (4-warp blocks: only 3)
            lf[r] = plan_wave<GP>(h, kfwd[r], sc.nc, hs.fwd_count[r], SW_PROT_THREADS / 32);
            lr[r] = plan_wave<GP>(h, krev[r], sc.nc, rev_upper, SW_PROT_THREADS / 32);
        } else {
            lf[r] = r == ROUTE_TAG ? plan_wave<G16F>(h, kfwd[r], sc.nc, hs.fwd_count[r])
                                   : plan_wave<G16>(h, kfwd[r], sc.nc, hs.fwd_count[r]);
            lr[r] = plan_wave<G16>(h, krev[r], sc.nc, rev_upper);
        }
    }
}

// Stripe hand-off scratch of a call: per resident warp, segment and parity, one boundary row
// (HO, F) of the longest reference (+ fill/drain); zero unless some query spans two stripes.
size_t scratch_bytes(const Launch* lf, const Launch* lr, const BatchStats& hs, bool protein, int64_t& seg_bytes) {
    size_t need = 0;
    seg_bytes = 0;
    // W slack slots before column 0, the item's longest reference plus fill / drain / prefetch after it
    const int64_t row_bytes = ((int64_t)hs.max_m + 64 + 16 + 16) * 8;
    for (int r = 0; r < N_ROUTES; ++r) {
        const int rows = r == ROUTE_S32 ? G32::ROWS : protein ? GP::ROWS : G16::ROWS;
        const int segs = r == ROUTE_S32 ? G32::SEGS : protein ? GP::SEGS : G16::SEGS;
        if (hs.fwd_count[r] && hs.max_n > rows) {
            seg_bytes = row_bytes;
            need = std::max(need, (size_t)std::max(lf[r].blocks * lf[r].warps, lr[r].blocks * lr[r].warps) * segs * 2 * row_bytes);
        }
    }
    return need;
}

// What the host already knows about a batch (host-buffer entry point): with it the
// pipeline needs no stream synchronisation between enqueueing and completion.
struct HostPlan {
    int64_t ext[4];            // q0, qN, r0, rN of the whole batch (code positions are batch-global)
    int64_t lo, hi;            // this chunk's pairs
    int32_t max_n, max_m;      // longest query / reference of the chunk
    int32_t route_upper[N_ROUTES];  // pairs per route by lengths alone (>= the device's counts)
    bool reset_cumulative;     // first chunk of the slot in a user call
    int slot;                  // per-slot state (statistics, queues, bins, scratch)
};

// Workspace for a batch of N pairs with tq / tr payload bytes (every chunk of a host-buffer
// call uses the batch's sizes, so no buffer moves while two streams run).
sw_status_t prepare_workspace(sw_context* h, size_t N, size_t tq, size_t tr, int alphabet, cudaStream_t s) {
#define ENS(buf, n) do { sw_status_t _s = ensure(h, h->buf, (n)); if (_s != SW_OK) return _s; } while (0)
    ENS(nlen, N); ENS(mlen, N); ENS(nlen_rev, N); ENS(mlen_rev, N); ENS(target, N); ENS(iota, N);
    ENS(order, N); ENS(order_rev, N); ENS(qpos, N); ENS(rpos, N); ENS(flags, N); ENS(key, N); ENS(key_sorted, N);
    ENS(keys_fwd, N); ENS(keys_rev, N);
    ENS(qcode, tq + 32);
    // Every byte of the reference code buffers must be a valid code of the batch's
    // alphabet: finished halves of a work item keep reading past their reference.
    const size_t rbytes = tr + N * (PADL + PADR) + GUARD + 16;
    uint8_t* old_r = h->rcode.p; uint8_t* old_rr = h->rrev.p;
    ENS(rcode, rbytes); ENS(rrev, rbytes);
    if (h->rcode.p != old_r || h->rrev.p != old_rr || h->codes_alphabet != alphabet) {
        SW_CUDA(h, cudaMemsetAsync(h->rcode.p, 0, h->rcode.cap, s));
        SW_CUDA(h, cudaMemsetAsync(h->rrev.p, 0, h->rrev.cap, s));
        h->codes_alphabet = alphabet;
    }
    // banded reverse pass (sw_band.cuh): slot 0 = pads (query pad codes, reference pad selectors: the empty
    // halves of a work item read them), pair p's reversed prefixes in slot p + 1
    uint8_t* old_b = h->bslots.p;
    ENS(bslots, (N + 1) * BAND_SLOT);
    if (h->bslots.p != old_b) {
        SW_CUDA(h, cudaMemsetAsync(h->bslots.p, 0x04, h->bslots.cap, s));
        SW_CUDA(h, cudaMemsetAsync(h->bslots.p + QREV_STRIDE, SEL_PAD, BAND_SLOT - QREV_STRIDE, s));
    }
#undef ENS
    return SW_OK;
}

// Cumulative statistics of the last user call: slot 0's, plus slot 1's totals.
cudaError_t read_stats(sw_context* h, BatchStats& t) {
    cudaError_t e = cudaMemcpy(h->h_stats, h->d_stats, N_SLOTS * sizeof(BatchStats), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    t = h->h_stats[0];
    for (int k = 1; k < N_SLOTS; ++k) {
        const BatchStats& u = h->h_stats[k];
        t.n_bad += u.n_bad; t.internal_err += u.internal_err; t.cells += u.cells;
        t.swept_fwd += u.swept_fwd; t.swept_rev += u.swept_rev; t.malformed |= u.malformed; t.rejected |= u.rejected;
    }
    return cudaSuccess;
}

// Order the pairs by work key (h->key), most work first.  Small-region batches
// (sw_bin.cuh): counting sort on the exact bins pack / finish_fwd histogrammed;
// otherwise a radix sort of the full 32-bit keys.  Leaves the histogram zero.
sw_status_t bin_order(sw_context* h, int32_t* order, int64_t lo, int64_t hi, bool small, int slot, cudaStream_t s) {
    uint32_t* hist = h->d_hist + (size_t)slot * NBINS;
    uint32_t* base = h->d_binbase + (size_t)slot * NBINS;
    const int64_t n = hi - lo;
    if (small) {
        bin_scan_kernel<<<1, BIN_SCAN_THREADS, BIN_SCAN_SMEM, s>>>(hist, base);
        const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)h->sm_count * 8);
        bin_scatter_kernel<<<blocks, 256, 0, s>>>(h->key.p, base, order, lo, hi, &h->d_stats[slot].malformed);
        SW_CUDA(h, cudaGetLastError());
        h->own_launches += 2;
        return SW_OK;
    }
    SW_CUDA(h, cudaMemsetAsync(hist, 0, NBINS * sizeof(uint32_t), s));
    size_t tb = 0;
    SW_CUDA(h, cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, h->key.p + lo, h->key_sorted.p + lo, h->iota.p + lo,
                                                         order, (int)n, 0, 32, s));
    {
        sw_status_t e = ensure(h, h->cub_temp[slot], tb);
        if (e != SW_OK) return e;
    }
    tb = h->cub_temp[slot].cap;
    SW_CUDA(h, cub::DeviceRadixSort::SortPairsDescending(h->cub_temp[slot].p, tb, h->key.p + lo, h->key_sorted.p + lo,
                                                         h->iota.p + lo, order, (int)n, 0, 32, s));
    ++h->lib_launches;
    return SW_OK;
}

// The batch pipeline on device pointers.  host_ext (optional) = {q0, qN, r0, rN}.  With a
// HostPlan, only the plan's pairs [lo, hi) of the n_pairs-pair batch are processed, on the
// plan's slot, with no stream synchronisation.
sw_status_t align_impl(sw_context* h, const uint8_t* queries, const int64_t* q_off, const uint8_t* refs,
                       const int64_t* r_off, int64_t n_pairs, const sw_scoring_t* scoring,
                       const sw_result_t* out, cudaStream_t s, const int64_t* host_ext,
                       const HostPlan* hp = nullptr) {
    int dev = -1;
    SW_CUDA(h, cudaGetDevice(&dev));
    if (dev != h->device) return fail(h, SW_ERR_WRONG_DEVICE, "current device differs from the handle's device");
    Scoring sc;
    bool s16_ok = false;
    sw_status_t st = check_scoring(h, scoring, sc, s16_ok);
    if (st != SW_OK) return st;
    if (n_pairs < 0) return fail(h, SW_ERR_INVALID_ARGUMENT, "n_pairs < 0");
    if (n_pairs > 0x7ffffff0LL) return fail(h, SW_ERR_INVALID_ARGUMENT, "n_pairs exceeds 2^31 - 16");
    if (!hp || (hp->reset_cumulative && hp->slot == 0)) {
        h->own_launches = 0;
        h->lib_launches = 0;
    }
    const int slot = hp ? hp->slot : 0;
    const int64_t lo = hp ? hp->lo : 0, hi = hp ? hp->hi : n_pairs;
    BatchStats* stats = h->d_stats + slot;
    uint32_t* hist = h->d_hist + (size_t)slot * NBINS;
    int32_t* counters = h->d_counters + slot * 8;
    h->ev_valid = false;
    if (n_pairs == 0) return SW_OK;
    const bool end_only = (h->mode & SW_MODE_END_ONLY) != 0;
    if (!queries || !q_off || !refs || !r_off || !out || !out->score || !out->q_end || !out->r_end ||
        (!end_only && (!out->q_start || !out->r_start)))
        return fail(h, SW_ERR_INVALID_ARGUMENT, "NULL pointer argument");
    h->last_stream = s;
    h->have_last = true;
    // reserved call (sw_reserve): nothing is read back; launches are sized from the reservation and
    // the device-side counts, and pack rejects a batch beyond the reservation on the device
    const bool async = !hp && !host_ext && h->reserved && n_pairs <= h->res_pairs;

    // 1. payload extents
    int64_t ext[4] = {0, 0, 0, 0};
    // speculative extents (device-buffer calls once the code buffers exist): pack reads the
    // extents itself and checks they fit the buffers' capacity; the host learns the outcome from
    // the statistics read-back it does anyway (one host round trip per call instead of two)
    const bool spec = async || (!hp && !host_ext && !h->no_spec_ext && h->qcode.cap > 0 && h->rcode.cap > 0 && h->rrev.cap > 0);
    if (hp) {
        std::memcpy(ext, hp->ext, sizeof(ext));
    } else if (host_ext) {
        std::memcpy(ext, host_ext, sizeof(ext));
    } else if (!spec) {
        SW_CUDA(h, cudaMemcpyAsync(h->h_ext + 0, q_off, 8, cudaMemcpyDeviceToHost, s));
        SW_CUDA(h, cudaMemcpyAsync(h->h_ext + 1, q_off + n_pairs, 8, cudaMemcpyDeviceToHost, s));
        SW_CUDA(h, cudaMemcpyAsync(h->h_ext + 2, r_off, 8, cudaMemcpyDeviceToHost, s));
        SW_CUDA(h, cudaMemcpyAsync(h->h_ext + 3, r_off + n_pairs, 8, cudaMemcpyDeviceToHost, s));
        SW_CUDA(h, cudaStreamSynchronize(s));
        std::memcpy(ext, h->h_ext, sizeof(ext));
    }
    const int64_t q0 = ext[0], qN = ext[1], r0 = ext[2], rN = ext[3];
    const size_t N = (size_t)n_pairs;
    if (qN < q0 || rN < r0) {
        fill_invalid_kernel<<<std::min<int64_t>((n_pairs + 255) / 256, 4096), 256, 0, s>>>(*out, 0, n_pairs);
        return fail(h, SW_ERR_INVALID_ARGUMENT, "offsets are not non-decreasing");
    }
    const size_t tq = (size_t)(qN - q0), tr = (size_t)(rN - r0);
    // code buffers keep the payloads' 16-byte phase so pack moves aligned vectors
    const int64_t qshift = spec ? 0 : (int64_t)(((uintptr_t)(queries + q0)) & 15);
    const int64_t rshift = spec ? 0 : (int64_t)(((uintptr_t)(refs + r0)) & 15);

    // 2. workspace
    st = prepare_workspace(h, N, tq, tr, sc.alphabet, s);
    if (st != SW_OK) return st;
#define ENS(buf, n) do { sw_status_t _s = ensure(h, h->buf, (n)); if (_s != SW_OK) return _s; } while (0)

    const bool protein = sc.alphabet == SW_ALPHABET_PROTEIN;
    const int rows16 = protein ? GP::ROWS : G16::ROWS, rows32 = G32::ROWS;
    const bool timing = h->timing && !hp;
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[0], s));

    // debugging (SW_MODE_POISON): whatever this call does not write reads back as poison
    if (h->mode & SW_MODE_POISON) {
        int32_t* fields[5] = {out->score, out->q_end, out->r_end, out->q_start, out->r_start};
        for (int k = 0; k < (end_only ? 3 : 5); ++k)
            SW_CUDA(h, cudaMemsetAsync(fields[k] + lo, 0x7f, (size_t)(hi - lo) * 4, s));
        SW_CUDA(h, cudaMemsetAsync(h->order.p + lo, 0xff, (size_t)(hi - lo) * 4, s));
        SW_CUDA(h, cudaMemsetAsync(h->order_rev.p + lo, 0xff, (size_t)(hi - lo) * 4, s));
        SW_CUDA(h, cudaMemsetAsync(h->nlen_rev.p + lo, 0x7f, (size_t)(hi - lo) * 4, s));
        SW_CUDA(h, cudaMemsetAsync(h->mlen_rev.p + lo, 0x7f, (size_t)(hi - lo) * 4, s));
        SW_CUDA(h, cudaMemsetAsync(h->target.p + lo, 0x7f, (size_t)(hi - lo) * 4, s));
        SW_CUDA(h, cudaMemsetAsync(h->keys_rev.p + lo, 0x7f, (size_t)(hi - lo) * 8, s));
    }

    // 3. pack
    if (!hp) SW_CUDA(h, cudaMemsetAsync(h->d_stats, 0, N_SLOTS * sizeof(BatchStats), s));  // all slots' totals
    else if (hp->reset_cumulative) SW_CUDA(h, cudaMemsetAsync(stats, 0, sizeof(BatchStats), s));
    else SW_CUDA(h, cudaMemsetAsync(reinterpret_cast<uint8_t*>(stats) + STATS_PER_BATCH_OFFSET, 0,
                                    sizeof(BatchStats) - STATS_PER_BATCH_OFFSET, s));
    {
        PackParams P;
        P.queries = queries; P.q_off = q_off; P.refs = refs; P.r_off = r_off; P.lo = lo; P.hi = hi;
        P.q0 = q0; P.qN = qN; P.r0 = r0; P.rN = rN; P.qshift = qshift; P.rshift = rshift;
        P.alphabet = sc.alphabet; P.s16_ok = s16_ok ? 1 : 0; P.max_sigma = sc.max_sigma; P.tag_ok = tag_max_score(sc.alphabet) > 0 && (K16 <= 16 || protein) ? 1 : 0;  // TAG route (DNA; protein: PT)
        P.rows_s16 = rows16; P.rows_s32 = rows32;
        P.ext_dev = spec ? 1 : 0; P.n_all = n_pairs;
        P.qcap = (int64_t)h->qcode.cap; P.rcap = (int64_t)std::min(h->rcode.cap, h->rrev.cap);
        P.cap_n = async ? h->res_n : 0; P.cap_m = async ? h->res_m : 0;
        P.qcode = h->qcode.p; P.rcode = h->rcode.p;
        P.nlen = h->nlen.p; P.mlen = h->mlen.p; P.qpos = h->qpos.p; P.rpos = h->rpos.p; P.flags = h->flags.p; P.key = h->key.p;
        P.hist = hist; P.keys_fwd = h->keys_fwd.p; P.iota = h->iota.p; P.stats = stats;
        // one warp per PACK_PPW pairs, at most one full wave of warps
        const int64_t warps = std::min<int64_t>((hi - lo + PACK_PPW - 1) / PACK_PPW, (int64_t)h->sm_count * 64);
        const int blocks = (int)((warps + PACK_WARPS - 1) / PACK_WARPS);
        pack_kernel<<<blocks, PACK_WARPS * 32, 0, s>>>(P);
        SW_CUDA(h, cudaGetLastError());
        ++h->own_launches;
        SW_DBG(h, s, "launch at sw_api.cu:527");
    }
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[1], s));
    // forward binning enqueued before the read-back below, assuming the common small-region
    // batch: the GPU bins while the host waits; a batch outside it is re-sorted (radix) after
    // (a reserved call knows from the reservation whether every key lies in the small region)
    const int min_rows0 = std::min(rows16, G32::ROWS);
    const bool res_small = async && h->res_m < BIN_COLS && (h->res_n + min_rows0 - 1) / min_rows0 <= BIN_MAX_STRIPES;
    const bool spec_bin = !hp && (!async || res_small);
    if (spec_bin) {
        st = bin_order(h, h->order.p + lo, lo, hi, true, slot, s);
        if (st != SW_OK) return st;
        SW_CUDA(h, cudaMemsetAsync(counters, 0, 8 * sizeof(int32_t), s));  // work queues (step 6)
    }
    // 4. statistics -> grids and scratch (read back, unless the host already knows bounds)
    BatchStats hs;
    if (hp) {
        std::memset(&hs, 0, sizeof(hs));
        hs.max_n = hp->max_n;
        hs.max_m = hp->max_m;
        for (int r = 0; r < N_ROUTES; ++r) hs.fwd_count[r] = hp->route_upper[r];
    } else if (async) {
        // bounds from the reservation: every route may hold every pair (the persistent grids read
        // the real counts on the device), lengths up to the reserved ones
        std::memset(&hs, 0, sizeof(hs));
        hs.max_n = h->res_n;
        hs.max_m = h->res_m;
        // routes a pair within the reservation can take (pack's rule): launch only those
        const bool tag_ok = tag_max_score(sc.alphabet) > 0 && (K16 <= 16 || protein);
        const int64_t smax_all = (int64_t)sc.max_sigma * std::min(h->res_n, h->res_m);
        const bool all_tag = s16_ok && tag_ok && (int64_t)sc.max_sigma * h->res_n <= tag_max_score(sc.alphabet);
        const bool any_s32 = !s16_ok || smax_all > S16_MAX_SCORE;
        hs.fwd_count[ROUTE_TAG] = (s16_ok && tag_ok) ? (int32_t)n_pairs : 0;
        hs.fwd_count[ROUTE_S16] = (s16_ok && !all_tag) ? (int32_t)n_pairs : 0;
        hs.fwd_count[ROUTE_S32] = any_s32 ? (int32_t)n_pairs : 0;
    } else {
        SW_CUDA(h, cudaMemcpyAsync(h->h_stats, stats, sizeof(BatchStats), cudaMemcpyDeviceToHost, s));
        SW_CUDA(h, cudaStreamSynchronize(s));
        hs = *h->h_stats;
    }
    if (hs.overflow) {  // speculative extents did not fit: grow with the synchronous read, re-run
        h->no_spec_ext = true;
        st = align_impl(h, queries, q_off, refs, r_off, n_pairs, scoring, out, s, nullptr, nullptr);
        h->no_spec_ext = false;
        return st;
    }
    if (hs.malformed) {
        SW_CUDA(h, cudaMemsetAsync(hist, 0, NBINS * sizeof(uint32_t), s));  // pack binned some pairs
        fill_invalid_kernel<<<std::min<int64_t>((n_pairs + 255) / 256, 4096), 256, 0, s>>>(*out, 0, n_pairs);
        return fail(h, SW_ERR_INVALID_ARGUMENT, "offsets are not non-decreasing");
    }
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[2], s));

    // one kernel per route and pass (routes: TAG, S16, S32; sw_common.cuh)
    // linear gaps (gap_open == gap_extend) take the two-state kernels of the s16x2 routes
    const bool lin = sc.gap_open == sc.gap_extend && !(h->mode & SW_MODE_AFFINE_ONLY);
    const void* kfwd[N_ROUTES];
    const void* krev[N_ROUTES];
    wave_kernels(protein, lin, kfwd, krev);
    Launch lf[N_ROUTES], lr[N_ROUTES];
    plan_waves(h, sc, protein, hs, kfwd, krev, lf, lr);

    // stripe hand-off scratch: only if some query spans more than one stripe
    int64_t seg_bytes = 0;
    {
        const size_t need = scratch_bytes(lf, lr, hs, protein, seg_bytes);
        if (need) {
            size_t wmax = 0;
            for (int r = 0; r < N_ROUTES; ++r) wmax = std::max(wmax, (size_t)lr[r].blocks * lr[r].warps);
            ENS(progress[slot], 2 * wmax);
        }
        if (need && h->scratch[slot].cap < need) {
            ENS(scratch[slot], need);
            // defined contents: the first stripe of an item loads (and discards) its row
            SW_CUDA(h, cudaMemsetAsync(h->scratch[slot].p, 0, h->scratch[slot].cap, s));
        }
        // SW_MODE_POISON: hand-off rows a stripe reads but no earlier stripe of its item wrote come
        // out as H = F = 496 in every s16 half (0x01f001f0): above most scores yet inside the TAG
        // route's 511 range, so a stale read shows up as a wrong maximum instead of a wrapped
        // (negative, ignored) tagged value
        if ((h->mode & SW_MODE_POISON) && h->scratch[slot].p) {
            const size_t words = h->scratch[slot].cap / 4;
            fill_u32_kernel<<<(int)std::min<size_t>((words + 255) / 256, (size_t)h->sm_count * 8), 256, 0, s>>>(
                reinterpret_cast<uint32_t*>(h->scratch[slot].p), words, 0x01f001f0u);
            SW_CUDA(h, cudaGetLastError());
        }
    }

    // 5. forward binning (length-sorted, longest first)
    // counting sort when every key is in the small region (sw_bin.cuh): bounded by the extents
    const int min_rows = std::min(rows16, rows32);
    const bool small_fwd = hs.max_m < BIN_COLS && (hs.max_n + min_rows - 1) / min_rows <= BIN_MAX_STRIPES;
    const bool small_rev = small_fwd && (int64_t)sc.max_sigma * std::min(hs.max_n, hs.max_m) < BIN_COLS;
    if (!spec_bin || !small_fwd) {
        st = bin_order(h, h->order.p + lo, lo, hi, small_fwd, slot, s);
        if (st != SW_OK) return st;
    }
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[3], s));

    // 6. forward wavefront
    if (!spec_bin) SW_CUDA(h, cudaMemsetAsync(counters, 0, 8 * sizeof(int32_t), s));
    WaveParams W;
#if SW_CODE4
    if (!protein) {
        const size_t words = h->rcode.cap / 8;
        ENS(rcode4, words + 4);
        nibble_kernel<<<(int)std::min<size_t>((words + 255) / 256, (size_t)h->sm_count * 8), 256, 0, s>>>(h->rcode.p, h->rcode4.p, words);
        SW_CUDA(h, cudaGetLastError());
    }
#endif
    W.qpos = h->qpos.p; W.rpos = h->rpos.p; W.scratch = h->scratch[slot].p; W.scratch_seg_bytes = seg_bytes; W.sc = sc;
    W.rcode4 = h->rcode4.p; W.sixteen = 16;
    W.progress = h->progress[slot].p;
    W.tag_mul = protein ? 8 : 64;  // DNA TAG: H * 64 + 6 tag bits; protein (PT): H * 8 + 3 row bits
    W.one = 1;
    W.qcode = h->qcode.p; W.rcode = h->rcode.p; W.nlen = h->nlen.p; W.mlen = h->mlen.p; W.order = h->order.p + lo;
    W.target = nullptr; W.keys = h->keys_fwd.p; W.swept = &stats->swept_fwd; W.counts = stats->fwd_count;
    W.pre = nullptr;
    W.stats = stats;
    for (int r = 0; r < N_ROUTES; ++r) {
        if (lf[r].blocks <= 0) continue;
        W.route = r;
        W.item_counter = counters + r;
        void* args[] = {&W};
        SW_CUDA(h, cudaLaunchKernel(kfwd[r], dim3(lf[r].blocks), dim3(lf[r].warps * 32), args, (size_t)lf[r].smem, s));
        ++h->own_launches;
        SW_DBG(h, s, "launch at sw_api.cu:652");
    }
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[4], s));

    // 7. decode forward keys, prepare the reverse pass
    FinishParams F;
    F.lo = lo; F.hi = hi; F.flags = h->flags.p; F.keys_fwd = h->keys_fwd.p; F.keys_rev = h->keys_rev.p;
    F.rcode = h->rcode.p; F.rrev = h->rrev.p;
    F.qpos = h->qpos.p; F.rpos = h->rpos.p; F.nlen_rev = h->nlen_rev.p; F.mlen_rev = h->mlen_rev.p;
    F.target = h->target.p; F.key_rev = h->key.p; F.hist = hist; F.rows_s16 = rows16; F.rows_s32 = rows32;
    F.max_sigma = sc.max_sigma; F.gap_open = sc.gap_open; F.gap_extend = sc.gap_extend; F.pad_code = (uint8_t)(sc.nc - 1);
    // banded reverse pass (sw_band.cuh): a work item holds 16 / 32 pairs and sweeps ~2 n2 + 64 steps, so a
    // small batch (c1: 1,000 pairs) leaves most SMs idle on it -- the row sweep (4 pairs per item) is faster there
    const bool band_ok = !protein && s16_ok && K16 <= 16 && !(h->mode & SW_MODE_NO_BAND) &&
                         ((hi - lo) >= BAND_MIN_PAIRS || (h->mode & SW_MODE_BAND_ALWAYS));
    F.band_ok = band_ok ? 1 : 0; F.protein = protein ? 1 : 0; F.qcode = h->qcode.p; F.bslots = h->bslots.p;
    F.rrev_bytes = (int64_t)h->rrev.cap; F.band_bytes = (int64_t)h->bslots.cap;
    F.out = *out; F.stats = stats; F.end_only = end_only ? 1 : 0; F.rev_small = small_rev ? 1 : 0;
    {
        const int64_t warps = std::min<int64_t>((hi - lo + FIN_PPW - 1) / FIN_PPW, (int64_t)h->sm_count * 64);
        finish_fwd_kernel<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(F);
        SW_CUDA(h, cudaGetLastError());
        ++h->own_launches;
        SW_DBG(h, s, "launch at sw_api.cu:671");
    }
    if (end_only) {  // forward pass only (sw_set_mode)
        if (timing) {
            for (int k = 5; k < 8; ++k) SW_CUDA(h, cudaEventRecord(h->ev[k], s));
            h->ev_valid = true;
        }
        return SW_OK;
    }
    st = bin_order(h, h->order_rev.p + lo, lo, hi, small_rev, slot, s);
    if (st != SW_OK) return st;
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[5], s));

    // 8. reverse wavefront on the reversed prefixes (cooperative items' progress words start at 0)
    if (seg_bytes && h->progress[slot].p)
        SW_CUDA(h, cudaMemsetAsync(h->progress[slot].p, 0, h->progress[slot].cap * sizeof(unsigned long long), s));
    W.rcode = h->rrev.p; W.nlen = h->nlen_rev.p; W.mlen = h->mlen_rev.p; W.order = h->order_rev.p + lo;
    W.target = h->target.p; W.keys = h->keys_rev.p; W.swept = &stats->swept_rev; W.counts = stats->rev_count;
    W.pre = stats->rev_band;  // the band pairs lead the reverse order
    if (band_ok && hs.fwd_count[ROUTE_TAG] > 0) {
        BandParams B;
        B.slots = h->bslots.p; B.nlen = h->nlen_rev.p;
        B.mlen = h->mlen_rev.p; B.target = h->target.p; B.order = h->order_rev.p + lo; B.band_counts = stats->rev_band;
        B.keys = h->keys_rev.p; B.swept = &stats->swept_rev; B.sc = sc; B.stats = stats; B.tag_mul = 64;
        const void* kb[N_BAND] = {(const void*)band_rev_kernel<2>, (const void*)band_rev_kernel<4>};
        for (int b = 0; b < N_BAND; ++b) {
            const int slots = 64 / band_lanes(b);
            const int64_t items = (hs.fwd_count[ROUTE_TAG] + slots - 1) / slots;
            const int64_t maxb = (int64_t)h->sm_count * occupancy_blocks(kb[b], 128, 0);
            const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((items + 3) / 4, maxb));
            B.item_counter = counters + (b == 0 ? 3 : 7);
            void* args[] = {&B};
            SW_CUDA(h, cudaLaunchKernel(kb[b], dim3(blocks), dim3(128), args, 0, s));
            ++h->own_launches;
            SW_DBG(h, s, "launch at sw_api.cu:705");
        }
    }
    for (int r = 0; r < N_ROUTES; ++r) {
        if (lr[r].blocks <= 0) continue;
        W.route = r;
        W.item_counter = counters + 4 + r;
        void* args[] = {&W};
        SW_CUDA(h, cudaLaunchKernel(krev[r], dim3(lr[r].blocks), dim3(lr[r].warps * 32), args, (size_t)lr[r].smem, s));
        ++h->own_launches;
        SW_DBG(h, s, "launch at sw_api.cu:714");
    }
    if (timing) SW_CUDA(h, cudaEventRecord(h->ev[6], s));

    // 9. starts
    finish_rev_kernel<<<(int)std::min<int64_t>((hi - lo + 255) / 256, (int64_t)h->sm_count * 16), 256, 0, s>>>(F);
    SW_CUDA(h, cudaGetLastError());
    ++h->own_launches;
    SW_DBG(h, s, "launch at sw_api.cu:721");
    if (timing) {
        SW_CUDA(h, cudaEventRecord(h->ev[7], s));
        h->ev_valid = true;
    }
    return SW_OK;
#undef ENS
}

}  // namespace

extern "C" {

const char* sw_status_string(sw_status_t s) {
    switch (s) {
        case SW_OK: return "SW_OK";
        case SW_ERR_INVALID_ARGUMENT: return "SW_ERR_INVALID_ARGUMENT";
        case SW_ERR_INVALID_SCORING: return "SW_ERR_INVALID_SCORING";
        case SW_ERR_CUDA: return "SW_ERR_CUDA";
        case SW_ERR_OUT_OF_MEMORY: return "SW_ERR_OUT_OF_MEMORY";
        case SW_ERR_WRONG_DEVICE: return "SW_ERR_WRONG_DEVICE";
        case SW_ERR_BAD_PAIRS: return "SW_ERR_BAD_PAIRS";
        case SW_ERR_INTERNAL: return "SW_ERR_INTERNAL";
    }
    return "SW_ERR_UNKNOWN";
}

const char* sw_last_error_message(sw_handle_t h) { return h ? h->err.c_str() : "null handle"; }

sw_status_t sw_init(sw_handle_t* handle, int device) {
    if (!handle) return SW_ERR_INVALID_ARGUMENT;
    *handle = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) return SW_ERR_CUDA;
    if (device < 0 || device >= n) return SW_ERR_INVALID_ARGUMENT;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return SW_ERR_CUDA;
    if (cur != device) return SW_ERR_WRONG_DEVICE;
    sw_context* h = new (std::nothrow) sw_context();
    if (!h) return SW_ERR_OUT_OF_MEMORY;
    h->device = device;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) { delete h; return SW_ERR_CUDA; }
    h->sm_count = p.multiProcessorCount;
    // opt in to large dynamic shared memory (protein profiles)
    const int big = 200 * 1024;
    for (int pr = 0; pr < 2; ++pr)
        for (int r = 0; r < N_ROUTES; ++r) {
            set_smem_attr(wave_kernel_ptr<false, false>(pr, r), big);
            set_smem_attr(wave_kernel_ptr<true, false>(pr, r), big);
            set_smem_attr(wave_kernel_ptr<false, true>(pr, r), big);
            set_smem_attr(wave_kernel_ptr<true, true>(pr, r), big);
        }
    set_smem_attr(bin_scan_kernel, BIN_SCAN_SMEM);
    if (cudaMalloc(&h->d_stats, N_SLOTS * sizeof(BatchStats)) != cudaSuccess ||
        cudaMallocHost(&h->h_stats, N_SLOTS * sizeof(BatchStats)) != cudaSuccess ||
        cudaMallocHost(&h->h_ext, 4 * sizeof(int64_t)) != cudaSuccess ||
        cudaMalloc(&h->d_counters, N_SLOTS * 8 * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&h->d_sink, 1024 * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&h->d_hist, N_SLOTS * NBINS * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&h->d_binbase, N_SLOTS * NBINS * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&h->d_tb, 12 * sizeof(int32_t)) != cudaSuccess ||
        cudaMallocHost(&h->h_tb, 12 * sizeof(int32_t)) != cudaSuccess) {
        sw_free(h);
        return SW_ERR_OUT_OF_MEMORY;
    }
    cudaMemset(h->d_stats, 0, N_SLOTS * sizeof(BatchStats));
    cudaMemset(h->d_hist, 0, N_SLOTS * NBINS * sizeof(uint32_t));
    for (auto& ev : h->ev) {
        if (cudaEventCreate(&ev) != cudaSuccess) { sw_free(h); return SW_ERR_CUDA; }
    }
    if (cudaEventCreateWithFlags(&h->ev_prep, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->as_start, cudaEventDisableTiming) != cudaSuccess) { sw_free(h); return SW_ERR_CUDA; }
    for (int k = 0; k < 2; ++k)
        if (cudaEventCreateWithFlags(&h->as_in[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->as_comp[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->as_done[k], cudaEventDisableTiming) != cudaSuccess) { sw_free(h); return SW_ERR_CUDA; }
    for (int k = 0; k < MAX_CHUNKS; ++k) {
        if (cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_out[k], cudaEventDisableTiming) != cudaSuccess) { sw_free(h); return SW_ERR_CUDA; }
    }
    if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->out_stream, cudaStreamNonBlocking) != cudaSuccess) { sw_free(h); return SW_ERR_CUDA; }
    *handle = h;
    return SW_OK;
}

sw_status_t sw_align_batch(sw_handle_t h, const uint8_t* queries, const int64_t* q_offsets, const uint8_t* refs,
                           const int64_t* r_offsets, int64_t n_pairs, const sw_scoring_t* scoring,
                           const sw_result_t* out, void* stream) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    return align_impl(h, queries, q_offsets, refs, r_offsets, n_pairs, scoring, out, (cudaStream_t)stream, nullptr);
}

sw_status_t sw_reserve(sw_handle_t h, int64_t max_pairs, int64_t max_query_bytes, int64_t max_ref_bytes,
                       int32_t max_query_len, int32_t max_ref_len) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (max_pairs < 1 || max_pairs > 0x7ffffff0LL || max_query_bytes < 0 || max_ref_bytes < 0 || max_query_len < 0 ||
        max_ref_len < 0 || max_query_len > SW_MAX_SEQ_LEN || max_ref_len > SW_MAX_SEQ_LEN)
        return fail(h, SW_ERR_INVALID_ARGUMENT, "sw_reserve: bounds out of range");
    int dev = -1;
    SW_CUDA(h, cudaGetDevice(&dev));
    if (dev != h->device) return fail(h, SW_ERR_WRONG_DEVICE, "current device differs from the handle's device");
    SW_CUDA(h, cudaDeviceSynchronize());  // buffers may move: nothing of the handle may be in flight
    h->reserved = false;
    const size_t N = (size_t)max_pairs;
    sw_status_t st = prepare_workspace(h, N, (size_t)max_query_bytes, (size_t)max_ref_bytes, h->codes_alphabet < 0 ? 0 : h->codes_alphabet, 0);
    if (st != SW_OK) return st;
    // radix-sort temporary storage (reserved calls whose keys may leave the counting sort's region)
    {
        size_t tb = 0;
        SW_CUDA(h, cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, h->key.p, h->key_sorted.p, h->iota.p,
                                                             h->order.p, (int)max_pairs, 0, 32, (cudaStream_t)0));
        st = ensure(h, h->cub_temp[0], tb);
        if (st != SW_OK) return st;
    }
    // stripe hand-off scratch for the largest grid of any alphabet / gap model / route
    BatchStats hs;
    std::memset(&hs, 0, sizeof(hs));
    hs.max_n = max_query_len;
    hs.max_m = max_ref_len;
    for (int r = 0; r < N_ROUTES; ++r) hs.fwd_count[r] = (int32_t)max_pairs;
    size_t need = 0;
    for (int pr = 0; pr < 2; ++pr)
        for (int lin = 0; lin < 2; ++lin) {
            Scoring sc;
            std::memset(&sc, 0, sizeof(sc));
            sc.alphabet = pr ? SW_ALPHABET_PROTEIN : SW_ALPHABET_DNA;
            sc.nc = pr ? NC_PROTEIN : NC_DNA;
            sc.max_sigma = 32767;
            const void* kf[N_ROUTES];
            const void* kr[N_ROUTES];
            wave_kernels(pr != 0, lin != 0, kf, kr);
            Launch lf[N_ROUTES], lr[N_ROUTES];
            plan_waves(h, sc, pr != 0, hs, kf, kr, lf, lr);
            int64_t seg = 0;
            need = std::max(need, scratch_bytes(lf, lr, hs, pr != 0, seg));
        }
    if (need) {
        st = ensure(h, h->scratch[0], need);
        if (st != SW_OK) return st;
        SW_CUDA(h, cudaMemset(h->scratch[0].p, 0, h->scratch[0].cap));
        st = ensure(h, h->progress[0], (size_t)h->sm_count * 64 * 2);  // every resident warp, two rows
        if (st != SW_OK) return st;
    }
    SW_CUDA(h, cudaDeviceSynchronize());
    h->res_pairs = max_pairs; h->res_qbytes = max_query_bytes; h->res_rbytes = max_ref_bytes;
    h->res_n = max_query_len; h->res_m = max_ref_len;
    h->reserved = true;
    return SW_OK;
}

namespace {
// sw_align_query_db: q[p * n + i] = query[i], qo[p] = p * n (16-byte stores when n is a multiple of 16)
__global__ void broadcast_query_kernel(const uint8_t* __restrict__ query, int64_t n, int64_t n_refs,
                                       uint8_t* __restrict__ q, int64_t* __restrict__ qo) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t p = tid; p <= n_refs; p += stride) qo[p] = p * n;
    if ((n & 15) == 0 && (((uintptr_t)query) & 15) == 0) {
        const int64_t nv = n >> 4, total = nv * n_refs;
        for (int64_t k = tid; k < total; k += stride)
            reinterpret_cast<uint4*>(q)[k] = __ldg(reinterpret_cast<const uint4*>(query) + k % nv);
    } else {
        const int64_t total = n * n_refs;
        for (int64_t k = tid; k < total; k += stride) q[k] = query[k % n];
    }
}
}  // namespace

sw_status_t sw_align_query_db(sw_handle_t h, const uint8_t* query, int64_t n, const uint8_t* refs,
                              const int64_t* r_offsets, int64_t n_refs, const sw_scoring_t* scoring,
                              const sw_result_t* out, void* stream) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (n < 0 || (n > 0 && !query)) return fail(h, SW_ERR_INVALID_ARGUMENT, "query: n < 0 or NULL pointer");
    if (n_refs < 0) return fail(h, SW_ERR_INVALID_ARGUMENT, "n_refs < 0");
    if (n_refs == 0) return SW_OK;
    int dev = -1;
    SW_CUDA(h, cudaGetDevice(&dev));
    if (dev != h->device) return fail(h, SW_ERR_WRONG_DEVICE, "current device differs from the handle's device");
    cudaStream_t s = (cudaStream_t)stream;
    sw_status_t st = ensure(h, h->db_q, (size_t)std::max<int64_t>(n * n_refs, 16));
    if (st != SW_OK) return st;
    st = ensure(h, h->db_qo, (size_t)n_refs + 1);
    if (st != SW_OK) return st;
    const int64_t work = std::max<int64_t>(n_refs + 1, n * n_refs / 16);
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)h->sm_count * 8);
    broadcast_query_kernel<<<blocks, 256, 0, s>>>(query, n, n_refs, h->db_q.p, h->db_qo.p);
    SW_CUDA(h, cudaGetLastError());
    return align_impl(h, h->db_q.p, h->db_qo.p, refs, r_offsets, n_refs, scoring, out, s, nullptr);
}

sw_status_t sw_align_batch_host(sw_handle_t h, const uint8_t* queries, const int64_t* q_offsets, const uint8_t* refs,
                                const int64_t* r_offsets, int64_t n_pairs, const sw_scoring_t* scoring,
                                const sw_result_t* out_host, void* stream) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (n_pairs < 0) return fail(h, SW_ERR_INVALID_ARGUMENT, "n_pairs < 0");
    if (n_pairs == 0) return SW_OK;
    if (!queries || !q_offsets || !refs || !r_offsets || !out_host)
        return fail(h, SW_ERR_INVALID_ARGUMENT, "NULL pointer argument");
    Scoring sc;
    bool s16_ok = false;
    sw_status_t st = check_scoring(h, scoring, sc, s16_ok);
    if (st != SW_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t N = (size_t)n_pairs;
    int32_t* dst[5] = {out_host->score, out_host->q_end, out_host->r_end, out_host->q_start, out_host->r_start};
    // host-side validation: offsets must be non-decreasing (reading R15)
    for (int64_t p = 0; p < n_pairs; ++p) {
        if (q_offsets[p + 1] < q_offsets[p] || r_offsets[p + 1] < r_offsets[p]) {
            for (int k = 0; k < 5; ++k)
                if (dst[k]) for (size_t i = 0; i < N; ++i) dst[k][i] = -1;
            return fail(h, SW_ERR_INVALID_ARGUMENT, "offsets are not non-decreasing");
        }
    }
    const int64_t q0 = q_offsets[0], qN = q_offsets[n_pairs], r0 = r_offsets[0], rN = r_offsets[n_pairs];
    const size_t tq = (size_t)(qN - q0), tr = (size_t)(rN - r0);
#define ENS(buf, n) do { sw_status_t _s = ensure(h, h->buf, (n)); if (_s != SW_OK) return _s; } while (0)
    ENS(st_q, tq + 1); ENS(st_r, tr + 1); ENS(st_qo, N + 1); ENS(st_ro, N + 1); ENS(st_out, 5 * N);
#undef ENS
    // Chunks of about equal cell count; chunk k+1's host-to-device copy (copy stream) overlaps
    // chunk k's kernels (caller's stream), and chunk k's results return while k+1 computes.
    const bool tag_ok = tag_max_score(sc.alphabet) > 0 && (K16 <= 16 || sc.alphabet == SW_ALPHABET_PROTEIN);
    double total_cells = 0;
    for (int64_t p = 0; p < n_pairs; ++p)
        total_cells += (double)(q_offsets[p + 1] - q_offsets[p]) * (double)(r_offsets[p + 1] - r_offsets[p]);
    int want = 4;
    if (const char* e = std::getenv("SW_HOST_CHUNKS")) want = std::max(1, std::min(MAX_CHUNKS, std::atoi(e)));  // experiments
    const int n_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(want, n_pairs / 16384));
    int64_t cut[MAX_CHUNKS + 1];
    cut[0] = 0;
    {
        double acc = 0;
        int k = 1;
        for (int64_t p = 0; p < n_pairs && k < n_chunks; ++p) {
            acc += (double)(q_offsets[p + 1] - q_offsets[p]) * (double)(r_offsets[p + 1] - r_offsets[p]);
            if (acc >= total_cells * k / n_chunks) cut[k++] = p + 1;
        }
        while (k <= n_chunks) cut[k++] = n_pairs;
    }
    // all input copies first (offsets whole, payload per chunk)
    SW_CUDA(h, cudaMemcpyAsync(h->st_qo.p, q_offsets, (N + 1) * 8, cudaMemcpyHostToDevice, h->copy_stream));
    SW_CUDA(h, cudaMemcpyAsync(h->st_ro.p, r_offsets, (N + 1) * 8, cudaMemcpyHostToDevice, h->copy_stream));
    for (int k = 0; k < n_chunks; ++k) {
        const int64_t a = cut[k], b = cut[k + 1];
        const int64_t qa = q_offsets[a], qb = q_offsets[b], ra = r_offsets[a], rb = r_offsets[b];
        if (qb > qa) SW_CUDA(h, cudaMemcpyAsync(h->st_q.p + (qa - q0), queries + qa, (size_t)(qb - qa), cudaMemcpyHostToDevice, h->copy_stream));
        if (rb > ra) SW_CUDA(h, cudaMemcpyAsync(h->st_r.p + (ra - r0), refs + ra, (size_t)(rb - ra), cudaMemcpyHostToDevice, h->copy_stream));
        SW_CUDA(h, cudaEventRecord(h->ev_in[k], h->copy_stream));
    }
    // the whole batch's workspace first, then chunk k runs on slot k & 1 (caller's stream /
    // the auxiliary stream), waiting only for its own payload
    st = prepare_workspace(h, N, (size_t)(qN - q0), (size_t)(rN - r0), sc.alphabet, s);
    if (st != SW_OK) return st;
    SW_CUDA(h, cudaEventRecord(h->ev_prep, s));
    SW_CUDA(h, cudaStreamWaitEvent(h->aux_stream, h->ev_prep, 0));
    sw_result_t dout;
    dout.score = h->st_out.p; dout.q_end = h->st_out.p + N; dout.r_end = h->st_out.p + 2 * N;
    dout.q_start = h->st_out.p + 3 * N; dout.r_start = h->st_out.p + 4 * N;
    sw_status_t result = SW_OK;
    for (int k = 0; k < n_chunks; ++k) {
        const int64_t a = cut[k], b = cut[k + 1];
        if (b <= a) continue;
        HostPlan hp;
        hp.ext[0] = q0; hp.ext[1] = qN; hp.ext[2] = r0; hp.ext[3] = rN;
        hp.lo = a; hp.hi = b;
        hp.slot = k & 1;
        hp.reset_cumulative = k < N_SLOTS;
        hp.max_n = 0; hp.max_m = 0;
        for (int r = 0; r < N_ROUTES; ++r) hp.route_upper[r] = 0;
        for (int64_t p = a; p < b; ++p) {
            const int64_t n = q_offsets[p + 1] - q_offsets[p], m = r_offsets[p + 1] - r_offsets[p];
            if (n > SW_MAX_SEQ_LEN || m > SW_MAX_SEQ_LEN) continue;  // invalid pair
            hp.max_n = std::max<int32_t>(hp.max_n, (int32_t)n);
            hp.max_m = std::max<int32_t>(hp.max_m, (int32_t)m);
            if (n == 0 || m == 0) continue;
            const int64_t smax = (int64_t)sc.max_sigma * std::min(n, m);
            const int route = (s16_ok && tag_ok && (int64_t)sc.max_sigma * n <= tag_max_score(sc.alphabet)) ? ROUTE_TAG
                            : (s16_ok && smax <= S16_MAX_SCORE) ? ROUTE_S16 : ROUTE_S32;
            ++hp.route_upper[route];
        }
        cudaStream_t cs = hp.slot ? h->aux_stream : s;
        SW_CUDA(h, cudaStreamWaitEvent(cs, h->ev_in[k], 0));
        st = align_impl(h, h->st_q.p - q0, h->st_qo.p, h->st_r.p - r0, h->st_ro.p, n_pairs, scoring, &dout, cs,
                        nullptr, &hp);  // launch counters accumulate over the chunks
        if (st != SW_OK) { result = st; break; }
        SW_CUDA(h, cudaEventRecord(h->ev_out[k], cs));
        SW_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_out[k], 0));
        for (int f = 0; f < ((h->mode & SW_MODE_END_ONLY) ? 3 : 5); ++f)
            if (dst[f]) SW_CUDA(h, cudaMemcpyAsync(dst[f] + a, h->st_out.p + f * N + a, (size_t)(b - a) * 4,
                                                   cudaMemcpyDeviceToHost, h->copy_stream));
    }
    SW_CUDA(h, cudaStreamSynchronize(h->copy_stream));
    SW_CUDA(h, cudaStreamSynchronize(h->aux_stream));
    SW_CUDA(h, cudaStreamSynchronize(s));
    h->last_stream = s;
    return result;
}

sw_status_t sw_traceback(sw_handle_t h, const uint8_t* queries, const int64_t* q_offsets, const uint8_t* refs,
                         const int64_t* r_offsets, int64_t n_pairs, const sw_scoring_t* scoring, const sw_result_t* res,
                         uint8_t* ops, int32_t* n_ops, void* stream) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (n_pairs < 0) return fail(h, SW_ERR_INVALID_ARGUMENT, "n_pairs < 0");
    if (n_pairs == 0) return SW_OK;
    if (!queries || !q_offsets || !refs || !r_offsets || !res || !res->score || !res->q_end || !res->r_end ||
        !res->q_start || !res->r_start || !ops || !n_ops)
        return fail(h, SW_ERR_INVALID_ARGUMENT, "NULL pointer argument");
    int dev = -1;
    SW_CUDA(h, cudaGetDevice(&dev));
    if (dev != h->device) return fail(h, SW_ERR_WRONG_DEVICE, "current device differs from the handle's device");
    Scoring sc;
    bool s16_ok = false;
    sw_status_t st = check_scoring(h, scoring, sc, s16_ok);
    if (st != SW_OK) return st;
    if (h->mode & SW_MODE_END_ONLY)
        return fail(h, SW_ERR_INVALID_ARGUMENT, "sw_traceback needs start positions: the handle is in SW_MODE_END_ONLY");
    cudaStream_t s = (cudaStream_t)stream;
    // 1. the batch's largest interval (sizes the per-warp scratch) and the offset bases
    SW_CUDA(h, cudaMemsetAsync(h->d_tb, 0, 12 * sizeof(int32_t), s));
    if (h->mode & SW_MODE_POISON) {
        SW_CUDA(h, cudaMemsetAsync(n_ops, 0x7f, (size_t)n_pairs * 4, s));
        if (h->tb_dir.p) SW_CUDA(h, cudaMemsetAsync(h->tb_dir.p, 0x7f, h->tb_dir.cap * 4, s));
        if (h->tb_bnd.p) SW_CUDA(h, cudaMemsetAsync(h->tb_bnd.p, 0x7f, h->tb_bnd.cap * 8, s));
    }
    int64_t* base = reinterpret_cast<int64_t*>(h->d_tb + 4);
    trace_extent_kernel<<<(int)std::min<int64_t>((n_pairs + 255) / 256, (int64_t)h->sm_count * 8), 256, 0, s>>>(
        *res, n_pairs, q_offsets, r_offsets, h->d_tb, base);
    SW_CUDA(h, cudaGetLastError());
    SW_CUDA(h, cudaMemcpyAsync(h->h_tb, h->d_tb, 12 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SW_CUDA(h, cudaStreamSynchronize(s));
    const int32_t max_a = h->h_tb[0], max_b = h->h_tb[1], bad_intervals = h->h_tb[9];
    const int64_t q0 = reinterpret_cast<int64_t*>(h->h_tb + 4)[0], r0 = reinterpret_cast<int64_t*>(h->h_tb + 4)[1];
    // 2. one warp per pair; the warp count is capped so the direction scratch stays <= 4 GiB
    const int64_t ns = std::max<int64_t>(1, ((int64_t)max_a + TB_ROWS - 1) / TB_ROWS);
    const int64_t dir_words = ns * (((int64_t)max_b + 31 + 31) & ~(int64_t)31) * 32;
    const int64_t bnd_len = (int64_t)max_b + 1;
    const int64_t budget_words = ((int64_t)4 << 30) / 4;
    // DNA batches: the s16x2 kernel (two pairs per warp, two direction regions per warp) takes the
    // pairs tb16_ok() admits, then the int32 kernel the rest
    const bool use16 = sc.alphabet == SW_ALPHABET_DNA && !(h->mode & SW_MODE_TB_INT32);
    int64_t warps = std::min<int64_t>((int64_t)h->sm_count * 4 * occupancy_blocks((const void*)traceback_kernel, 128, 0),
                                      std::max<int64_t>(4, budget_words / std::max<int64_t>((use16 ? 2 : 1) * dir_words, 1)));
    warps = std::min<int64_t>(warps, std::max<int64_t>(4, n_pairs));
    warps = (warps + 3) / 4 * 4;
    {
        sw_status_t e = ensure(h, h->tb_dir, (size_t)(warps * dir_words * (use16 ? 2 : 1)));
        if (e != SW_OK) return e;
        e = ensure(h, h->tb_bnd, (size_t)(warps * bnd_len));
        if (e != SW_OK) return e;
    }
    TraceParams T;
    T.queries = queries; T.q_off = q_offsets; T.refs = refs; T.r_off = r_offsets; T.n_pairs = n_pairs;
    T.q0 = q0; T.r0 = r0; T.res = *res; T.ops = ops; T.n_ops = n_ops; T.sc = sc;
    T.dir = h->tb_dir.p; T.dir_words = dir_words; T.bnd = h->tb_bnd.p; T.bnd_len = bnd_len;
    T.counter = h->d_tb + 2; T.err = h->d_tb + 3; T.counter16 = h->d_tb + 8; T.skip16 = use16 ? 1 : 0;
    if (use16) {
        traceback16_kernel<<<(int)(warps / 4), 128, 0, s>>>(T);
        SW_CUDA(h, cudaGetLastError());
    }
    traceback_kernel<<<(int)(warps / 4), 128, 0, s>>>(T);
    SW_CUDA(h, cudaGetLastError());
    h->last_stream = s;
    h->have_last = true;
    h->tb_pending = true;  // the kernels' internal-error count is read by sw_batch_status
    if (bad_intervals)
        return fail(h, SW_ERR_INVALID_ARGUMENT, std::to_string(bad_intervals) +
                    " pair(s) with score > 0 have an interval outside their sequences (n_ops = -1)");
    return SW_OK;
}

sw_status_t sw_set_mode(sw_handle_t h, int32_t mode) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (mode & ~(SW_MODE_END_ONLY | SW_MODE_AFFINE_ONLY | SW_MODE_TB_INT32 | SW_MODE_POISON | SW_MODE_NO_BAND | SW_MODE_BAND_ALWAYS))
        return fail(h, SW_ERR_INVALID_ARGUMENT, "unknown mode");
    h->mode = mode;
    return SW_OK;
}

sw_status_t sw_submit_host(sw_handle_t h, const uint8_t* queries, const int64_t* q_offsets, const uint8_t* refs,
                           const int64_t* r_offsets, int64_t n_pairs, const sw_scoring_t* scoring,
                           const sw_result_t* out_host, void* stream) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (n_pairs < 0) return fail(h, SW_ERR_INVALID_ARGUMENT, "n_pairs < 0");
    if (n_pairs == 0) return SW_OK;
    if (!queries || !q_offsets || !refs || !r_offsets || !out_host)
        return fail(h, SW_ERR_INVALID_ARGUMENT, "NULL pointer argument");
    Scoring sc;
    bool s16_ok = false;
    sw_status_t st = check_scoring(h, scoring, sc, s16_ok);
    if (st != SW_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t N = (size_t)n_pairs;
    // host-side validation and the plan (reading R15): no device round trip in the pipeline
    HostPlan hp;
    hp.lo = 0; hp.hi = n_pairs; hp.slot = 0; hp.reset_cumulative = true;
    hp.max_n = 0; hp.max_m = 0;
    for (int r = 0; r < N_ROUTES; ++r) hp.route_upper[r] = 0;
    const bool tag_ok = tag_max_score(sc.alphabet) > 0 && (K16 <= 16 || sc.alphabet == SW_ALPHABET_PROTEIN);
    for (int64_t p = 0; p < n_pairs; ++p) {
        const int64_t n = q_offsets[p + 1] - q_offsets[p], m = r_offsets[p + 1] - r_offsets[p];
        if (n < 0 || m < 0) return fail(h, SW_ERR_INVALID_ARGUMENT, "offsets are not non-decreasing");
        if (n > SW_MAX_SEQ_LEN || m > SW_MAX_SEQ_LEN) continue;  // invalid pair
        hp.max_n = std::max<int32_t>(hp.max_n, (int32_t)n);
        hp.max_m = std::max<int32_t>(hp.max_m, (int32_t)m);
        if (n == 0 || m == 0) continue;
        const int64_t smax = (int64_t)sc.max_sigma * std::min(n, m);
        const int route = (s16_ok && tag_ok && (int64_t)sc.max_sigma * n <= tag_max_score(sc.alphabet)) ? ROUTE_TAG
                        : (s16_ok && smax <= S16_MAX_SCORE) ? ROUTE_S16 : ROUTE_S32;
        ++hp.route_upper[route];
    }
    const int64_t q0 = q_offsets[0], qN = q_offsets[n_pairs], r0 = r_offsets[0], rN = r_offsets[n_pairs];
    hp.ext[0] = q0; hp.ext[1] = qN; hp.ext[2] = r0; hp.ext[3] = rN;
    const int k = h->as_next;
    h->as_next ^= 1;
    // staging slot k: its previous batch must be fully out before it is reused or resized
    if (h->as_used[k]) {
        const bool grow = h->as_q[k].cap < (size_t)(qN - q0) + 1 || h->as_r[k].cap < (size_t)(rN - r0) + 1 ||
                          h->as_qo[k].cap < N + 1 || h->as_out[k].cap < 5 * N;
        if (grow) SW_CUDA(h, cudaEventSynchronize(h->as_done[k]));
    }
#define ENS(buf, n) do { sw_status_t _s = ensure(h, h->buf, (n)); if (_s != SW_OK) return _s; } while (0)
    ENS(as_q[k], (size_t)(qN - q0) + 1); ENS(as_r[k], (size_t)(rN - r0) + 1);
    ENS(as_qo[k], N + 1); ENS(as_ro[k], N + 1); ENS(as_out[k], 5 * N);
#undef ENS
    // copy-in: the first batch of a pipeline starts after earlier work on the caller's stream
    // (so events recorded there bracket the whole pipeline); later batches start at once (the
    // previous batch is still aligning: that is the overlap).  A staging slot is reused only
    // after its last copy-out.
    if (!h->as_inflight) {
        SW_CUDA(h, cudaEventRecord(h->as_start, s));
        SW_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->as_start, 0));
    }
    if (h->as_used[k]) SW_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->as_done[k], 0));
    SW_CUDA(h, cudaMemcpyAsync(h->as_qo[k].p, q_offsets, (N + 1) * 8, cudaMemcpyHostToDevice, h->copy_stream));
    SW_CUDA(h, cudaMemcpyAsync(h->as_ro[k].p, r_offsets, (N + 1) * 8, cudaMemcpyHostToDevice, h->copy_stream));
    if (qN > q0) SW_CUDA(h, cudaMemcpyAsync(h->as_q[k].p, queries + q0, (size_t)(qN - q0), cudaMemcpyHostToDevice, h->copy_stream));
    if (rN > r0) SW_CUDA(h, cudaMemcpyAsync(h->as_r[k].p, refs + r0, (size_t)(rN - r0), cudaMemcpyHostToDevice, h->copy_stream));
    SW_CUDA(h, cudaEventRecord(h->as_in[k], h->copy_stream));
    // align on the caller's stream once the inputs are in (batches in submission order)
    st = prepare_workspace(h, N, (size_t)(qN - q0), (size_t)(rN - r0), sc.alphabet, s);
    if (st != SW_OK) return st;
    SW_CUDA(h, cudaStreamWaitEvent(s, h->as_in[k], 0));
    sw_result_t dout;
    int32_t* o = h->as_out[k].p;
    dout.score = o; dout.q_end = o + N; dout.r_end = o + 2 * N; dout.q_start = o + 3 * N; dout.r_start = o + 4 * N;
    st = align_impl(h, h->as_q[k].p - q0, h->as_qo[k].p, h->as_r[k].p - r0, h->as_ro[k].p, n_pairs, scoring, &dout, s,
                    nullptr, &hp);
    if (st != SW_OK) return st;
    SW_CUDA(h, cudaEventRecord(h->as_comp[k], s));
    // results out on their own stream (the copy-in stream keeps feeding the next batch)
    SW_CUDA(h, cudaStreamWaitEvent(h->out_stream, h->as_comp[k], 0));
    int32_t* dst[5] = {out_host->score, out_host->q_end, out_host->r_end, out_host->q_start, out_host->r_start};
    for (int f = 0; f < ((h->mode & SW_MODE_END_ONLY) ? 3 : 5); ++f)
        if (dst[f]) SW_CUDA(h, cudaMemcpyAsync(dst[f], o + f * N, N * 4, cudaMemcpyDeviceToHost, h->out_stream));
    SW_CUDA(h, cudaEventRecord(h->as_done[k], h->out_stream));
    h->as_used[k] = true;
    h->as_inflight = true;
    h->as_stream = s;
    h->last_stream = s;
    return SW_OK;
}

sw_status_t sw_wait(sw_handle_t h) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    for (int k = 0; k < 2; ++k)
        if (h->as_used[k]) {
            SW_CUDA(h, cudaEventSynchronize(h->as_done[k]));
            if (h->as_stream) SW_CUDA(h, cudaStreamWaitEvent(h->as_stream, h->as_done[k], 0));
        }
    h->as_inflight = false;
    return SW_OK;
}

sw_status_t sw_batch_status(sw_handle_t h, int64_t* n_bad_pairs) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (n_bad_pairs) *n_bad_pairs = 0;
    if (!h->have_last) return SW_OK;
    SW_CUDA(h, cudaStreamSynchronize(h->last_stream));
    BatchStats t;
    SW_CUDA(h, read_stats(h, t));
    if (n_bad_pairs) *n_bad_pairs = t.n_bad;
    if (t.internal_err) return fail(h, SW_ERR_INTERNAL, "reverse-pass self-check failed");
    if (t.rejected) {
        if (n_bad_pairs) *n_bad_pairs = -1;
        return fail(h, SW_ERR_INVALID_ARGUMENT, "the batch exceeds the handle's reservation (sw_reserve): every output is -1");
    }
    if (h->tb_pending) {
        int32_t tb_err = 0;
        SW_CUDA(h, cudaMemcpy(&tb_err, h->d_tb + 3, sizeof(int32_t), cudaMemcpyDeviceToHost));
        h->tb_pending = false;
        if (tb_err) return fail(h, SW_ERR_INTERNAL, std::to_string(tb_err) + " alignment path(s) failed (walk or scratch)");
    }
    if (t.malformed) {
        if (n_bad_pairs) *n_bad_pairs = -1;
        return SW_ERR_BAD_PAIRS;
    }
    return t.n_bad ? SW_ERR_BAD_PAIRS : SW_OK;
}

sw_status_t sw_free(sw_handle_t h) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (h->have_last) cudaStreamSynchronize(h->last_stream);
    cudaDeviceSynchronize();
    release(h->nlen); release(h->mlen); release(h->nlen_rev); release(h->mlen_rev); release(h->target);
    release(h->iota); release(h->order); release(h->order_rev); release(h->qpos); release(h->rpos); release(h->flags);
    release(h->key); release(h->key_sorted);
    for (int k = 0; k < N_SLOTS; ++k) { release(h->cub_temp[k]); release(h->scratch[k]); release(h->progress[k]); } release(h->keys_fwd); release(h->keys_rev);
    release(h->qcode); release(h->rcode); release(h->rrev); release(h->bslots);
    release(h->st_q); release(h->st_r); release(h->st_qo); release(h->st_ro); release(h->st_out);
    release(h->db_q); release(h->db_qo);
    if (h->d_stats) cudaFree(h->d_stats);
    if (h->h_stats) cudaFreeHost(h->h_stats);
    if (h->h_ext) cudaFreeHost(h->h_ext);
    if (h->d_counters) cudaFree(h->d_counters);
    if (h->d_sink) cudaFree(h->d_sink);
    if (h->d_hist) cudaFree(h->d_hist);
    if (h->d_tb) cudaFree(h->d_tb);
    if (h->h_tb) cudaFreeHost(h->h_tb);
    release(h->tb_dir); release(h->tb_bnd);
    if (h->d_binbase) cudaFree(h->d_binbase);
    for (auto& ev : h->ev) if (ev) cudaEventDestroy(ev);
    for (int k = 0; k < MAX_CHUNKS; ++k) {
        if (h->ev_in[k]) cudaEventDestroy(h->ev_in[k]);
        if (h->ev_out[k]) cudaEventDestroy(h->ev_out[k]);
    }
    if (h->ev_prep) cudaEventDestroy(h->ev_prep);
    if (h->as_start) cudaEventDestroy(h->as_start);
    for (int k = 0; k < 2; ++k) {
        if (h->as_in[k]) cudaEventDestroy(h->as_in[k]);
        if (h->as_comp[k]) cudaEventDestroy(h->as_comp[k]);
        if (h->as_done[k]) cudaEventDestroy(h->as_done[k]);
        release(h->as_q[k]); release(h->as_r[k]); release(h->as_qo[k]); release(h->as_ro[k]); release(h->as_out[k]);
    }
    if (h->out_stream) cudaStreamDestroy(h->out_stream);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->aux_stream) cudaStreamDestroy(h->aux_stream);
    delete h;
    return SW_OK;
}

sw_status_t sw_plan_shards(const int64_t* q_off, const int64_t* r_off, int64_t n_pairs, int32_t n_shards,
                           int64_t* shard_begin) {
    if (!q_off || !r_off || !shard_begin || n_pairs < 0 || n_shards < 1) return SW_ERR_INVALID_ARGUMENT;
    std::vector<double> pre((size_t)n_pairs + 1, 0.0);
    for (int64_t p = 0; p < n_pairs; ++p) {
        const int64_t n = q_off[p + 1] - q_off[p], m = r_off[p + 1] - r_off[p];
        const double c = (n > 0 && m > 0) ? (double)n * (double)m : 1.0;
        pre[(size_t)p + 1] = pre[(size_t)p] + c;
    }
    const double total = pre[(size_t)n_pairs];
    shard_begin[0] = 0;
    int64_t p = 0;
    for (int32_t k = 1; k < n_shards; ++k) {
        const double goal = total * k / n_shards;
        while (p < n_pairs && pre[(size_t)p + 1] <= goal) ++p;
        // choose the cut (p or p+1) whose prefix is closer to the goal
        int64_t cut = p;
        if (p < n_pairs && (pre[(size_t)p + 1] - goal) < (goal - pre[(size_t)p])) cut = p + 1;
        cut = std::max(cut, shard_begin[k - 1]);
        shard_begin[k] = std::min(cut, n_pairs);
    }
    shard_begin[n_shards] = n_pairs;
    return SW_OK;
}

sw_status_t sw_enable_stage_timing(sw_handle_t h, int enable) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    h->timing = enable != 0;
    return SW_OK;
}

sw_status_t sw_get_stage_ms(sw_handle_t h, float ms[SW_STAGE_COUNT]) {
    if (!h || !ms) return SW_ERR_INVALID_ARGUMENT;
    for (int k = 0; k < SW_STAGE_COUNT; ++k) ms[k] = 0.f;
    if (!h->ev_valid) return fail(h, SW_ERR_INVALID_ARGUMENT, "no timed batch");
    SW_CUDA(h, cudaEventSynchronize(h->ev[7]));
    // stage k spans events: pack 0-1, sort 2-3, fwd 3-4, mid 4-5, rev 5-6, finish 6-7
    const int a[SW_STAGE_COUNT] = {0, 2, 3, 4, 5, 6};
    const int b[SW_STAGE_COUNT] = {1, 3, 4, 5, 6, 7};
    for (int k = 0; k < SW_STAGE_COUNT; ++k) SW_CUDA(h, cudaEventElapsedTime(&ms[k], h->ev[a[k]], h->ev[b[k]]));
    return SW_OK;
}

sw_status_t sw_last_launch_count(sw_handle_t h, int32_t* own, int32_t* lib) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (own) *own = h->own_launches;
    if (lib) *lib = h->lib_launches;
    return SW_OK;
}

sw_status_t sw_last_cell_counts(sw_handle_t h, int64_t* fwd, int64_t* swept) {
    if (!h) return SW_ERR_INVALID_ARGUMENT;
    if (h->have_last) SW_CUDA(h, cudaStreamSynchronize(h->last_stream));
    BatchStats t;
    SW_CUDA(h, read_stats(h, t));
    if (fwd) *fwd = (int64_t)t.cells;
    if (swept) *swept = (int64_t)t.swept_fwd;
    return SW_OK;
}

sw_status_t sw_last_reverse_cells(sw_handle_t h, int64_t* swept) {
    if (!h || !swept) return SW_ERR_INVALID_ARGUMENT;
    if (h->have_last) SW_CUDA(h, cudaStreamSynchronize(h->last_stream));
    BatchStats t;
    SW_CUDA(h, read_stats(h, t));
    *swept = (int64_t)t.swept_rev;
    return SW_OK;
}

#if SW_TRACE_ITEMS
// development builds only: copy the per-item trace out (and reset it); returns the entry count
int64_t sw_debug_item_trace(unsigned long long* host, int64_t max_entries) {
    unsigned n = 0;
    if (cudaMemcpyFromSymbol(&n, swb::g_trace_n, sizeof(n)) != cudaSuccess) return -1;
    const int64_t k = std::min<int64_t>(std::min<int64_t>(n, swb::TRACE_CAP), max_entries);
    if (host && k > 0 && cudaMemcpyFromSymbol(host, swb::g_trace, (size_t)k * 32) != cudaSuccess) return -1;
    unsigned z = 0;
    cudaMemcpyToSymbol(swb::g_trace_n, &z, sizeof(z));
    return k;
}
#endif

sw_status_t sw_dpx_peak(int device, double milliseconds, double* cups, void* stream) {
    if (!cups) return SW_ERR_INVALID_ARGUMENT;
    *cups = 0;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return SW_ERR_CUDA;
    if (cur != device) return SW_ERR_WRONG_DEVICE;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return SW_ERR_CUDA;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 1024 * 4) != cudaSuccess) return SW_ERR_OUT_OF_MEMORY;
    const int blocks = p.multiProcessorCount * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 256;
    float ms = 0.f;
    sw_status_t st = SW_OK;
    for (int round = 0; round < 8; ++round) {
        cudaEventRecord(a, s);
        dpx_peak_kernel<<<blocks, threads, 0, s>>>(sink, iters, 3u, 0xfffafffau, 0xffffffffu);
        cudaEventRecord(b, s);
        if (cudaEventSynchronize(b) != cudaSuccess) { st = SW_ERR_CUDA; break; }
        cudaEventElapsedTime(&ms, a, b);
        if (ms >= 0.8 * milliseconds) break;
        const double scale = std::min(64.0, std::max(2.0, milliseconds / std::max(ms, 0.01f)));
        iters = (int)std::min(1e8, iters * scale);
    }
    if (st == SW_OK) {
        const double cellpairs = (double)blocks * threads * iters * DPX_CHAINS;
        *cups = 2.0 * cellpairs / (ms * 1e-3);
    }
    cudaEventDestroy(a); cudaEventDestroy(b);
    cudaFree(sink);
    return st;
}

}  // extern "C"
