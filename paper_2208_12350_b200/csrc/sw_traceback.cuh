// sw_traceback.cuh -- alignment paths (the step after
// start-finding: "the reverse pass ... determines the alignment").
//
// For a pair with S > 0 and its reported interval A = q[q_start..q_end],
// B = r[r_start..r_end], the path is the optimal GLOBAL affine alignment of A
// and B (its score is S), ties broken reverse-lexicographically with M > I > D
// (reading R20; SPEC.md:395/464 diagonal > up > left).  One warp per
// pair:
//   1. the global Gotoh recurrence over the a x b rectangle as an anti-diagonal
//      wavefront (32 lanes x 5 rows = 160-row stripes, int32 lanes), storing 5
//      bits per cell -- H's preferred predecessor (diagonal / F / E, in that
//      priority), F opened here, F extended here, E opened here -- as one
//      32-bit word per lane and step, staged per 32 steps in shared memory and
//      written lane-major (each lane one 128-byte line), so the walk below
//      stays inside a line for up to 32 consecutive steps (L1 hits);
//   2. one lane walks the path back from (a, b) through the stored bits with
//      the state machine of oracle_traceback's definition (the bits of the
//      cell above / to the left give the next op's preference in gap states);
//   3. the warp reverses the op string in place.
#pragma once
#include "sw_common.cuh"
#include "sw_pack.cuh"

namespace swb {

constexpr int TB_K = 5;                 // rows per lane
constexpr int TB_ROWS = 32 * TB_K;      // rows per stripe
constexpr int TB_NEG = -(1 << 28);      // -inf of the global recurrence (no overflow with int32 adds)

struct TraceParams {
    const uint8_t* queries;
    const int64_t* q_off;
    const uint8_t* refs;
    const int64_t* r_off;
    int64_t n_pairs;
    int64_t q0, r0;                     // q_off[0], r_off[0] (output offsets are relative to them)
    sw_result_t res;                    // the batch's sw_align_batch results
    uint8_t* ops;
    int32_t* n_ops;
    Scoring sc;
    uint32_t* dir;                      // per-warp direction words
    int64_t dir_words;                  // per warp
    int2* bnd;                          // per-warp stripe boundary row (H, F) per column
    int64_t bnd_len;                    // per warp
    int32_t* counter;                   // work queue head
    int32_t* err;                       // internal-error count
    int32_t* counter16;                 // work queue head of the s16x2 kernel (pairs of pairs)
    int skip16;                         // int32 kernel: pairs tb16_ok() selects were done by the s16x2 kernel
};

// The s16x2 kernel (two pairs per warp, 16-bit lanes) takes a pair when every value of its
// global recurrence fits: scores <= S <= 16000, every cell >= 2 o + (a + b) e >= -16000 (the
// two-gap path), the -inf sentinel -16384 plus one gap score stays > -32768, and the DNA
// substitution scores fit the int8 table bytes.  Same comparisons, same bits as int32.
constexpr int TB16_NEG = -16384;
__device__ __forceinline__ bool tb16_ok(const Scoring& sc, int S, int a, int b) {
    return sc.alphabet == SW_ALPHABET_DNA && S > 0 && S <= 16000 && sc.match <= 127 && sc.mismatch >= -128 &&
           sc.gap_open >= -8000 && -2LL * sc.gap_open - (long long)(a + b) * sc.gap_extend <= 16000;
}

// Walk the path back from (a, b) through the stored direction bits (one thread), writing the
// ops end -> start; returns their count, or -1 if the bits do not lead back to an aligned pair.
// Position of cell (i, j) (1-based): row i - 1 lives in stripe s, lane L, bit group r; its word
// for column j is dir[rowoff + j] with rowoff = (32 s + L) * steps_pad + L - 1.  The walk keeps
// (r, L, rowoff) and the current word incrementally: an up move inside a lane's 5 rows reuses the
// word, every other move loads exactly the word the next decision needs.
// Bit encodings: RAW = false (int32 kernel): bits 1:0 = H's preferred move (0 diagonal, 1 F,
// 2 E); RAW = true (s16x2 kernel): bit 0 = not diagonal, bit 1 = E preferred over F.  Both:
// bit 2 F opened here, bit 3 F extended here, bit 4 E opened here.
template <bool RAW>
__device__ __forceinline__ int tb_pref(uint32_t c) {
    if (RAW) return (c & 1u) ? ((c & 2u) ? 2 : 1) : 0;
    return (int)(c & 3u);
}

// The direction words were written by this warp earlier in the same kernel: every load below is
// an L2-coherent ld.global.cg (never the non-coherent read-only path, which may return stale lines).
template <bool RAW>
__device__ int tb_walk(const uint32_t* dir, int64_t steps_pad, int a, int b, uint8_t* out) {
    int len = 0;
    int i = a, j = b, state = 0;
    int r = (a - 1) % TB_K, Lc = ((a - 1) % TB_ROWS) / TB_K;
    int64_t rowoff = (int64_t)(((a - 1) / TB_ROWS) * 32 + Lc) * steps_pad + Lc - 1;
    uint32_t w = __ldcg(dir + rowoff + j);
    // one row up: returns true when the row's word lives in another lane's line
    auto up = [&]() -> bool {
        --i;
        if (r > 0) { --r; return false; }
        r = TB_K - 1;
        if (Lc > 0) { --Lc; rowoff -= steps_pad + 1; }
        else { Lc = 31; rowoff += 31 - steps_pad; }
        return true;
    };
    while (i > 0 || j > 0) {
        if (i == 0 || j == 0) return -1;  // optimal paths start with an aligned pair
        const uint32_t c = (w >> (5 * r)) & 31u;
        if (state == 0) {
            const int pr = tb_pref<RAW>(c);
            if (pr == 0) {
                out[len++] = 'M';
                up();
                --j;
                if (i > 0 && j > 0) w = __ldcg(dir + rowoff + j);
            } else {
                state = pr;  // 1: F, 2: E
            }
        } else if (state == 1) {
            out[len++] = 'I';
            const bool open = c & 4u, ext = c & 8u;
            if (up() && i > 0) w = __ldcg(dir + rowoff + j);
            // H's preferred move of the cell above (row 0 is the border: E)
            const int upr = i >= 1 ? tb_pref<RAW>((w >> (5 * r)) & 31u) : 2;
            state = (open && upr == 0) ? 0 : ((ext || (open && upr == 1)) ? 1 : 0);
        } else {
            out[len++] = 'D';
            const bool open = c & 16u;
            --j;
            int left = 1;  // column 0 (i >= 1): H == F
            if (j >= 1) { w = __ldcg(dir + rowoff + j); left = tb_pref<RAW>((w >> (5 * r)) & 31u); }
            state = (open && left != 2) ? 0 : 2;
        }
    }
    return len > a + b ? -1 : len;
}

// A pair with S > 0 has a path only if its interval lies inside its sequences:
// 0 <= q_start <= q_end < n and 0 <= r_start <= r_end < m.  The kernels below never trust the
// caller's (or an earlier call's) coordinates beyond that: a pair outside it gets n_ops = -1.
__device__ __forceinline__ bool tb_interval_ok(const sw_result_t& res, int64_t p, const int64_t* q_off, const int64_t* r_off) {
    const int64_t n = q_off[p + 1] - q_off[p], m = r_off[p + 1] - r_off[p];
    const int qs = res.q_start[p], qe = res.q_end[p], rs = res.r_start[p], re = res.r_end[p];
    return qs >= 0 && qs <= qe && qe < n && rs >= 0 && rs <= re && re < m;
}

// Largest valid interval of the batch (sizes the per-warp scratch), the offset bases, and the
// number of pairs with S > 0 whose interval is not inside their sequences (ext[9]).
__global__ void trace_extent_kernel(sw_result_t res, int64_t n_pairs, const int64_t* q_off, const int64_t* r_off,
                                    int32_t* ext /* [0] max a, [1] max b, [9] bad intervals */, int64_t* base /* q0, r0 */) {
    int la = 0, lb = 0, bad = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_pairs; p += (int64_t)gridDim.x * blockDim.x) {
        if (res.score[p] > 0) {
            if (!tb_interval_ok(res, p, q_off, r_off)) { ++bad; continue; }
            la = max(la, res.q_end[p] - res.q_start[p] + 1);
            lb = max(lb, res.r_end[p] - res.r_start[p] + 1);
        }
    }
    if (la) atomicMax(ext + 0, la);
    if (lb) atomicMax(ext + 1, lb);
    if (bad) atomicAdd(ext + 9, bad);
    if (blockIdx.x == 0 && threadIdx.x == 0) { base[0] = q_off[0]; base[1] = r_off[0]; }
}

__global__ void __launch_bounds__(128) traceback_kernel(const TraceParams P) {
    __shared__ uint8_t lut[256];
    __shared__ uint32_t tbuf[4][32][33];  // per warp: 32 steps x 32 lanes of direction words (padded)
    __shared__ int8_t s_sigma[24 * 24];
    for (int c = threadIdx.x; c < 256; c += blockDim.x) lut[c] = ascii_code(P.sc.alphabet, c);
    for (int k = threadIdx.x; k < 24 * 24; k += blockDim.x)
        s_sigma[k] = (int8_t)(P.sc.alphabet == SW_ALPHABET_DNA ? 0 : c_blosum62[k / 24][k % 24]);
    __syncthreads();
    const bool dna = P.sc.alphabet == SW_ALPHABET_DNA;
    auto sigma = [&](int a, int b) -> int {
        return dna ? (a == b ? P.sc.match : P.sc.mismatch) : (int)s_sigma[a * 24 + b];
    };
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t* dir = P.dir + gwarp * P.dir_words;
    int2* bnd = P.bnd + gwarp * P.bnd_len;
    const int o = P.sc.gap_open, e = P.sc.gap_extend;

    // one pair, warp-cooperative: recurrence + direction bits, walk, reversal
    auto one_pair = [&](const int64_t p) {
        const int qs = P.res.q_start[p], qe = P.res.q_end[p], rs = P.res.r_start[p], re = P.res.r_end[p];
        const int a = qe - qs + 1, b = re - rs + 1;
        const int ns = (a + TB_ROWS - 1) / TB_ROWS;
        const int steps = b + 31;           // column j (1-based) of lane L at step t: j = t - L + 1
        const int steps_pad = (steps + 31) & ~31;
        if ((int64_t)ns * steps_pad * 32 > P.dir_words || b + 1 > P.bnd_len) {
            if (lane == 0) { P.n_ops[p] = -1; atomicAdd(P.err, 1); }
            return;
        }
        const uint8_t* A = P.queries + P.q_off[p] + qs;
        const uint8_t* B = P.refs + P.r_off[p] + rs;

        // ---- 1. global Gotoh over the rectangle, 5 direction bits per cell ----
        for (int s = 0; s < ns; ++s) {
            const int row0 = s * TB_ROWS + lane * TB_K;  // 0-based row of this lane's first row
            int qc[TB_K], Hl[TB_K], El[TB_K];
#pragma unroll
            for (int r = 0; r < TB_K; ++r) {
                const int i = row0 + r + 1;              // 1-based
                qc[r] = i <= a ? lut[A[i - 1]] : 0;
                Hl[r] = o + (i - 1) * e;                 // H[i][0]
                El[r] = TB_NEG;                          // E[i][0]
            }
            // this lane's last row at its current column (column 0 until it starts: the left border)
            int hoLast = Hl[TB_K - 1], fLast = TB_NEG;
            int diagUp = s == 0 ? 0 : bnd[0].x;          // H of the row above at the previous column
            __syncwarp();
            for (int t = 0; t < steps; ++t) {
                const int j = t - lane + 1;              // this lane's column (1-based)
                // row above at column j: the previous lane's last row (computed at step t-1) or the
                // stripe boundary (border row / the previous stripe's bottom row)
                int upH = __shfl_up_sync(FULL, hoLast, 1);
                int upF = __shfl_up_sync(FULL, fLast, 1);
                if (lane == 0) {
                    if (j >= 1 && j <= b) {
                        if (s == 0) { upH = o + (j - 1) * e; upF = TB_NEG; }
                        else { const int2 v = bnd[j]; upH = v.x; upF = v.y; }
                    }
                }
                uint32_t word = 0;
                if (j >= 1 && j <= b) {
                    const int rc = lut[B[j - 1]];
                    int hd = diagUp, hu = upH, F = upF;
#pragma unroll
                    for (int r = 0; r < TB_K; ++r) {
                        const int ev = El[r] + e, eo = Hl[r] + o;
                        const int En = max(ev, eo);
                        const int fv = F + e, fo = hu + o;
                        const int Fn = max(fv, fo);
                        const int d = hd + sigma(qc[r], rc);
                        const int Hn = max(d, max(Fn, En));
                        const uint32_t pref = Hn == d ? 0u : (Hn == Fn ? 1u : 2u);
                        word |= (pref | (fo >= fv ? 4u : 0u) | (fv >= fo ? 8u : 0u) | (eo >= ev ? 16u : 0u)) << (5 * r);
                        hd = Hl[r];
                        Hl[r] = Hn; El[r] = En; F = Fn; hu = Hn;
                    }
                    hoLast = Hl[TB_K - 1];
                    fLast = F;
                    if (lane == 31) bnd[j] = make_int2(hoLast, fLast);  // for the next stripe
                }
                diagUp = upH;
                tbuf[wib][lane][t & 31] = word;
                if ((t & 31) == 31 || t == steps - 1) {  // flush 32 steps: lane L writes its own line
                    __syncwarp();
                    uint32_t* dst = dir + ((int64_t)(s * 32 + lane) * steps_pad + (t & ~31));
#pragma unroll
                    for (int k = 0; k < 32; k += 4)
                        *reinterpret_cast<uint4*>(dst + k) =
                            make_uint4(tbuf[wib][lane][k], tbuf[wib][lane][k + 1], tbuf[wib][lane][k + 2], tbuf[wib][lane][k + 3]);
                    __syncwarp();
                }
            }
            __syncwarp();
            if (lane == 31) bnd[0] = make_int2(o + (s + 1) * TB_ROWS * e - e, 0);  // H[row0 of next stripe - 1][0]
            __syncwarp();
        }
        __syncwarp();

        // ---- 2. walk back from (a, b) (lane 0) ----
        uint8_t* out = P.ops + (P.q_off[p] - P.q0) + (P.r_off[p] - P.r0);
        int len = 0;
        if (lane == 0) {
            len = tb_walk<false>(dir, steps_pad, a, b, out);
            if (len < 0) atomicAdd(P.err, 1);
        }
        len = __shfl_sync(FULL, len, 0);
        __syncwarp();
        // ---- 3. ops were written end -> start: reverse in place ----
        for (int k = lane; k < len / 2; k += 32) {
            const uint8_t x = out[k];
            out[k] = out[len - 1 - k];
            out[len - 1 - k] = x;
        }
        if (lane == 0) P.n_ops[p] = len;
        __syncwarp();
    };

    for (;;) {
        // 32 pairs per queue step: the lanes sort out S <= 0 pairs and the pairs the s16x2 kernel
        // took, then the warp aligns the rest one by one (one pair per step when there is no
        // s16x2 kernel: every pair is work, keep the warps busy)
        const int grab = P.skip16 ? 32 : 1;
        int b32 = 0;
        if (lane == 0) b32 = atomicAdd(P.counter, grab);
        const int64_t pbase = __shfl_sync(FULL, b32, 0);
        if (pbase >= P.n_pairs) break;
        bool need = false;
        const int64_t pl = pbase + lane;
        if (lane < grab && pl < P.n_pairs) {
            const int Sl = P.res.score[pl];
            if (Sl <= 0 || !tb_interval_ok(P.res, pl, P.q_off, P.r_off)) {
                P.n_ops[pl] = Sl == 0 ? 0 : -1;  // invalid pair, or an interval outside its sequences
            } else {
                const int al = P.res.q_end[pl] - P.res.q_start[pl] + 1, bl = P.res.r_end[pl] - P.res.r_start[pl] + 1;
                need = !(P.skip16 && tb16_ok(P.sc, Sl, al, bl));  // else done by traceback16_kernel
            }
        }
        for (uint32_t todo = __ballot_sync(FULL, need); todo; todo &= todo - 1) one_pair(pbase + (__ffs(todo) - 1));
    }
}

// s16x2 alignment paths: the int32 kernel's recurrence, bits and walk, with two pairs per warp
// -- pair 2k in the low and pair 2k + 1 in the high 16 bits of every register (DNA pairs that
// tb16_ok() admits).  Each DPX VIMNMX.S16x2 returns the maximum of both halves and both "a >= b"
// predicates, which are exactly the direction bits (E opened, F opened, F extended, F over E,
// diagonal over gaps), so a cell pair costs ~11 ALU operations instead of ~40.  The substitution
// score of a row comes from a per-row 4-byte table (s(q_i, c) for the four codes) per half: one
// PRMT picks and sign-extends both halves' bytes for the column's two reference codes.  Lanes 0
// and 1 walk the two paths; half-warps reverse them.
__device__ __forceinline__ uint32_t v2add(uint32_t a, uint32_t b) { return __vadd2(a, b); }
__device__ __forceinline__ void or_if(uint32_t& w, bool p, uint32_t bit) {
    asm("{ .reg .pred q; setp.ne.u32 q, %1, 0; @q or.b32 %0, %0, %2; }" : "+r"(w) : "r"((uint32_t)p), "r"(bit));
}
__device__ __forceinline__ uint32_t splat16(int v) { return ((uint32_t)v & 0xffffu) * 0x10001u; }

__global__ void __launch_bounds__(128) traceback16_kernel(const TraceParams P) {
    __shared__ uint8_t lut[256];
    __shared__ uint32_t tbuf[4][2][32][33];  // per warp and half: 32 steps x 32 lanes of direction words
    __shared__ uint16_t selring[4][64];      // per warp: PRMT selector of columns j (index j & 63)
    for (int c = threadIdx.x; c < 256; c += blockDim.x) lut[c] = ascii_code(P.sc.alphabet, c);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t* dirw = P.dir + gwarp * 2 * P.dir_words;  // two regions: low / high half
    uint2* bnd = reinterpret_cast<uint2*>(P.bnd) + gwarp * P.bnd_len;
    const int o = P.sc.gap_open, e = P.sc.gap_extend;
    const uint32_t o2 = splat16(o), e2 = splat16(e), neg2 = splat16(TB16_NEG);
    const uint32_t mm = (uint32_t)(P.sc.mismatch & 0xff) * 0x01010101u, ma = (uint32_t)(P.sc.match & 0xff);

    for (;;) {
        int k32 = 0;
        if (lane == 0) k32 = atomicAdd(P.counter16, 1);
        const int64_t p0 = 2 * (int64_t)__shfl_sync(FULL, k32, 0);
        if (p0 >= P.n_pairs) break;
        int aa[2], bb[2], qs[2], rs[2];
        int64_t pp[2];
        bool any = false;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            pp[h] = p0 + h;
            aa[h] = 0; bb[h] = 0; qs[h] = 0; rs[h] = 0;
            if (pp[h] < P.n_pairs) {
                const int S = P.res.score[pp[h]];
                if (S > 0 && tb_interval_ok(P.res, pp[h], P.q_off, P.r_off)) {  // else the int32 kernel writes -1
                    const int a = P.res.q_end[pp[h]] - P.res.q_start[pp[h]] + 1;
                    const int b = P.res.r_end[pp[h]] - P.res.r_start[pp[h]] + 1;
                    if (tb16_ok(P.sc, S, a, b)) {
                        aa[h] = a; bb[h] = b; qs[h] = P.res.q_start[pp[h]]; rs[h] = P.res.r_start[pp[h]];
                        any = true;
                    }
                }
            }
        }
        if (!any) continue;
        const int amax = max(aa[0], aa[1]), bmax = max(bb[0], bb[1]);
        const int ns = (amax + TB_ROWS - 1) / TB_ROWS;
        const int steps = bmax + 31;
        const int steps_pad = (steps + 31) & ~31;
        if ((int64_t)ns * steps_pad * 32 > P.dir_words || bmax + 1 > P.bnd_len) {
            if (lane < 2 && (lane == 0 ? aa[0] : aa[1]) > 0) { P.n_ops[p0 + lane] = -1; atomicAdd(P.err, 1); }
            continue;
        }
        const uint8_t* A0 = P.queries + P.q_off[pp[0]] + qs[0];
        const uint8_t* A1 = P.queries + (aa[1] ? P.q_off[pp[1]] + qs[1] : 0);
        const uint8_t* B0 = P.refs + P.r_off[pp[0]] + rs[0];
        const uint8_t* B1 = P.refs + (bb[1] ? P.r_off[pp[1]] + rs[1] : 0);

        for (int s = 0; s < ns; ++s) {
            const int row0 = s * TB_ROWS + lane * TB_K;
            uint32_t T0[TB_K], T1[TB_K], Hl[TB_K], El[TB_K];
#pragma unroll
            for (int r = 0; r < TB_K; ++r) {
                const int i = row0 + r + 1;
                const int c0 = i <= aa[0] ? lut[A0[i - 1]] : 0, c1 = i <= aa[1] ? lut[A1[i - 1]] : 0;
                T0[r] = (mm & ~(0xffu << (8 * c0))) | (ma << (8 * c0));
                T1[r] = (mm & ~(0xffu << (8 * c1))) | (ma << (8 * c1));
                Hl[r] = splat16(o + (i - 1) * e);  // H[i][0]: saturates only past the rows tb16_ok admits
                El[r] = neg2;
            }
            uint32_t hoLast = Hl[TB_K - 1], fLast = neg2;
            uint32_t diagUp = s == 0 ? 0u : bnd[0].x;
            __syncwarp();
            for (int t = 0; t < steps; ++t) {
                const int j = t - lane + 1;
                if ((t & 31) == 0) {
                    // selectors of columns t + 1 .. t + 32, one per lane (the ring keeps the previous
                    // 32, which the lagging lanes still read): bytes s(q, r0c) sign-extended into
                    // the low half, s(q, r1c) into the high half
                    const int jj = t + 1 + lane;
                    const uint32_t r0c = jj <= bb[0] ? lut[B0[jj - 1]] : 0u, r1c = jj <= bb[1] ? lut[B1[jj - 1]] : 0u;
                    selring[wib][jj & 63] =
                        (uint16_t)(r0c | ((r0c | 8u) << 4) | ((r1c + 4u) << 8) | (((r1c + 4u) | 8u) << 12));
                    __syncwarp();
                }
                uint32_t upH = __shfl_up_sync(FULL, hoLast, 1);
                uint32_t upF = __shfl_up_sync(FULL, fLast, 1);
                if (lane == 0 && j >= 1 && j <= bmax) {
                    if (s == 0) { upH = splat16(o + (j - 1) * e); upF = neg2; }
                    else { const uint2 v = bnd[j]; upH = v.x; upF = v.y; }
                }
                uint32_t w0 = 0, w1 = 0;
                if (j >= 1 && j <= bmax) {
                    const uint32_t sel = selring[wib][j & 63];
                    uint32_t hd = diagUp, hu = upH, F = upF;
#pragma unroll
                    for (int r = 0; r < TB_K; ++r) {
                        bool eH, eL, foH, foL, fxH, fxL, pfH, pfL, pdH, pdL;
                        const uint32_t ev = v2add(El[r], e2), eo = v2add(Hl[r], o2);
                        const uint32_t En = __vibmax_s16x2(eo, ev, &eH, &eL);
                        const uint32_t fv = v2add(F, e2), fo = v2add(hu, o2);
                        const uint32_t Fn = __vibmax_s16x2(fo, fv, &foH, &foL);
                        (void)__vibmax_s16x2(fv, fo, &fxH, &fxL);
                        uint32_t sg;
                        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(T0[r]), "r"(T1[r]), "r"(sel));
                        const uint32_t d = v2add(hd, sg);
                        const uint32_t FE = __vibmax_s16x2(Fn, En, &pfH, &pfL);
                        const uint32_t Hn = __vibmax_s16x2(d, FE, &pdH, &pdL);
                        // one predicated LOP3 per bit (ptxas forwards the VIMNMX predicates)
                        const uint32_t sh = 5u * r;
                        or_if(w0, !pdL, 1u << sh); or_if(w0, !pfL, 2u << sh); or_if(w0, foL, 4u << sh);
                        or_if(w0, fxL, 8u << sh); or_if(w0, eL, 16u << sh);
                        or_if(w1, !pdH, 1u << sh); or_if(w1, !pfH, 2u << sh); or_if(w1, foH, 4u << sh);
                        or_if(w1, fxH, 8u << sh); or_if(w1, eH, 16u << sh);
                        hd = Hl[r];
                        Hl[r] = Hn; El[r] = En; F = Fn; hu = Hn;
                    }
                    hoLast = Hl[TB_K - 1];
                    fLast = F;
                    if (lane == 31) bnd[j] = make_uint2(hoLast, fLast);
                }
                diagUp = upH;
                tbuf[wib][0][lane][t & 31] = w0;
                tbuf[wib][1][lane][t & 31] = w1;
                if ((t & 31) == 31 || t == steps - 1) {
                    __syncwarp();
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t* dst = dirw + h * P.dir_words + ((int64_t)(s * 32 + lane) * steps_pad + (t & ~31));
#pragma unroll
                        for (int k = 0; k < 32; k += 4)
                            *reinterpret_cast<uint4*>(dst + k) = make_uint4(tbuf[wib][h][lane][k], tbuf[wib][h][lane][k + 1],
                                                                            tbuf[wib][h][lane][k + 2], tbuf[wib][h][lane][k + 3]);
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
            if (lane == 31) bnd[0] = make_uint2(splat16(o + (s + 1) * TB_ROWS * e - e), 0u);
            __syncwarp();
        }
        __syncwarp();

        // walks: lane h walks half h's path; then half-warp h reverses it
        int len = 0;
        const int hh = lane >> 4, hl = lane & 15;
        const int aw = lane == 0 ? aa[0] : aa[1], bw = lane == 0 ? bb[0] : bb[1];
        const int64_t pw = lane == 0 ? pp[0] : pp[1];
        if (lane < 2 && aw > 0) {
            uint8_t* out = P.ops + (P.q_off[pw] - P.q0) + (P.r_off[pw] - P.r0);
            len = tb_walk<true>(dirw + lane * P.dir_words, steps_pad, aw, bw, out);
            if (len < 0) atomicAdd(P.err, 1);
        }
        const int lenh = __shfl_sync(FULL, len, hh);
        const int ah = hh ? aa[1] : aa[0];
        const int64_t ph = hh ? pp[1] : pp[0];
        __syncwarp();
        if (ah > 0 && lenh > 0) {
            uint8_t* o8 = P.ops + (P.q_off[ph] - P.q0) + (P.r_off[ph] - P.r0);
            for (int k = hl; k < lenh / 2; k += 16) {
                const uint8_t x = o8[k];
                o8[k] = o8[lenh - 1 - k];
                o8[lenh - 1 - k] = x;
            }
        }
        if (lane < 2 && aw > 0) P.n_ops[pw] = len;
        __syncwarp();
    }
}

}  // namespace swb
