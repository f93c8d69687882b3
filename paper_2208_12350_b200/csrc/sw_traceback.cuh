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
};

// Largest interval of the batch (sizes the per-warp scratch) and the offset bases.
__global__ void trace_extent_kernel(sw_result_t res, int64_t n_pairs, const int64_t* q_off, const int64_t* r_off,
                                    int32_t* ext /* [0] max a, [1] max b */, int64_t* base /* q0, r0 */) {
    int la = 0, lb = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_pairs; p += (int64_t)gridDim.x * blockDim.x) {
        if (res.score[p] > 0) {
            la = max(la, res.q_end[p] - res.q_start[p] + 1);
            lb = max(lb, res.r_end[p] - res.r_start[p] + 1);
        }
    }
    if (la) atomicMax(ext + 0, la);
    if (lb) atomicMax(ext + 1, lb);
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

    for (;;) {
        int p32 = 0;
        if (lane == 0) p32 = atomicAdd(P.counter, 1);
        const int64_t p = __shfl_sync(FULL, p32, 0);
        if (p >= P.n_pairs) break;
        const int S = P.res.score[p];
        if (S <= 0) {
            if (lane == 0) P.n_ops[p] = S == 0 ? 0 : -1;
            continue;
        }
        const int qs = P.res.q_start[p], qe = P.res.q_end[p], rs = P.res.r_start[p], re = P.res.r_end[p];
        const int a = qe - qs + 1, b = re - rs + 1;
        const int ns = (a + TB_ROWS - 1) / TB_ROWS;
        const int steps = b + 31;           // column j (1-based) of lane L at step t: j = t - L + 1
        const int steps_pad = (steps + 31) & ~31;
        if ((int64_t)ns * steps_pad * 32 > P.dir_words || b + 1 > P.bnd_len) {
            if (lane == 0) { P.n_ops[p] = -1; atomicAdd(P.err, 1); }
            continue;
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
            // position of cell (i, j) (1-based) in the direction words: row i - 1 lives in stripe
            // s, lane L, bit group r; its word for column j is dir[rowoff + j] with
            // rowoff = (32 s + L) * steps_pad + L - 1.  The walk keeps (r, rowoff) and the current
            // word incrementally: an up move inside a lane's 5 rows reuses the word, every other
            // move loads exactly the word the next decision needs.
            int i = a, j = b, state = 0;
            int r = (a - 1) % TB_K, Lc = ((a - 1) % TB_ROWS) / TB_K;
            int64_t rowoff = (int64_t)(((a - 1) / TB_ROWS) * 32 + Lc) * steps_pad + Lc - 1;
            uint32_t w = dir[rowoff + j];
            bool bad = false;
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
                if (i == 0 || j == 0) { bad = true; break; }  // optimal paths start with an aligned pair
                const uint32_t c = (w >> (5 * r)) & 31u;
                if (state == 0) {
                    const int pr = (int)(c & 3u);
                    if (pr == 0) {
                        out[len++] = 'M';
                        up();
                        --j;
                        if (i > 0 && j > 0) w = dir[rowoff + j];
                    } else {
                        state = pr;  // 1: F, 2: E
                    }
                } else if (state == 1) {
                    out[len++] = 'I';
                    const bool open = c & 4u, ext = c & 8u;
                    if (up() && i > 0) w = dir[rowoff + j];
                    // H's preferred move of the cell above (row 0 is the border: E)
                    const int upr = i >= 1 ? (int)((w >> (5 * r)) & 3u) : 2;
                    state = (open && upr == 0) ? 0 : ((ext || (open && upr == 1)) ? 1 : 0);
                } else {
                    out[len++] = 'D';
                    const bool open = c & 16u;
                    --j;
                    int left = 1;  // column 0 (i >= 1): H == F
                    if (j >= 1) { w = dir[rowoff + j]; left = (int)((w >> (5 * r)) & 3u); }
                    state = (open && left != 2) ? 0 : 2;
                }
            }
            if (bad || len > a + b) { len = -1; atomicAdd(P.err, 1); }
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
    }
}

}  // namespace swb
