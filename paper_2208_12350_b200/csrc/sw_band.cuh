// sw_band.cuh -- step a4 of SURVEY.md sec. 8(a) (reverse pass: the start) for DNA pairs whose
// score-S paths are confined to a narrow diagonal band: an anti-diagonal wavefront in which the
// lanes own DIAGONALS of the band instead of rows of the rectangle.
//
// Why ("Banded reverse pass").  Every score-S path of the reversed rectangle
// starts at its origin (reading R6), so its cells lie on diagonals d = j' - i' in [-DI, DD]
// (sw_common.cuh rev_band).  For an ADEPT-shaped read (150 bp, 2-3 % divergence) that band is
// ~30 diagonals wide, but a row-owning sweep (sw_wavefront.cuh) must visit the whole 160-row x
// (span + 31)-column parallelogram: its skew ties every lane to every column.  Here the work is
// (band width) x n2 cells.
//
// Geometry.  A segment of W lanes covers CAP = 16 W consecutive diagonals [dlo, dlo + CAP) of two
// pairs (the low / high s16x2 halves, each with its own dlo); lane L owns the 16 diagonals
// dlo + 16 L + s, s = 0..15.  All lanes sweep the anti-diagonals t = 2 i' + (d - dlo) together:
// at step t the slots of parity t & 1 are due, and every dependency of cell (i', d) -- left (i', d-1),
// up (i'-1, d+1), both on anti-diagonal t-1, and diagonal (i'-1, d) on t-2 -- is a slot of the
// other parity (this lane, or lane L-1's last / lane L+1's first slot by one shuffle), so the 8
// cells of a step are independent (no dependency chain inside a step).  Cells outside the band
// take the border (H = 0, E = F = 0): lower bounds, exact on every score-S path (band argument of
// sw_wavefront.cuh), so the cells holding S and their lexmin (j', i') are unchanged.
//
// Substitution scores with one PRMT per cell pair: the query side keeps, per cell, the profile
// word of its query code (byte c = s(q, c) - o for reference codes c = 0..3; 0 for a pad), the
// reference side the PRMT selector of its two reference codes (nibbles c, c|8 for the low half,
// 4+c, (4+c)|8 for the high half: the byte of the right profile word, sign-extended; a pad
// reference code selects the sign of a profile byte: s - o in {0, -1}, i.e. s < 0).  Along a lane's
// cells the query index falls and the reference index rises by one, and from one step to the next
// one of the two windows moves by one: both are 8-entry rings whose slot of a cell is a
// compile-time function of the step within a 16-step loop body (pure register renaming).
//
// The running maximum carries the TAG encoding of the forward TAG route: X * 64 + tag, the tag
// ordering the 32 cells of a lane's 4-step block by (j', i') (lexmin first); a block whose maximum
// reaches S * 64 emits its lexmin cell holding S with atomicMax on the (S, -j', -i') key.  Unlike
// a row sweep, a later block of a lane can hold a smaller j', so every block is checked (no early
// stop); keys merge associatively.
#pragma once
#include "sw_common.cuh"
#include "sw_pack.cuh"
#include "sw_wavefront.cuh"  // pack_key, opaque

namespace swb {

constexpr int BAND_K = 16;            // diagonals per lane
constexpr int BAND_KH = BAND_K / 2;   // cells per lane and step
constexpr int N_BAND = 2;             // band routes: 32 diagonals (2 lanes), 64 diagonals (4 lanes)
__host__ __device__ constexpr int band_cap(int b) { return b == 0 ? 32 : 64; }
__host__ __device__ constexpr int band_lanes(int b) { return b == 0 ? 2 : 4; }
// Per band pair one BAND_SLOT-byte slot of the band buffer (slot p + 1; slot 0 holds pads and serves the
// empty halves of a work item): the reversed query prefix q'[i] = q[q_end - i] as codes at
// QREV_PAD + i (pad codes elsewhere in its QREV_STRIDE bytes), then the reversed reference prefix as
// A-form PRMT selectors at BAND_ROFF + j' for j' in [-32, band_jw) (pad selectors outside [0, m2)).
// A buffer of its own: the row-sweep kernels read rrev as codes, also past a pair's region.
constexpr int QREV_STRIDE = 256;
constexpr int QREV_PAD = 32;
constexpr int BAND_SLOT = 576;
constexpr int BAND_ROFF = QREV_STRIDE + 32;
// longest reversed query of a band pair: the kernel reads q' up to i < n2 + CAP/2 + 15 (< QREV_STRIDE - QREV_PAD)
constexpr int BAND_MAX_N2 = 176;
#ifndef SW_BAND_MIN_PAIRS
#define SW_BAND_MIN_PAIRS 16384
#endif
constexpr int64_t BAND_MIN_PAIRS = SW_BAND_MIN_PAIRS;  // batches (chunks) below this keep the row-sweep reverse pass
constexpr int BAND_DLO_ALIGN = 8;     // dlo = -DI rounded down to a multiple of 8 (aligned reference words)
constexpr int BAND_JPAD = 16;         // selector bytes written for j' < n2 + CAP + BAND_JPAD
constexpr uint8_t SEL_PAD = 0x88;     // A-form selector of a pad reference code (sign of byte 0, twice)
__host__ __device__ __forceinline__ int band_dlo(int DI) { return -((DI + BAND_DLO_ALIGN - 1) / BAND_DLO_ALIGN) * BAND_DLO_ALIGN; }
__host__ __device__ __forceinline__ int band_jw(int n2, int cap) { return (n2 + cap + BAND_JPAD + 3) & ~3; }
static_assert(BAND_ROFF + ((BAND_MAX_N2 + 64 + BAND_JPAD + 3) & ~3) <= BAND_SLOT, "band slot holds the selectors");

// Tags of a lane's BAND_BLK-step block: cell k of step u sits at (j', i') = (J + k + ceil(u/2), I - k + floor(u/2));
// tag = 63 - rank of (j', i') among the block's 8 BAND_BLK cells (the running max picks the lexmin; the
// pairs (j', i') are distinct: their sum fixes u).  8 steps = 64 cells fill the 6 tag bits.
#ifndef SW_BAND_BLK
#define SW_BAND_BLK 4
#endif
constexpr int BAND_BLK = SW_BAND_BLK;
static_assert(BAND_BLK == 4 || BAND_BLK == 8, "band tag block: 4 or 8 steps");
__host__ __device__ constexpr int band_tag(int u, int k) {
    int rank = 0;
    for (int u2 = 0; u2 < BAND_BLK; ++u2)
        for (int k2 = 0; k2 < BAND_KH; ++k2) {
            const int jo = k + (u + 1) / 2, io = u / 2 - k, jo2 = k2 + (u2 + 1) / 2, io2 = u2 / 2 - k2;
            if (jo2 < jo || (jo2 == jo && io2 < io)) ++rank;
        }
    return 63 - rank;
}

struct BandParams {
    const uint8_t* slots;         // band buffer: pair p's slot at (p + 1) * BAND_SLOT, slot 0 = pads
    const int32_t* nlen;          // reverse rows n2 = q_end + 1
    const int32_t* mlen;          // reverse columns m2 (bounded, finish_fwd)
    const int32_t* target;        // forward score S
    const int32_t* order;         // reverse order: band pairs (route 0, route 1) first
    const int32_t* band_counts;   // pairs per band route (BatchStats::rev_band)
    unsigned long long* keys;     // reverse argmax keys
    int32_t* item_counter;        // work queue head (zeroed before launch)
    unsigned long long* swept;    // cells swept (statistics)
    Scoring sc;
    const BatchStats* stats;
    uint32_t tag_mul;             // = 64 (a parameter: the tag is an IMAD on the FMA pipe)
};

__device__ __forceinline__ uint32_t ldg_cg32(const uint8_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

#ifndef SW_BAND_CHECK
#define SW_BAND_CHECK 0  // development builds: trap on a read outside the pair's qrev slot / rrev region
#endif

#ifndef SW_BAND_MINB
#define SW_BAND_MINB 2  // 4-warp blocks per SM: 2 (163 registers, more of the 8-cell step in flight) measured faster than 3 or 4
#endif

template <int W>
__global__ void __launch_bounds__(128, SW_BAND_MINB) band_rev_kernel(BandParams P) {
    using T = TS16;
    constexpr int K = BAND_K, KH = BAND_KH;
    constexpr int SEGS = 32 / W, SLOTS = 2 * SEGS, CAP = W * K;
    constexpr int BR = W == 2 ? 0 : 1;  // band route
    static_assert(CAP == band_cap(BR) && W == band_lanes(BR), "band geometry");
    __shared__ uint32_t s_qprof[8];      // profile word per query code (4..7: pad)
    if (batch_rejected(P.stats)) return;
    if (threadIdx.x < 8) {
        uint32_t w = 0;
        const int c = threadIdx.x;
        if (c < 4)
            for (int k = 0; k < 4; ++k)
                w |= (uint32_t)(((c == k ? P.sc.match : P.sc.mismatch) - P.sc.gap_open) & 0xff) << (8 * k);
        s_qprof[c] = w;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int seg = lane / W, L = lane % W;
    const int first = BR == 0 ? 0 : P.band_counts[0];
    const int n_path = P.band_counts[BR];
    const int items = (n_path + SLOTS - 1) / SLOTS;
    const int o = P.sc.gap_open;
    const uint32_t o2s = T::splat(o), e2 = T::splat(P.sc.gap_extend);
    const uint32_t qtab = (uint32_t)__cvta_generic_to_shared(s_qprof);
    const uint32_t tag_mul = P.tag_mul;
#ifndef SW_BAND_QIMAD
#define SW_BAND_QIMAD 0
#endif
    // (SW_BAND_QIMAD) opaque shift multipliers so the byte extraction stays IMAD + IMAD.HI
    const uint32_t shl_c[4] = {opaque(1u << 24), opaque(1u << 16), opaque(1u << 8), opaque(1u)};
    // neighbours across lanes: lane L-1's last slot (left of slot 0), lane L+1's first (above slot K-1);
    // the band's own edges take the border (R = H + o = o, E = F = 0) by multiply-add (FMA pipe)
    const uint32_t notFirst = opaque(L != 0 ? 1u : 0u), notLast = opaque(L != W - 1 ? 1u : 0u);
    const uint32_t bR_lo = L == 0 ? o2s : 0u, bR_hi = L == W - 1 ? o2s : 0u;

    for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(P.item_counter, 1);
        item = __shfl_sync(FULL, item, 0);
        if (item >= items) break;
        // ---- slot descriptors (lane s < SLOTS holds slot s = 2 seg + half) ----
        int s_pid = -1, s_n = 0, s_m = 0, s_S = 0, s_dlo = 0;
        if (lane < SLOTS) {
            const int idx = item * SLOTS + lane;
            if (idx < n_path) {
                s_pid = P.order[first + idx];
                s_n = P.nlen[s_pid];
                s_m = P.mlen[s_pid];
                s_S = P.target[s_pid];
                int DI, DD;
                rev_band(P.sc.max_sigma, -o, -P.sc.gap_extend, s_S, s_n, s_m, DI, DD);
                s_dlo = band_dlo(DI);
            }
        }
        int nmax = s_n;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) nmax = max(nmax, __shfl_xor_sync(FULL, nmax, d));
        int h_pid[2], h_n[2], h_m[2], h_S[2], h_dlo[2];
        const uint8_t* qb[2];   // &q'[0] of the half
        const uint8_t* rb[2];   // &selector of j' = 0
        int rl[2];              // last readable reference word offset (the written region's end - 8)
        uint32_t tgt64 = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int sl = seg * 2 + h;
            h_pid[h] = __shfl_sync(FULL, s_pid, sl);
            h_n[h] = __shfl_sync(FULL, s_n, sl);
            h_m[h] = __shfl_sync(FULL, s_m, sl);
            h_S[h] = __shfl_sync(FULL, s_S, sl);
            h_dlo[h] = __shfl_sync(FULL, s_dlo, sl);
            // an empty half reads the pad slot 0 (its values stay at the border and never carry into the
            // other half's tag)
            const uint8_t* slot = P.slots + (int64_t)(h_pid[h] + 1) * BAND_SLOT;
            qb[h] = slot + QREV_PAD;
            rb[h] = slot + BAND_ROFF;
            rl[h] = h_pid[h] >= 0 ? band_jw(h_n[h], CAP) - 8 : 0;
            tgt64 = T::set(tgt64, h, h_pid[h] >= 0 ? h_S[h] * 64 : 0x7fff);
        }
        // steps: the last cell (lane W-1, slot K-1, i' = nmax - 1) is due at t = 2 nmax + CAP - 3
        const int Tn = 2 * nmax + CAP - 2;
        const int nbodies = (Tn + 15) / 16;

        uint32_t R[K], E[K], F[K];  // per slot: R = H + o, E^ = max(E, 0), F^ = max(F, 0) of its latest cell
#pragma unroll
        for (int s = 0; s < K; ++s) { R[s] = o2s; E[s] = 0u; F[s] = 0u; }
        // query ring: slot (i' mod 8); before step 0 it holds i' < 0 (pads: profile word 0)
        uint32_t QA[KH], QB[KH];
#pragma unroll
        for (int k = 0; k < KH; ++k) { QA[k] = 0u; QB[k] = 0u; }
        // reference ring: slot ((j' - 8L - dlo) mod 8); before step 1 it holds j' = 8L + dlo + k
        uint32_t RS[KH];
        {
            uint32_t a[2][2];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int w = 0; w < 2; ++w)
                    a[h][w] = ldg_cg32(rb[h] + min(8 * L + h_dlo[h] + 4 * w, rl[h] + 4 * w)) + (h ? 0x44444444u : 0u);
#pragma unroll
            for (int k = 0; k < KH; ++k)
                RS[k] = prmt(a[0][k >> 2], a[1][k >> 2], (uint32_t)((k & 3) | (((k & 3) + 4) << 4)));
        }
        // words of body b: query codes q'[8b - 8L + e], reference selectors j' = 8(b+1) + 8L + dlo + e
        auto ldq = [&](int b, int h, int w) {
            if (SW_BAND_CHECK && (8 * b - 8 * L + 4 * w < -QREV_PAD || 8 * b - 8 * L + 4 * w + 4 > QREV_STRIDE - QREV_PAD)) {
                printf("band qrev read out of slot: b %d L %d w %d nmax %d\n", b, L, w, nmax);
                __trap();
            }
            return ldg_cg32(qb[h] + 8 * b - 8 * L + 4 * w);
        };
        auto ldr = [&](int b, int h, int w) {  // the high half's selectors in B form (+4 per nibble pair)
            if (SW_BAND_CHECK) {
                const int off = min(8 * (b + 1) + 8 * L + h_dlo[h] + 4 * w, rl[h] + 4 * w);
                if (off < -32 || (h_pid[h] >= 0 && off + 4 > band_jw(h_n[h], CAP)) || (h_pid[h] < 0 && off + 4 > 16)) {
                    printf("band rrev read out of region: off %d b %d L %d h %d dlo %d n %d\n", off, b, L, h, h_dlo[h], h_n[h]);
                    __trap();
                }
            }
            return ldg_cg32(rb[h] + min(8 * (b + 1) + 8 * L + h_dlo[h] + 4 * w, rl[h] + 4 * w)) + (h ? 0x44444444u : 0u);
        };
        uint32_t qw[2][2], rw[2][2];  // [half][word] of the current body
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int w = 0; w < 2; ++w) { qw[h][w] = ldq(0, h, w); rw[h][w] = ldr(0, h, w); }

        uint32_t nbt = 0u;  // running max of the current 4-step block
        for (int b = 0; b < nbodies; ++b) {
            uint32_t qn[2][2], rn[2][2];  // next body's words (issued when the current ones are used up)
            const int ib = 8 * b - 8 * L;           // query index of the body's first new entry
            const int jb = 8 * b + 8 * L;           // j' - dlo of the cells' ring origin at u = 0
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (u == 8 && 16 * b + 8 >= Tn) break;  // warp-uniform: the body's second half is past the end
                if ((u & 1) == 0) {
                    // query shift: q'[8b - 8L + u/2] into ring slot u/2
                    const int e = u >> 1;
#if SW_BAND_QIMAD
                    // byte e & 3 of the word by multiply-high (FMA pipe): (w * 2^(24 - 8b)) mod 2^32, then >> 24
                    const uint32_t ca = __umulhi(qw[0][e >> 2] * shl_c[e & 3], 256u);
                    const uint32_t cb = __umulhi(qw[1][e >> 2] * shl_c[e & 3], 256u);
#else
                    const uint32_t ca = prmt(qw[0][e >> 2], 0u, (uint32_t)(0x4440 | (e & 3)));
                    const uint32_t cb = prmt(qw[1][e >> 2], 0u, (uint32_t)(0x4440 | (e & 3)));
#endif
                    if (SW_BAND_CHECK && (ca > 7u || cb > 7u)) { printf("band code %u %u\n", ca, cb); __trap(); }
                    QA[e] = lds32(qtab + ca * 4u);
                    QB[e] = lds32(qtab + cb * 4u);
                } else {
                    // reference shift: j' = 8(b+1) + 8L + dlo + (u-1)/2 into ring slot (u-1)/2
                    const int e = u >> 1;
                    RS[e] = prmt(rw[0][e >> 2], rw[1][e >> 2], (uint32_t)((e & 3) | (((e & 3) + 4) << 4)));
                }
                if (u == 7) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) { qn[h][0] = ldq(b + 1, h, 0); rn[h][0] = ldr(b + 1, h, 0); }
                }
                if (u == 15) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) { qn[h][1] = ldq(b + 1, h, 1); rn[h][1] = ldr(b + 1, h, 1); }
                }
                const int p = u & 1;
                uint32_t xR, xV;  // the cross-lane neighbour: (R, E) of lane L-1's slot K-1 or (R, F) of lane L+1's slot 0
                if (p == 0) {
                    xR = __shfl_up_sync(FULL, R[K - 1], 1, W) * notFirst + bR_lo;
                    xV = __shfl_up_sync(FULL, E[K - 1], 1, W) * notFirst;
                } else {
                    xR = __shfl_down_sync(FULL, R[0], 1, W) * notLast + bR_hi;
                    xV = __shfl_down_sync(FULL, F[0], 1, W) * notLast;
                }
                uint32_t Xt[KH];
#pragma unroll
                for (int k = 0; k < KH; ++k) {
                    const int s = 2 * k + p;
                    const uint32_t lR = s == 0 ? xR : R[s - 1], lE = s == 0 ? xV : E[s - 1];
                    const uint32_t uR = s == K - 1 ? xR : R[s + 1], uF = s == K - 1 ? xV : F[s + 1];
                    const int qi = ((u >> 1) - k) & 7;        // query slot of the cell: i' = I0 - k
                    const int ri = (((u + 1) >> 1) + k) & 7;  // reference slot: j' = J0 + k
                    const uint32_t sc = prmt(QA[qi], QB[qi], RS[ri]);
                    E[s] = T::addmax_relu(lE, e2, lR);                        // E^ = max(E^ + e, H + o, 0), left cell
                    F[s] = T::addmax_relu(uF, e2, uR);                        // F^ = max(F^ + e, H + o, 0), cell above
                    const uint32_t X = T::addmax(R[s], sc, E[s]);             // max(H_diag + s, E^)
                    R[s] = T::addmax(F[s], o2s, T::add(X, o2s));              // H + o = max(F^, X) + o
                    Xt[k] = X * tag_mul + (uint32_t)band_tag(u & (BAND_BLK - 1), k) * 0x10001u;
                }
#pragma unroll
                for (int k = 0; k < KH; k += 2) nbt = T::max3(nbt, Xt[k], Xt[k + 1]);
                if ((u & (BAND_BLK - 1)) == BAND_BLK - 1) {
                    // block check: some half's maximum reached S * 64 (every in-band cell holds <= S)
                    const uint32_t x = T::max2(nbt, tgt64) ^ nbt;
                    if (((x - 0x00010001u) & ~x & 0x80008000u) != 0u) {
                        const int ub = u - (BAND_BLK - 1);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int v = T::get(nbt, h);
                            if (h_pid[h] >= 0 && (v >> 6) == h_S[h]) {
                                const int tag = v & 63;
                                int cu = 0, ck = 0;
#pragma unroll
                                for (int uu = 0; uu < BAND_BLK; ++uu)
#pragma unroll
                                    for (int kk = 0; kk < KH; ++kk)
                                        if (band_tag(uu, kk) == tag) { cu = uu; ck = kk; }
                                const int JU = (cu + 1) >> 1, IU = cu >> 1;
                                const int i = ib + (ub >> 1) + IU - ck;
                                const int j = jb + h_dlo[h] + (ub >> 1) + JU + ck;
                                if (i >= 0 && i < h_n[h] && j >= 0 && j < h_m[h])
                                    atomicMax(P.keys + h_pid[h], pack_key(h_S[h], j, i));
                            }
                        }
                    }
                    nbt = 0u;
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int w = 0; w < 2; ++w) { qw[h][w] = qn[h][w]; rw[h][w] = rn[h][w]; }
        }
        if (lane == 0) atomicAdd(P.swept, (unsigned long long)Tn * (CAP / 2) * SLOTS);
    }
}

}  // namespace swb
