// tools/dpx_probe.cu -- issue-rate probe for the integer/DPX instructions the
// Smith-Waterman inner loop uses (VIADDMNMX.S16x2, VIMNMX(3).S16x2, VIADD,
// PRMT, IMAD, LOP3, SHFL).  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a.
// Prints, per probe, the event-timed warp-instruction rate of the whole GPU and that
// rate per SM per cycle of the maximum SM clock (a lower bound of the per-cycle rate
// when the clock runs below its maximum).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

__device__ __forceinline__ unsigned hmax2(unsigned a, unsigned b) {
    unsigned d; asm volatile("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}

struct Out { unsigned long long cycles; unsigned v; };

__device__ __forceinline__ unsigned prmt(unsigned a, unsigned b, unsigned s) {
    unsigned d; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s)); return d;
}

// variant 0: 5.5-instruction Gotoh cell-pair mix (the roofline mix)
// variant 1: VIADDMNMX.S16x2 only
// variant 2: VIMNMX3.S16x2 only
// variant 3: PRMT only
// variant 4: IMAD only
// variant 5: mix + 1 PRMT per cell pair (6.5)
// variant 6: mix with the H+o add done by IMAD (FMA pipe)
// variant 7: VIADDMNMX + IMAD interleaved 1:1
// variant 8: LOP3 only
// variant 9: SHFL only
template <int V>
__global__ void probe(Out* out, unsigned seed, unsigned o2, unsigned e2) {
    unsigned h[CHAINS], e[CHAINS], f[CHAINS], x[CHAINS];
    unsigned best = 0, tgp = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        h[c] = seed * (c + 1) + threadIdx.x; e[c] = h[c] ^ 0x5555; f[c] = h[c] + 77; x[c] = h[c] * 3;
    }
    unsigned s = seed ^ 0x00030003u;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (V == 0 || V == 5 || V == 6) {
                unsigned ho;
                if (V == 6) ho = h[c] * seed + o2; else ho = __vadd2(h[c], o2);
                e[c] = __viaddmax_s16x2(e[c], e2, ho);
                f[c] = __viaddmax_s16x2(f[c], e2, ho);
                unsigned t = __vimax_s16x2_relu(e[c], f[c]);
                unsigned sc = s;
                if (V == 5) sc = prmt(x[c], s, 0x3210 + (c & 3));
                h[c] = __viaddmax_s16x2_relu(x[c], sc, t);
                x[c] = h[c];
                if (c & 1) best = __vimax3_s16x2_relu(best, h[c], h[c - 1]);
            } else if (V == 1) {
                h[c] = __viaddmax_s16x2(h[c], e2, e[c]);
            } else if (V == 2) {
                h[c] = __vimax3_s16x2_relu(h[c], e[c], f[c]);
                e[c] ^= h[c];
            } else if (V == 3) {
                h[c] = prmt(h[c], e[c], s + c);
            } else if (V == 4) {
                h[c] = h[c] * seed + e[c];
            } else if (V == 7) {
                h[c] = __viaddmax_s16x2(h[c], e2, e[c]);
                x[c] = x[c] * seed + f[c];
            } else if (V == 8) {
                h[c] = (h[c] & e[c]) ^ f[c];
                f[c] = (f[c] | h[c]) ^ e[c];
            } else if (V == 9) {
                h[c] = __shfl_up_sync(0xffffffffu, h[c], 1, 16);
            } else if (V == 10) {
                h[c] = __vadd2(h[c], e[c]);
            } else if (V == 11) {
                h[c] = __viaddmax_s16x2(h[c], e2, e[c]);
                x[c] = __vadd2(x[c], f[c]);
            } else if (V == 12) {
                // proposed cell: X = hd + s (VIADD), H = max3(X, E, F) relu, HO = H + o (VIADD), E, F addmax, PRMT, best/2
                unsigned hd = x[c];
                unsigned sc = prmt(hd, s, 0x3210 + (c & 3));
                e[c] = __viaddmax_s16x2(e[c], e2, h[c]);
                f[c] = __viaddmax_s16x2(f[c], e2, h[c]);
                unsigned X = __vadd2(hd, sc);
                unsigned H = __vimax3_s16x2_relu(X, e[c], f[c]);
                x[c] = h[c];
                h[c] = __vadd2(H, o2);
                if (c & 1) best = __vimax3_s16x2_relu(best, H, h[c - 1]);
            } else if (V == 13) {
                // same without PRMT
                unsigned hd = x[c];
                e[c] = __viaddmax_s16x2(e[c], e2, h[c]);
                f[c] = __viaddmax_s16x2(f[c], e2, h[c]);
                unsigned X = __vadd2(hd, s);
                unsigned H = __vimax3_s16x2_relu(X, e[c], f[c]);
                x[c] = h[c];
                h[c] = __vadd2(H, o2);
                if (c & 1) best = __vimax3_s16x2_relu(best, H, h[c - 1]);
            } else if (V == 15) {
                h[c] = hmax2(h[c], e[c]);
                e[c] = e[c] * seed + f[c];
            } else if (V == 16) {
                h[c] = __viaddmax_s16x2(h[c], e2, e[c]);
                x[c] = hmax2(x[c], h[c]);
            } else if (V == 17 || V == 18) {
                // the shipped TAG cell (E, F addmax; max3; H addmax; PRMT; HO and tag IMADs) with the
                // running max by VIMNMX3 (0.5 per cell pair, V17) or by max.f16x2 (1 per cell pair, V18)
                unsigned sc = prmt(x[c], s, 0x3210 + (c & 3));
                e[c] = __viaddmax_s16x2(e[c], e2, h[c]);
                f[c] = __viaddmax_s16x2(f[c], e2, h[c]);
                unsigned t = __vimax3_s16x2(e[c], f[c], e2);
                unsigned hb = __viaddmax_s16x2(x[c], sc, t);
                x[c] = h[c];
                h[c] = hb * seed + o2;
                unsigned tg = h[c] * 64u + (unsigned)c * 0x10001u;
                if (V == 17) { if (c & 1) best = __vimax3_s16x2(best, tg, tgp); else tgp = tg; }
                else best = hmax2(best, tg);
            } else if (V == 14) {
                h[c] = __viaddmax_s16x2(h[c], e2, e[c]);
                x[c] = (x[c] != f[c]) ? x[c] : e[c];
            }
        }
    }
    unsigned long long t1 = clock64();
    unsigned acc = best;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc ^= h[c] ^ e[c] ^ f[c] ^ x[c];
    if (threadIdx.x % 32 == 0) {
        Out* o = out + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
        o->cycles = t1 - t0;
        o->v = acc;
    }
}

// instructions per chain-iteration (per thread) that the probe is meant to measure
static const double INSTR_PER_CHAIN[19] = {5.5, 1, 1, 1, 1, 6.5, 5.5, 2, 2, 1, 1, 2, 6.5, 5.5, 3, 2, 2, 8.5, 8};
static const char* NAMES[19] = {"mix5.5(s16x2 gotoh)", "VIADDMNMX.S16x2", "VIMNMX3.S16x2(+LOP)", "PRMT", "IMAD",
                                "mix+PRMT(6.5)", "mix,IMAD for H+o", "VIADDMNMX+IMAD", "LOP3 x2", "SHFL",
                                "VIADD.16x2", "VIADDMNMX+VIADD.16x2", "cell v2 +PRMT (6.5)", "cell v2 (5.5)", "VIADDMNMX+ISETP+SEL",
                                "HMNMX2+IMAD", "VIADDMNMX+HMNMX2", "TAG cell, max3 best", "TAG cell, f16x2 best"};

template <int V>
void run(int sms, int blocks_per_sm, int threads) {
    int grid = sms * blocks_per_sm;
    int warps = grid * threads / 32;
    Out* d; cudaMalloc(&d, sizeof(Out) * warps);
    probe<V><<<grid, threads>>>(d, 3, 0xFFFAFFFAu, 0xFFFFFFFFu);  // warm
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<V><<<grid, threads>>>(d, 3, 0xFFFAFFFAu, 0xFFFFFFFFu);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    Out* h = new Out[warps];
    cudaMemcpy(h, d, sizeof(Out) * warps, cudaMemcpyDeviceToHost);
    double cyc = 0; for (int w = 0; w < warps; ++w) cyc += h[w].cycles; cyc /= warps;
    double winstr_per_warp = INSTR_PER_CHAIN[V] * CHAINS * ITERS;
    int warps_per_sm = blocks_per_sm * threads / 32;
    (void)cyc;  // per-warp clock64 spans do not measure SM cycles (warps of a block are not all
                // resident for the whole span): only the event-timed rate is reported
    double wall_rate = winstr_per_warp * warps / (ms * 1e-3);  // warp-instr / s (whole GPU)
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    double per_clk = wall_rate / ((double)sms * khz * 1e3);  // at the maximum SM clock (event-timed)
    printf("%-22s warps/SM=%2d  GPU warp-instr/s=%.3e  = %.3f warp-instr per SM per max-clock cycle  ms=%.3f\n",
           NAMES[V], warps_per_sm, wall_rate, per_clk, ms);
    if (V == 0 || V == 5 || V == 6 || V == 12 || V == 13 || V == 17 || V == 18) {
        double cellpairs = (double)CHAINS * ITERS * 32.0 * warps;
        printf("    -> cell updates/s (2 cells per s16x2 chain step) = %.3f TCUPS\n", 2 * cellpairs / (ms * 1e-3) / 1e12);
    }
    delete[] h; cudaFree(d);
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("device %s SMs=%d clockRate(kHz)=%d\n", p.name, p.multiProcessorCount, p.clockRate);
    int sms = p.multiProcessorCount;
    for (int bps : {4, 8}) {
        printf("--- blocks/SM=%d x 256 threads\n", bps);
        run<0>(sms, bps, 256); run<1>(sms, bps, 256); run<2>(sms, bps, 256); run<3>(sms, bps, 256);
        run<4>(sms, bps, 256); run<5>(sms, bps, 256); run<6>(sms, bps, 256); run<7>(sms, bps, 256);
        run<8>(sms, bps, 256); run<9>(sms, bps, 256); run<10>(sms, bps, 256); run<11>(sms, bps, 256);
        run<12>(sms, bps, 256); run<13>(sms, bps, 256); run<14>(sms, bps, 256);
        run<15>(sms, bps, 256); run<16>(sms, bps, 256); run<17>(sms, bps, 256); run<18>(sms, bps, 256);
    }
    return 0;
}
