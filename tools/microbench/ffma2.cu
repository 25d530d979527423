// Microbenchmark: sustained FP32 FMA throughput per SM on B200 for the
// operand patterns the fused step uses (debug/roofline aid; not product code).
#include <cuda_runtime.h>
#include <stdio.h>

template <int MODE>
__global__ void k(float *out, int iters, float s) {
    // 8 independent accumulator chains per thread
    float2 a[8], u[8];
    float g[8];
    for (int i = 0; i < 8; ++i) {
        a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        u[i] = make_float2(1.0001f + i * 1e-4f, 0.9999f - i * 1e-4f);
        g[i] = s * (i + 1);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {        // FFMA2 pair*pair+pair (u*u accumulate)
                a[i] = __ffma2_rn(u[i], u[(i + 1) & 7], a[i]);
            } else if (MODE == 1) { // FFMA2 pair*|scalar|+pair (Eq. 5 pattern)
                const float gg = fabsf(g[i]);
                a[i] = __ffma2_rn(u[i], make_float2(gg, gg), a[i]);
            } else if (MODE == 2) { // scalar FFMA, 3 registers
                a[i].x = fmaf(u[i].x, g[i], a[i].x);
                a[i].y = fmaf(u[i].y, g[(i + 3) & 7], a[i].y);
            } else if (MODE == 3) { // FADD2
                a[i] = __fadd2_rn(a[i], u[i]);
            } else if (MODE == 4) { // mix: FFMA2 on even chains, 2 scalar FFMA on odd chains
                if (i & 1) {
                    a[i].x = fmaf(u[i].x, g[i], a[i].x);
                    a[i].y = fmaf(u[i].y, g[(i + 3) & 7], a[i].y);
                } else {
                    const float gg = fabsf(g[i]);
                    a[i] = __ffma2_rn(u[i], make_float2(gg, gg), a[i]);
                }
            } else if (MODE == 5) { // scalar FADD
                a[i].x = a[i].x + u[i].x;
                a[i].y = a[i].y + g[i];
            } else {                // mix: 1 FFMA2 per 4 scalar FFMA
                if ((i & 3) == 0) {
                    const float gg = fabsf(g[i]);
                    a[i] = __ffma2_rn(u[i], make_float2(gg, gg), a[i]);
                } else {
                    a[i].x = fmaf(u[i].x, g[i], a[i].x);
                    a[i].y = fmaf(u[i].y, g[(i + 3) & 7], a[i].y);
                }
            }
        }
    }
    float r = 0.f;
    for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char *names[7] = {"FFMA2 pair*pair+pair", "FFMA2 pair*|scalar|+pair", "FFMA x2 scalar", "FADD2",
                            "mix 1 FFMA2 : 2 FFMA", "FADD x2 scalar", "mix 1 FFMA2 : 6 FFMA"};
    for (int mode = 0; mode < 7; ++mode) {
        for (int warps = 8; warps <= 16; warps *= 2) {
            const int blocks = 148 * (warps / 4), threads = 128, iters = 4096;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 1.0f);
                if (mode == 1) k<1><<<blocks, threads>>>(out, iters, 1.0f);
                if (mode == 2) k<2><<<blocks, threads>>>(out, iters, 1.0f);
                if (mode == 3) k<3><<<blocks, threads>>>(out, iters, 1.0f);
                if (mode == 4) k<4><<<blocks, threads>>>(out, iters, 1.0f);
                if (mode == 5) k<5><<<blocks, threads>>>(out, iters, 1.0f);
                if (mode == 6) k<6><<<blocks, threads>>>(out, iters, 1.0f);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 1) {
                    const double per = mode == 2 || mode == 5 ? 16 : (mode == 4 ? 12 : (mode == 6 ? 14 : 8));
                    const double instr = (double)blocks * threads / 32 * iters * per;
                    const double fmas = (double)blocks * threads * iters * 8 * 2;
                    printf("%-28s warps/SM %2d: %.3f ms, %.2f warp-instr/clk/SM, %.0f FMA/clk/SM (clock %d MHz assumed)\n",
                           names[mode], warps, ms, instr / (ms * 1e-3) / (clk * 1e3) / 148,
                           fmas / (ms * 1e-3) / (clk * 1e3) / 148, clk / 1000);
                }
            }
        }
    }
    return 0;
}
