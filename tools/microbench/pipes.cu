// Microbenchmark: FP32-pipe issue cost per SMSP of the instruction forms the
// fused step uses, measured in SM cycles (clock64 inside the kernel, so the
// result does not depend on the clock the GPU runs at).  Not product code:
// it fixes the per-instruction costs the DESIGN.md ceiling is derived from.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
//
// One CTA per SM (grid = #SMs, 100 KB of dynamic shared memory keeps a second
// CTA off the SM), W warps per CTA, NCH independent accumulator chains per
// thread whose operands are all per-thread registers (no uniform-register or
// immediate forms).  Reported: cycles per warp-instruction per SMSP of the
// instruction group under test (SM cycles / (W/4 warps x groups)).
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int NCH = 8;
constexpr int ITERS = 4096;

template <int MODE>
__global__ void kern(float *out, long long *cyc, const float *seed) {
    float2 a[NCH], b[NCH], u[NCH];
    float s[NCH], t[NCH];
    unsigned iv[NCH], jv[NCH];
    const float sd = seed[threadIdx.x & 31];
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
        a[i] = make_float2(sd * 1e-3f + i, sd * 0.5f - i);
        b[i] = make_float2(sd * 2e-3f - i, sd * 0.25f + i);
        u[i] = make_float2(1.0001f + sd * 1e-4f * i, 0.9999f - sd * 1e-4f * i);
        s[i] = sd * (i + 1) - 3.0f;
        t[i] = sd * (i + 2) + 1.0f;
        iv[i] = (unsigned)(sd * 1000.f) + i;
        jv[i] = (unsigned)(sd * 777.f) * 3u + i;
    }
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            // u, s, t are loop-carried so they stay in ordinary registers
            if (MODE == 0) {  // FFMA2 reg pair * reg pair + pair
                a[i] = __ffma2_rn(u[i], b[i], a[i]);
            } else if (MODE == 1) {  // FFMA2 pair * {|s|,|s|} + pair (Eq. 5 form)
                const float g = fabsf(s[i]);
                a[i] = __ffma2_rn(u[i], make_float2(g, g), a[i]);
            } else if (MODE == 2) {  // scalar FFMA, 3 registers
                s[i] = fmaf(a[i].x, t[i], s[i]);
            } else if (MODE == 3) {  // FADD2
                a[i] = __fadd2_rn(a[i], u[i]);
            } else if (MODE == 4) {  // scalar FADD
                s[i] = s[i] + t[i];
            } else if (MODE == 5) {  // FFMA2 and an independent scalar FFMA
                a[i] = __ffma2_rn(u[i], b[i], a[i]);
                s[i] = fmaf(b[i].x, t[i], s[i]);
            } else if (MODE == 6) {  // FFMA2 and an independent FADD
                a[i] = __ffma2_rn(u[i], b[i], a[i]);
                s[i] = s[i] + t[i];
            } else if (MODE == 7) {  // FFMA2 and an independent ALU op (IADD3)
                a[i] = __ffma2_rn(u[i], b[i], a[i]);
                iv[i] = iv[i] + jv[i] + 7u;
            } else if (MODE == 8) {  // FFMA2 and an independent FMNMX (ALU)
                a[i] = __ffma2_rn(u[i], b[i], a[i]);
                s[i] = fmaxf(s[i], t[i]);
            } else if (MODE == 9) {  // two scalar FFMA (H of clusters 0, 1 unpacked)
                s[i] = fmaf(a[i].x, t[i], s[i]);
                t[i] = fmaf(a[i].y, s[(i + 1) % NCH], t[i]);
            } else if (MODE == 10) {  // dependent FFMA2 chain (latency, chain 0 only)
                if (i == 0) {
#pragma unroll
                    for (int k = 0; k < NCH; ++k) a[0] = __ffma2_rn(u[k], b[k], a[0]);
                }
            } else if (MODE == 11) {  // dependent scalar FFMA chain (latency)
                if (i == 0) {
#pragma unroll
                    for (int k = 0; k < NCH; ++k) s[0] = fmaf(a[k].x, t[k], s[0]);
                }
            } else if (MODE == 12) {  // scalar FMUL
                s[i] = s[i] * t[i];
            } else if (MODE == 13) {  // FFMA2 + FFMA2 + FFMA (complement-class Eq. 5, 3 clusters + G)
                const float g = fabsf(s[i]);
                a[i] = __ffma2_rn(u[i], make_float2(g, g), a[i]);
                t[i] = fmaf(b[i].x, g, t[i]);
            }
        }
    }
    const long long t1 = clock64();
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < NCH; ++i) r += a[i].x + a[i].y + s[i] + t[i] + u[i].x + (float)(iv[i] & 1u);
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
static void run(const char *name, int W, float *out, long long *dcyc, const float *seed, int nsm) {
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long h[1024];
    for (int rep = 0; rep < 2; ++rep) {
        kern<MODE><<<nsm, 32 * W, smem>>>(out, dcyc, seed);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(h, dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int b = 0; b < nsm; ++b) mean += h[b];
    mean /= nsm;
    const double groups = (W / 4.0) * NCH * (double)ITERS;  // per SMSP
    printf("%-44s W %2d  cyc/group/SMSP %.3f\n", name, W, mean / groups);
}

int main() {
    float *out, *seed;
    long long *dcyc;
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&out, nsm * 1024 * sizeof(float));
    cudaMalloc(&seed, 32 * sizeof(float));
    float hs[32];
    for (int i = 0; i < 32; ++i) hs[i] = 0.5f + 0.01f * i;
    cudaMemcpy(seed, hs, sizeof(hs), cudaMemcpyHostToDevice);
    cudaMalloc(&dcyc, nsm * sizeof(long long));
    for (int W : {4, 8, 16, 32}) {
        run<0>("FFMA2 r*r+r", W, out, dcyc, seed, nsm);
        run<1>("FFMA2 r*|bcast|+r", W, out, dcyc, seed, nsm);
        run<2>("FFMA r*r+r", W, out, dcyc, seed, nsm);
        run<9>("2 x FFMA r*r+r", W, out, dcyc, seed, nsm);
        run<12>("FMUL", W, out, dcyc, seed, nsm);
        run<3>("FADD2", W, out, dcyc, seed, nsm);
        run<4>("FADD", W, out, dcyc, seed, nsm);
        run<5>("FFMA2 + FFMA", W, out, dcyc, seed, nsm);
        run<6>("FFMA2 + FADD", W, out, dcyc, seed, nsm);
        run<7>("FFMA2 + IADD3", W, out, dcyc, seed, nsm);
        run<8>("FFMA2 + FMNMX", W, out, dcyc, seed, nsm);
        run<10>("FFMA2 dependent (per instr)", W, out, dcyc, seed, nsm);
        run<11>("FFMA dependent (per instr)", W, out, dcyc, seed, nsm);
    }
    return 0;
}
