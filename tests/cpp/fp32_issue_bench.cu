// Microbenchmark (not product code): throughput of the exact-order
// multiply-then-add chains the router needs, in three instruction mixes.
//   A: scalar FMUL + FADD               (current router kernels)
//   B: packed FMUL2 (mul.rn.f32x2) + scalar FADD
//   C: packed FMUL2 + packed FADD2      (exact only if ptxas keeps them separate)
//   D: scalar FFMA                      (inexact; pipe reference)
// Each thread runs 7x8 independent accumulator chains like router_slab_kernel.
// Prints lane-ops (mul + add counted separately) per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TOK = 7, EXP = 8;

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

template <int MODE>
__global__ void __launch_bounds__(768, 1) chains(const float* __restrict__ xs_g,
                                                 const float* __restrict__ ws_g, int K,
                                                 float* __restrict__ out) {
    __shared__ float xs[8][64];
    __shared__ float ws[8][768];
    for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) (&xs[0][0])[i] = xs_g[i];
    for (int i = threadIdx.x; i < 8 * 768; i += blockDim.x) (&ws[0][0])[i] = ws_g[i];
    __syncthreads();
    const int tg = threadIdx.x / 96, eg = threadIdx.x % 96;
    float acc[TOK][EXP];
#pragma unroll
    for (int i = 0; i < TOK; ++i)
#pragma unroll
        for (int j = 0; j < EXP; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += 8) {
#pragma unroll 4
        for (int k = 0; k < 8; ++k) {
            const float4 a03 = *reinterpret_cast<const float4*>(&xs[k][8 * tg]);
            const float2 a45 = *reinterpret_cast<const float2*>(&xs[k][8 * tg + 4]);
            const float a6 = xs[k][8 * tg + 6];
            const float4 b03 = *reinterpret_cast<const float4*>(&ws[k][8 * eg]);
            const float4 b47 = *reinterpret_cast<const float4*>(&ws[k][8 * eg + 4]);
            const float av[7] = {a03.x, a03.y, a03.z, a03.w, a45.x, a45.y, a6};
            const float bv[8] = {b03.x, b03.y, b03.z, b03.w, b47.x, b47.y, b47.z, b47.w};
            if constexpr (MODE == 0) {
#pragma unroll
                for (int i = 0; i < TOK; ++i)
#pragma unroll
                    for (int j = 0; j < EXP; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
            } else if constexpr (MODE == 1 || MODE == 2) {
#pragma unroll
                for (int i = 0; i < TOK; ++i) {
                    const unsigned long long aa = pack2(av[i], av[i]);
#pragma unroll
                    for (int j = 0; j < EXP; j += 2) {
                        const unsigned long long p = fmul2(aa, pack2(bv[j], bv[j + 1]));
                        if constexpr (MODE == 1) {
                            float p0, p1;
                            unpack2(p, p0, p1);
                            acc[i][j] = __fadd_rn(acc[i][j], p0);
                            acc[i][j + 1] = __fadd_rn(acc[i][j + 1], p1);
                        } else {
                            const unsigned long long s = fadd2(pack2(acc[i][j], acc[i][j + 1]), p);
                            unpack2(s, acc[i][j], acc[i][j + 1]);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < TOK; ++i)
#pragma unroll
                    for (int j = 0; j < EXP; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < TOK; ++i)
#pragma unroll
        for (int j = 0; j < EXP; ++j) s += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, const float* xs, const float* ws, float* out, int K, int sms,
         double clk_ghz) {
    chains<MODE><<<sms, 768>>>(xs, ws, K, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) chains<MODE><<<sms, 768>>>(xs, ws, K, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    const double ops = 2.0 * TOK * EXP * (double)K * 768.0;  // per SM (mul + add)
    const double per_clk = ops / (ms * 1e-3 * clk_ghz * 1e9);
    printf("%-28s %8.3f ms  %6.1f lane-ops/clk/SM  (%s)\n", name, ms, per_clk,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double ghz = clk_khz / 1e6;
    float *xs, *ws, *out;
    cudaMalloc(&xs, 16 * 64 * 4);
    cudaMalloc(&ws, 16 * 768 * 4);
    cudaMalloc(&out, sms * 768 * 4);
    cudaMemset(xs, 0, 16 * 64 * 4);
    cudaMemset(ws, 0, 16 * 768 * 4);
    const int K = 6144 * 4;
    printf("SMs %d, clock %.3f GHz (nominal max)\n", sms, ghz);
    run<0>("A scalar FMUL+FADD", xs, ws, out, K, sms, ghz);
    run<1>("B FMUL2 + scalar FADD", xs, ws, out, K, sms, ghz);
    run<2>("C FMUL2 + FADD2", xs, ws, out, K, sms, ghz);
    run<3>("D FFMA (inexact)", xs, ws, out, K, sms, ghz);
    return 0;
}
