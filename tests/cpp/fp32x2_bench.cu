// Microbenchmark (not product code): exact-order multiply-then-add chains with
// packed f32x2 instructions (FMUL2 / FADD2), against the scalar FMUL + FADD
// form the router used first.  Each 2x2 (token pair x expert pair) block
// takes two FMUL2 (straight and expert-swapped operand) and two FADD2 whose
// product operand is half-swapped -- the swap keeps ptxas from contracting
// the pair into FFMA2 (it does contract a plain mul.rn.f32x2 -> add.rn.f32x2,
// even under --fmad=false).  Reports mul+add lane-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 swp(u64 a) {
    u64 r;
    asm("{.reg .b32 l,h; mov.b64 {l,h}, %1; mov.b64 %0, {h,l};}" : "=l"(r) : "l"(a));
    return r;
}

template <int TOK, int EXP, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) pairs(const float* __restrict__ g, int K,
                                                    float* __restrict__ out) {
    constexpr int EG = 128;
    __shared__ __align__(16) float xs[8][64];
    __shared__ __align__(16) float ws[8][EG * EXP];
    for (int i = threadIdx.x; i < 8 * 64; i += THREADS) (&xs[0][0])[i] = g[i % 1024];
    for (int i = threadIdx.x; i < 8 * EG * EXP; i += THREADS) (&ws[0][0])[i] = g[i % 1024];
    __syncthreads();
    const int tg = (threadIdx.x / EG) % 8, eg = threadIdx.x % EG;
    u64 accA[TOK / 2][EXP / 2], accB[TOK / 2][EXP / 2];
#pragma unroll
    for (int i = 0; i < TOK / 2; ++i)
#pragma unroll
        for (int j = 0; j < EXP / 2; ++j) accA[i][j] = accB[i][j] = 0;
    for (int k0 = 0; k0 < K; k0 += 8) {
#pragma unroll 4
        for (int k = 0; k < 8; ++k) {
            u64 av[TOK / 2], bv[EXP / 2];
#pragma unroll
            for (int i = 0; i < TOK / 2; ++i)
                av[i] = *reinterpret_cast<const u64*>(&xs[k][(8 * tg + 2 * i) % 64]);
#pragma unroll
            for (int j = 0; j < EXP / 2; ++j)
                bv[j] = *reinterpret_cast<const u64*>(&ws[k][EXP * eg + 2 * j]);
#pragma unroll
            for (int i = 0; i < TOK / 2; ++i)
#pragma unroll
                for (int j = 0; j < EXP / 2; ++j) {
                    accA[i][j] = add2(accA[i][j], swp(mul2(av[i], bv[j])));
                    accB[i][j] = add2(accB[i][j], swp(mul2(av[i], swp(bv[j]))));
                }
        }
    }
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < TOK / 2; ++i)
#pragma unroll
        for (int j = 0; j < EXP / 2; ++j) s ^= accA[i][j] ^ accB[i][j];
    out[blockIdx.x * THREADS + threadIdx.x] = (float)(s & 0xffff);
}

// Token broadcast: FMUL2 takes one scalar token operand against an expert pair.
__device__ __forceinline__ u64 dup(float x) {
    u64 r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
    return r;
}
template <int TOK, int EXP, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) bcast(const float* __restrict__ g, int K,
                                                    float* __restrict__ out) {
    constexpr int EG = 96;
    __shared__ __align__(16) float xs[8][64];
    __shared__ __align__(16) float ws[8][EG * EXP];
    for (int i = threadIdx.x; i < 8 * 64; i += THREADS) (&xs[0][0])[i] = g[i % 1024];
    for (int i = threadIdx.x; i < 8 * EG * EXP; i += THREADS) (&ws[0][0])[i] = g[i % 1024];
    __syncthreads();
    const int tg = (threadIdx.x / EG) % 8, eg = threadIdx.x % EG;
    u64 acc[TOK][EXP / 2];
#pragma unroll
    for (int i = 0; i < TOK; ++i)
#pragma unroll
        for (int j = 0; j < EXP / 2; ++j) acc[i][j] = 0;
    for (int k0 = 0; k0 < K; k0 += 8) {
#pragma unroll 4
        for (int k = 0; k < 8; ++k) {
            float av[TOK];
            u64 bv[EXP / 2];
#pragma unroll
            for (int i = 0; i < TOK; ++i) av[i] = xs[k][(8 * tg + i) % 64];
#pragma unroll
            for (int j = 0; j < EXP / 4; ++j) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&ws[k][(EG * 4) * j + 4 * eg]);
                bv[2 * j] = v.x;
                bv[2 * j + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < TOK; ++i)
#pragma unroll
                for (int j = 0; j < EXP / 2; ++j)
                    acc[i][j] = add2(acc[i][j], swp(mul2(dup(av[i]), bv[j])));
        }
    }
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < TOK; ++i)
#pragma unroll
        for (int j = 0; j < EXP / 2; ++j) s ^= acc[i][j];
    out[blockIdx.x * THREADS + threadIdx.x] = (float)(s & 0xffff);
}

template <int TOK, int EXP, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) scalar(const float* __restrict__ g, int K,
                                                     float* __restrict__ out) {
    constexpr int EG = 128;
    __shared__ __align__(16) float xs[8][64];
    __shared__ __align__(16) float ws[8][EG * EXP];
    for (int i = threadIdx.x; i < 8 * 64; i += THREADS) (&xs[0][0])[i] = g[i % 1024];
    for (int i = threadIdx.x; i < 8 * EG * EXP; i += THREADS) (&ws[0][0])[i] = g[i % 1024];
    __syncthreads();
    const int tg = (threadIdx.x / EG) % 8, eg = threadIdx.x % EG;
    float acc[TOK][EXP];
#pragma unroll
    for (int i = 0; i < TOK; ++i)
#pragma unroll
        for (int j = 0; j < EXP; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += 8) {
#pragma unroll 4
        for (int k = 0; k < 8; ++k) {
            float av[TOK], bv[EXP];
#pragma unroll
            for (int i = 0; i < TOK; ++i) av[i] = xs[k][(8 * tg + i) % 64];
#pragma unroll
            for (int j = 0; j < EXP; ++j) bv[j] = ws[k][EXP * eg + j];
#pragma unroll
            for (int i = 0; i < TOK; ++i)
#pragma unroll
                for (int j = 0; j < EXP; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < TOK; ++i)
#pragma unroll
        for (int j = 0; j < EXP; ++j) s += acc[i][j];
    out[blockIdx.x * THREADS + threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F kern, int tok, int exp, int threads, const float* g, float* out,
         int sms, double ghz) {
    const int K = 6144 * 2;
    kern<<<sms, threads>>>(g, K, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<sms, threads>>>(g, K, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    const double ops = 2.0 * tok * exp * (double)K * threads;
    printf("%-7s tile %dx%d threads %4d: %7.1f lane-ops/clk/SM  %s\n", name, tok, exp, threads,
           ops / (ms * 1e-3 * ghz * 1e9), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ghz = clk / 1e6;
    float *g, *out;
    cudaMalloc(&g, 4096);
    cudaMemset(g, 0, 4096);
    cudaMalloc(&out, sms * 1024 * 4);
    run("scalar", scalar<7, 8, 768>, 7, 8, 768, g, out, sms, ghz);
    run("bcast", bcast<7, 8, 768>, 7, 8, 768, g, out, sms, ghz);
    run("f32x2", pairs<8, 8, 512>, 8, 8, 512, g, out, sms, ghz);
    run("f32x2", pairs<8, 6, 768>, 8, 6, 768, g, out, sms, ghz);
    run("f32x2", pairs<6, 8, 768>, 6, 8, 768, g, out, sms, ghz);
    run("f32x2", pairs<4, 8, 1024>, 4, 8, 1024, g, out, sms, ghz);
    run("f32x2", pairs<8, 4, 1024>, 8, 4, 1024, g, out, sms, ghz);
    run("f32x2", pairs<4, 4, 1024>, 4, 4, 1024, g, out, sms, ghz);
    run("f32x2", pairs<8, 8, 768>, 8, 8, 768, g, out, sms, ghz);
    run("f32x2", pairs<6, 6, 1024>, 6, 6, 1024, g, out, sms, ghz);
    return 0;
}
