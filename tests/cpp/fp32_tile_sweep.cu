// Microbenchmark (not product code): exact-order FMUL+FADD chains, sweeping
// the per-thread register tile (tokens x experts) and CTA size, with operands
// streamed from shared memory as in the router kernels.  Reports mul+add
// lane-ops per clock per SM (B200 FP32 lanes: 128/clk/SM).
#include <cstdio>
#include <cuda_runtime.h>

template <int TOK, int EXP, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) chains(const float* __restrict__ g, int K,
                                                     float* __restrict__ out) {
    constexpr int EG = 128;  // expert groups per k row (lanes vary along experts)
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

template <int TOK, int EXP, int THREADS>
void run(const float* g, float* out, int sms, double ghz) {
    const int K = 6144 * 2;
    chains<TOK, EXP, THREADS><<<sms, THREADS>>>(g, K, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) chains<TOK, EXP, THREADS><<<sms, THREADS>>>(g, K, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    const double ops = 2.0 * TOK * EXP * (double)K * THREADS;
    printf("tile %dx%d threads %4d: %7.1f lane-ops/clk/SM  %s\n", TOK, EXP, THREADS,
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
    run<7, 8, 768>(g, out, sms, ghz);
    run<7, 6, 1024>(g, out, sms, ghz);
    run<8, 6, 768>(g, out, sms, ghz);
    run<6, 8, 768>(g, out, sms, ghz);
    run<4, 8, 1024>(g, out, sms, ghz);
    run<8, 4, 1024>(g, out, sms, ghz);
    run<4, 4, 1024>(g, out, sms, ghz);
    run<8, 8, 512>(g, out, sms, ghz);
    run<12, 4, 1024>(g, out, sms, ghz);
    run<10, 6, 768>(g, out, sms, ghz);
    return 0;
}
