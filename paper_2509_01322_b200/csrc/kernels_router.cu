// kernels_router.cu -- exact-order fp32 kernels for the router path.
//
// Everything here reproduces the reference's fp32 arithmetic bit for bit:
// products and sums are separately rounded (__fmul_rn / __fadd_rn, never
// contracted to FMA), reductions run in the reference's index order, and the
// exponential is the glibc-expf restatement in libm_port.h.  The file is also
// compiled with --fmad=false as a second line of defence; the build asserts
// on the SASS that the sequential GEMM's inner loop has no FFMA.
#include <float.h>

#include "internal.cuh"
#include "libm_port.h"

namespace scmoe {

// ---------------------------------------------------------------------------
// rmsnorm forward -- graph.hpp:322-335.  One warp per row; the sum of squares
// is a strictly sequential chain in j (lane 0), the products are computed by
// all lanes.  out = (x * inv) * gain, left to right.
// ---------------------------------------------------------------------------
constexpr int kNormChunk = 1024;

__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x,
                                                      const float* __restrict__ gain, int rows,
                                                      int d, float eps, float* __restrict__ out,
                                                      __nv_bfloat16* __restrict__ out_bf16) {
    __shared__ float sq[8][kNormChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    if (row >= rows) return;
    const float* xr = x + (size_t)row * d;
    float s2 = 0.0f;
    for (int j0 = 0; j0 < d; j0 += kNormChunk) {
        const int n = min(kNormChunk, d - j0);
        for (int j = lane; j < n; j += 32) {
            const float v = xr[j0 + j];
            sq[warp][j] = __fmul_rn(v, v);
        }
        __syncwarp();
        if (lane == 0) {
#pragma unroll 8
            for (int j = 0; j < n; ++j) s2 = __fadd_rn(s2, sq[warp][j]);
        }
        __syncwarp();
    }
    s2 = __shfl_sync(0xffffffffu, s2, 0);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(s2, (float)d), eps)));
    float* orow = out + (size_t)row * d;
    for (int j = lane; j < d; j += 32) {
        const float g = gain ? gain[j] : 1.0f;
        const float v = __fmul_rn(__fmul_rn(xr[j], inv), g);
        orow[j] = v;
        if (out_bf16) out_bf16[(size_t)row * d + j] = __float2bfloat16_rn(v);
    }
}

void launch_rmsnorm(scmoe_ctx* c, const float* x, const float* gain, size_t rows, size_t d,
                    float eps, float* out, __nv_bfloat16* out_bf16) {
    if (rows == 0) return;
    rmsnorm_kernel<<<ceil_div(rows, 8), 256, 0, c->stream>>>(x, gain, (int)rows, (int)d, eps, out,
                                                             out_bf16);
    SCMOE_LAUNCH_CHECK(c);
}

// ---------------------------------------------------------------------------
// Sequential-k GEMM -- tensor.hpp:95-112 (mm_into).  Each output element is
// c = 0; for p ascending: c = c + a[p]*b[p] with both operations rounded.
// Tiles of 64 rows x 64 columns, 256 threads, 4x4 outputs per thread, K
// staged through shared memory in chunks of 32.  Rows can be indirected
// (a_rows) and grouped (tiles: expert, first row, row count), which serves
// both the router projection (one group) and the fp32 expert FFN.
// ---------------------------------------------------------------------------
constexpr int kSeqTM = 64, kSeqTN = 64, kSeqKC = 32, kSeqPad = 4;

template <bool kSilu>
__global__ void __launch_bounds__(256) seq_gemm_kernel(
    const float* __restrict__ A, size_t lda, const int* __restrict__ a_rows,
    const float* __restrict__ B, size_t ldb, size_t b_group_stride, float* __restrict__ C,
    size_t ldc, int K, int N, const TokenTile* __restrict__ tiles, const int* __restrict__ n_tiles_dev,
    int n_tiles_host) {
    __shared__ __align__(16) float As[2][kSeqKC][kSeqTM + kSeqPad];
    __shared__ __align__(16) float Bs[2][kSeqKC][kSeqTN + kSeqPad];

    const int n_tiles = n_tiles_dev ? *n_tiles_dev : n_tiles_host;
    const int col0 = blockIdx.x * kSeqTN;
    const int tid = threadIdx.x;
    const int ty = tid >> 4, tx = tid & 15;

    for (int tile_id = blockIdx.y; tile_id < n_tiles; tile_id += gridDim.y) {
        const TokenTile tile = tiles[tile_id];
        const float* Bg = B + (size_t)tile.e * b_group_stride;
        // Row sources for the A loader: thread loads rows (tid>>3) and (tid>>3)+32.
        const int lr0 = tid >> 3, lk4 = tid & 7;
        const float* arow[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = lr0 + 32 * h;
            if (r < tile.count) {
                const int src = a_rows ? a_rows[tile.pos + r] : tile.pos + r;
                arow[h] = A + (size_t)src * lda;
            } else {
                arow[h] = nullptr;
            }
        }
        // B loader: 32 rows x 64 cols = 512 float4, 2 per thread.
        const int bk = tid >> 4, bc4 = tid & 15;

        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

        auto load_stage = [&](int buf, int k0) {
            const int kc = min(kSeqKC, K - k0);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                const int kk = 4 * lk4;
                if (arow[h]) {
                    if (kk + 3 < kc) {
                        v = *reinterpret_cast<const float4*>(arow[h] + k0 + kk);
                    } else {
                        if (kk + 0 < kc) v.x = arow[h][k0 + kk + 0];
                        if (kk + 1 < kc) v.y = arow[h][k0 + kk + 1];
                        if (kk + 2 < kc) v.z = arow[h][k0 + kk + 2];
                    }
                }
                const int r = lr0 + 32 * h;
                As[buf][kk + 0][r] = v.x;
                As[buf][kk + 1][r] = v.y;
                As[buf][kk + 2][r] = v.z;
                As[buf][kk + 3][r] = v.w;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int k = bk + 16 * h;
                const int col = col0 + 4 * bc4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k < kc) {
                    const float* src = Bg + (size_t)(k0 + k) * ldb + col;
                    if (col + 3 < N && (((uintptr_t)src & 15) == 0)) {
                        v = *reinterpret_cast<const float4*>(src);
                    } else {
                        if (col + 0 < N) v.x = src[0];
                        if (col + 1 < N) v.y = src[1];
                        if (col + 2 < N) v.z = src[2];
                        if (col + 3 < N) v.w = src[3];
                    }
                }
                *reinterpret_cast<float4*>(&Bs[buf][k][4 * bc4]) = v;
            }
        };

        int buf = 0;
        load_stage(0, 0);
        __syncthreads();
        for (int k0 = 0; k0 < K; k0 += kSeqKC) {
            const int kc = min(kSeqKC, K - k0);
            if (k0 + kSeqKC < K) load_stage(buf ^ 1, k0 + kSeqKC);
            if (kc == kSeqKC) {
#pragma unroll 8
                for (int k = 0; k < kSeqKC; ++k) {
                    const float4 a = *reinterpret_cast<const float4*>(&As[buf][k][4 * ty]);
                    const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][k][4 * tx]);
                    const float av[4] = {a.x, a.y, a.z, a.w};
                    const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
                }
            } else {
                for (int k = 0; k < kc; ++k) {
                    const float4 a = *reinterpret_cast<const float4*>(&As[buf][k][4 * ty]);
                    const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][k][4 * tx]);
                    const float av[4] = {a.x, a.y, a.z, a.w};
                    const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
                }
            }
            __syncthreads();
            buf ^= 1;
        }
        // Epilogue.
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = 4 * ty + i;
            if (r >= tile.count) continue;
            float* crow = C + (size_t)(tile.pos + r) * ldc;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int col = col0 + 4 * tx + j;
                if (col < N) crow[col] = kSilu ? scmoe_siluf(acc[i][j]) : acc[i][j];
            }
        }
        __syncthreads();
    }
}

void launch_seq_gemm(scmoe_ctx* c, const float* A, size_t lda, const int* a_rows, const float* B,
                     size_t ldb, size_t b_group_stride, float* C, size_t ldc, size_t K, size_t N,
                     int silu, const TokenTile* tiles, const int* n_tiles_dev, size_t max_tiles) {
    if (max_tiles == 0 || N == 0) return;
    dim3 grid((unsigned)ceil_div(N, kSeqTN), (unsigned)std::min<size_t>(max_tiles, 65535));
    if (silu)
        seq_gemm_kernel<true><<<grid, 256, 0, c->stream>>>(A, lda, a_rows, B, ldb, b_group_stride,
                                                           C, ldc, (int)K, (int)N, tiles,
                                                           n_tiles_dev, (int)max_tiles);
    else
        seq_gemm_kernel<false><<<grid, 256, 0, c->stream>>>(A, lda, a_rows, B, ldb, b_group_stride,
                                                            C, ldc, (int)K, (int)N, tiles,
                                                            n_tiles_dev, (int)max_tiles);
    SCMOE_LAUNCH_CHECK(c);
}

// ---------------------------------------------------------------------------
// Softmax + biased top-K -- tensor.hpp:174-192 and router.hpp:90-130.
// One warp per token.  The row max is order independent; the exponentials
// are elementwise; the normaliser is a sequential sum over j in fp32 (lane 0,
// from shared memory); then every lane divides.  Selection is K rounds of a
// warp arg-max under the reference's strict total order
// (double(p)+b descending, index ascending), which yields exactly the
// sequence std::partial_sort produces.
// ---------------------------------------------------------------------------
struct Cand {
    double s;
    int i;
};
__device__ __forceinline__ bool better(double sa, int ia, double sb, int ib) {
    return sa > sb || (sa == sb && ia < ib);
}

template <typename S, bool kFromLogits>
__global__ void __launch_bounds__(256) softmax_topk_kernel(
    const S* __restrict__ in, int T, int E, int K, int n_ffn, const double* __restrict__ bias,
    uint32_t* __restrict__ idx_out, double* __restrict__ gates_out,
    uint32_t* __restrict__ ffn_out, S* __restrict__ probs_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sbias = reinterpret_cast<double*>(smem_raw);
    S* rows = reinterpret_cast<S*>(smem_raw + sizeof(double) * E);
    unsigned char* taken_all = smem_raw + sizeof(double) * E + sizeof(S) * E * 8;

    for (int j = threadIdx.x; j < E; j += blockDim.x) sbias[j] = bias ? bias[j] : 0.0;
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 8 + warp;
    if (t >= T) return;
    S* p = rows + (size_t)warp * E;
    unsigned char* taken = taken_all + (size_t)warp * E;
    const S* row = in + (size_t)t * E;

    if constexpr (kFromLogits) {
        float mx = -FLT_MAX;
        bool first = true;
        for (int j = lane; j < E; j += 32) {
            const float v = row[j];
            mx = first ? v : (v > mx ? v : mx);
            first = false;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float other = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = other > mx ? other : mx;
        }
        for (int j = lane; j < E; j += 32) p[j] = scmoe_expf(__fsub_rn(row[j], mx));
        __syncwarp();
        float sum = 0.0f;
        if (lane == 0) {
#pragma unroll 8
            for (int j = 0; j < E; ++j) sum = __fadd_rn(sum, p[j]);
        }
        sum = __shfl_sync(0xffffffffu, sum, 0);
        for (int j = lane; j < E; j += 32) {
            const float q = __fdiv_rn(p[j], sum);
            p[j] = q;
            if (probs_out) probs_out[(size_t)t * E + j] = q;
        }
    } else {
        for (int j = lane; j < E; j += 32) p[j] = row[j];
    }
    for (int j = lane; j < E; j += 32) taken[j] = 0;
    __syncwarp();

    uint32_t ffn = 0;
    for (int s = 0; s < K; ++s) {
        double best_s = 0.0;
        int best_i = INT_MAX;
        for (int j = lane; j < E; j += 32) {
            if (taken[j]) continue;
            const double sc = __dadd_rn((double)p[j], sbias[j]);
            if (best_i == INT_MAX || better(sc, j, best_s, best_i)) {
                best_s = sc;
                best_i = j;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, best_s, o);
            const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            if (oi != INT_MAX && (best_i == INT_MAX || better(os, oi, best_s, best_i))) {
                best_s = os;
                best_i = oi;
            }
        }
        if (lane == 0) {
            idx_out[(size_t)t * K + s] = (uint32_t)best_i;
            gates_out[(size_t)t * K + s] = (double)p[best_i];
            taken[best_i] = 1;
        }
        ffn += best_i < n_ffn ? 1u : 0u;
        __syncwarp();
    }
    if (lane == 0) ffn_out[t] = ffn;
}

template <typename S, bool kFromLogits>
static void launch_topk_impl(scmoe_ctx* c, const S* in, size_t T, size_t E, size_t K,
                             size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                             uint32_t* ffn, S* probs) {
    if (T == 0) return;
    const size_t smem = sizeof(double) * E + sizeof(S) * E * 8 + E * 8;
    SCMOE_CHECK_ARG(smem <= 200 * 1024, SCMOE_ERR_CONFIG, "router: too many experts for top-k kernel");
    auto kern = softmax_topk_kernel<S, kFromLogits>;
    if (smem > 48 * 1024)
        SCMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<ceil_div(T, 8), 256, smem, c->stream>>>(in, (int)T, (int)E, (int)K, (int)n_ffn, bias,
                                                   idx, gates, ffn, probs);
    SCMOE_LAUNCH_CHECK(c);
}

void launch_softmax_topk(scmoe_ctx* c, const float* logits, size_t T, size_t E, size_t K,
                         size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                         uint32_t* ffn_count, float* probs_out) {
    launch_topk_impl<float, true>(c, logits, T, E, K, n_ffn, bias, idx, gates, ffn_count, probs_out);
}
void launch_topk_from_probs_f32(scmoe_ctx* c, const float* probs, size_t T, size_t E, size_t K,
                                size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                                uint32_t* ffn_count) {
    launch_topk_impl<float, false>(c, probs, T, E, K, n_ffn, bias, idx, gates, ffn_count,
                                   (float*)nullptr);
}
void launch_topk_from_probs_f64(scmoe_ctx* c, const double* probs, size_t T, size_t E, size_t K,
                                size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                                uint32_t* ffn_count) {
    launch_topk_impl<double, false>(c, probs, T, E, K, n_ffn, bias, idx, gates, ffn_count,
                                    (double*)nullptr);
}

__global__ void debug_expf_kernel(const float* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = scmoe_expf(in[i]);
}

__global__ void debug_expf_range_kernel(uint32_t first, float* __restrict__ out, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = scmoe_expf(__uint_as_float(first + (uint32_t)i));
}

void launch_debug_expf(scmoe_ctx* c, const float* in, float* out, size_t n) {
    if (n == 0) return;
    debug_expf_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(in, out, n);
    SCMOE_LAUNCH_CHECK(c);
}
void launch_debug_expf_range(scmoe_ctx* c, uint32_t first, float* out, size_t n) {
    if (n == 0) return;
    debug_expf_range_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(first, out, n);
    SCMOE_LAUNCH_CHECK(c);
}

}  // namespace scmoe
