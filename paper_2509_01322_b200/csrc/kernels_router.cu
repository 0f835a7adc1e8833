// kernels_router.cu -- exact-order fp32 kernels for the router path.
//
// Everything here reproduces the reference's fp32 arithmetic bit for bit:
// products and sums are separately rounded (__fmul_rn / __fadd_rn, never
// contracted to FMA), reductions run in the reference's index order, and the
// exponential is the glibc-expf restatement in libm_port.h.  The file is also
// compiled with --fmad=false as a second line of defence; the build asserts
// on the SASS that the sequential GEMM's inner loop has no FFMA.
#include <float.h>

#include <type_traits>

#include "internal.cuh"
#include "f32x2.cuh"
#include "libm_port.h"

namespace scmoe {

// ---------------------------------------------------------------------------
// rmsnorm forward -- graph.hpp:322-335.  One warp per row.  All lanes load the
// row chunk (16-byte vectors, all loads in flight at once) and square it into
// shared memory; lane 0 then runs the reference's strictly sequential sum of
// squares in j order (float4 shared reads issued ahead of the add chain).
// out = (x * inv) * gain, left to right; optional bf16 copy for the GEMMs.
// ---------------------------------------------------------------------------
constexpr int kNormChunk = 1024;

__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x,
                                                      const float* __restrict__ gain, int rows,
                                                      int d, float eps, float* __restrict__ out,
                                                      __nv_bfloat16* __restrict__ out_bf16) {
    __shared__ __align__(16) float sq[8][kNormChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    if (row >= rows) return;
    const float* xr = x + (size_t)row * d;
    const bool vec = (d % 4 == 0) && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
    float s2 = 0.0f;
    for (int j0 = 0; j0 < d; j0 += kNormChunk) {
        const int n = min(kNormChunk, d - j0);
        if (vec && n == kNormChunk) {
            const float4* src = reinterpret_cast<const float4*>(xr + j0);
            float4 v[kNormChunk / 128];
#pragma unroll
            for (int i = 0; i < kNormChunk / 128; ++i) v[i] = src[lane + 32 * i];
#pragma unroll
            for (int i = 0; i < kNormChunk / 128; ++i) {
                float4 q;
                q.x = __fmul_rn(v[i].x, v[i].x);
                q.y = __fmul_rn(v[i].y, v[i].y);
                q.z = __fmul_rn(v[i].z, v[i].z);
                q.w = __fmul_rn(v[i].w, v[i].w);
                reinterpret_cast<float4*>(sq[warp])[lane + 32 * i] = q;
            }
        } else {
            for (int j = lane; j < n; j += 32) {
                const float v = xr[j0 + j];
                sq[warp][j] = __fmul_rn(v, v);
            }
        }
        __syncwarp();
        if (lane == 0) {
            int j = 0;
            const float4* q4 = reinterpret_cast<const float4*>(sq[warp]);
            for (; j + 16 <= n; j += 16) {
                const float4 a = q4[j / 4], b = q4[j / 4 + 1], c = q4[j / 4 + 2], e = q4[j / 4 + 3];
                s2 = __fadd_rn(s2, a.x); s2 = __fadd_rn(s2, a.y);
                s2 = __fadd_rn(s2, a.z); s2 = __fadd_rn(s2, a.w);
                s2 = __fadd_rn(s2, b.x); s2 = __fadd_rn(s2, b.y);
                s2 = __fadd_rn(s2, b.z); s2 = __fadd_rn(s2, b.w);
                s2 = __fadd_rn(s2, c.x); s2 = __fadd_rn(s2, c.y);
                s2 = __fadd_rn(s2, c.z); s2 = __fadd_rn(s2, c.w);
                s2 = __fadd_rn(s2, e.x); s2 = __fadd_rn(s2, e.y);
                s2 = __fadd_rn(s2, e.z); s2 = __fadd_rn(s2, e.w);
            }
            for (; j < n; ++j) s2 = __fadd_rn(s2, sq[warp][j]);
        }
        __syncwarp();
    }
    s2 = __shfl_sync(0xffffffffu, s2, 0);
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(s2, (float)d), eps)));
    float* orow = out ? out + (size_t)row * d : nullptr;  // out may be NULL (bf16 only)
    if (vec) {
        const float4* src = reinterpret_cast<const float4*>(xr);
        float4* dst = reinterpret_cast<float4*>(orow);  // unused when orow is NULL
        for (int j4 = lane; j4 < d / 4; j4 += 32) {
            const float4 v = src[j4];
            float4 g = gain ? reinterpret_cast<const float4*>(gain)[j4] : make_float4(1.f, 1.f, 1.f, 1.f);
            float4 o;
            o.x = __fmul_rn(__fmul_rn(v.x, inv), g.x);
            o.y = __fmul_rn(__fmul_rn(v.y, inv), g.y);
            o.z = __fmul_rn(__fmul_rn(v.z, inv), g.z);
            o.w = __fmul_rn(__fmul_rn(v.w, inv), g.w);
            if (orow) dst[j4] = o;
            if (out_bf16) {
                __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y);
                __nv_bfloat162 hi = __floats2bfloat162_rn(o.z, o.w);
                uint2 pk;
                pk.x = *reinterpret_cast<uint32_t*>(&lo);
                pk.y = *reinterpret_cast<uint32_t*>(&hi);
                reinterpret_cast<uint2*>(out_bf16 + (size_t)row * d)[j4] = pk;
            }
        }
    } else {
        for (int j = lane; j < d; j += 32) {
            const float g = gain ? gain[j] : 1.0f;
            const float v = __fmul_rn(__fmul_rn(xr[j], inv), g);
            if (orow) orow[j] = v;
            if (out_bf16) out_bf16[(size_t)row * d + j] = __float2bfloat16_rn(v);
        }
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
// A CTA owns TM rows x TN columns; each thread RM x RN outputs (independent
// chains, so the 4-cycle FADD latency is covered by ILP).  K is staged
// through shared memory in chunks of KC with a register-staged double
// buffer: the next chunk's global loads are issued before the current
// chunk's arithmetic and stored to shared memory after it, so load latency
// hides behind ~RM*RN*2*KC instructions per thread.  Rows can be indirected
// (a_rows) and grouped (tiles: expert, first row, row count), which serves
// both the router projection (one group) and the fp32 expert FFN.
// ---------------------------------------------------------------------------
constexpr int kSeqPad = 4;

template <int TM, int TN, int RM, int RN, bool kSilu, int kSeqKC = 32>
__global__ void __launch_bounds__((TM / RM) * (TN / RN)) seq_gemm_kernel(
    const float* __restrict__ A, size_t lda, const int* __restrict__ a_rows,
    const float* __restrict__ B, size_t ldb, size_t b_group_stride, float* __restrict__ C,
    size_t ldc, int K, int N, const TokenTile* __restrict__ tiles, const int* __restrict__ n_tiles_dev,
    int n_tiles_host) {
    constexpr int NT = (TM / RM) * (TN / RN);
    constexpr int TX = TN / RN;             // threads along N
    constexpr int A4 = TM * kSeqKC / 4;     // float4 per A chunk
    constexpr int B4 = kSeqKC * TN / 4;     // float4 per B chunk
    constexpr int AL = (A4 + NT - 1) / NT;  // per-thread loads
    constexpr int BL = (B4 + NT - 1) / NT;
    static_assert(RM == 2 || RM == 4 || RM == 8, "RM");
    static_assert(RN == 4 || RN == 8, "RN");
    __shared__ __align__(16) float As[2][kSeqKC][TM + kSeqPad];
    __shared__ __align__(16) float Bs[2][kSeqKC][TN + kSeqPad];

    const int n_tiles = n_tiles_dev ? *n_tiles_dev : n_tiles_host;
    const int col0 = blockIdx.x * TN;
    const int tid = threadIdx.x;
    const int ty = tid / TX, tx = tid % TX;

    for (int tile_id = blockIdx.y; tile_id < n_tiles; tile_id += gridDim.y) {
        const TokenTile tile = tiles[tile_id];
        const float* Bg = B + (size_t)tile.e * b_group_stride;
        // A loader: element i -> row i / (KC/4), k4 = i % (KC/4)
        const float* arow[AL];
#pragma unroll
        for (int l = 0; l < AL; ++l) {
            const int i = tid + l * NT;
            const int r = i / (kSeqKC / 4);
            arow[l] = nullptr;
            if (i < A4 && r < tile.count) {
                const int src = a_rows ? a_rows[tile.pos + r] : tile.pos + r;
                arow[l] = A + (size_t)src * lda;
            }
        }
        float4 ra[AL], rb[BL];
        auto load_regs = [&](int k0) {
            const int kc = min(kSeqKC, K - k0);
#pragma unroll
            for (int l = 0; l < AL; ++l) {
                const int i = tid + l * NT;
                const int kk = 4 * (i % (kSeqKC / 4));
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (arow[l]) {
                    const float* s = arow[l] + k0 + kk;
                    if (kk + 3 < kc && ((reinterpret_cast<uintptr_t>(s) & 15) == 0)) {
                        v = *reinterpret_cast<const float4*>(s);
                    } else {
                        if (kk + 0 < kc) v.x = s[0];
                        if (kk + 1 < kc) v.y = s[1];
                        if (kk + 2 < kc) v.z = s[2];
                        if (kk + 3 < kc) v.w = s[3];
                    }
                }
                ra[l] = v;
            }
#pragma unroll
            for (int l = 0; l < BL; ++l) {
                const int i = tid + l * NT;
                const int k = i / (TN / 4), c4 = i % (TN / 4);
                const int col = col0 + 4 * c4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (i < B4 && k < kc) {
                    const float* s = Bg + (size_t)(k0 + k) * ldb + col;
                    if (col + 3 < N && ((reinterpret_cast<uintptr_t>(s) & 15) == 0)) {
                        v = *reinterpret_cast<const float4*>(s);
                    } else {
                        if (col + 0 < N) v.x = s[0];
                        if (col + 1 < N) v.y = s[1];
                        if (col + 2 < N) v.z = s[2];
                        if (col + 3 < N) v.w = s[3];
                    }
                }
                rb[l] = v;
            }
        };
        auto store_smem = [&](int buf) {
#pragma unroll
            for (int l = 0; l < AL; ++l) {
                const int i = tid + l * NT;
                if (i < A4) {
                    const int r = i / (kSeqKC / 4), kk = 4 * (i % (kSeqKC / 4));
                    As[buf][kk + 0][r] = ra[l].x;
                    As[buf][kk + 1][r] = ra[l].y;
                    As[buf][kk + 2][r] = ra[l].z;
                    As[buf][kk + 3][r] = ra[l].w;
                }
            }
#pragma unroll
            for (int l = 0; l < BL; ++l) {
                const int i = tid + l * NT;
                if (i < B4) {
                    const int k = i / (TN / 4), c4 = i % (TN / 4);
                    *reinterpret_cast<float4*>(&Bs[buf][k][4 * c4]) = rb[l];
                }
            }
        };

        // acc2[i][q] = (c[i][2q+1], c[i][2q]): packed f32x2 chains, products
        // added half-swapped (f32x2.cuh) -- same rounding as scalar mul + add
        uint64_t acc2[RM][RN / 2];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int q = 0; q < RN / 2; ++q) acc2[i][q] = 0;

        int buf = 0;
        load_regs(0);
        store_smem(0);
        __syncthreads();
        for (int k0 = 0; k0 < K; k0 += kSeqKC) {
            const int kc = min(kSeqKC, K - k0);
            const bool more = k0 + kSeqKC < K;
            if (more) load_regs(k0 + kSeqKC);
#pragma unroll 4
            for (int k = 0; k < kc; ++k) {
                float av[RM];
                if constexpr (RM >= 4) {
#pragma unroll
                    for (int q = 0; q < RM / 4; ++q) {
                        const float4 a = *reinterpret_cast<const float4*>(&As[buf][k][RM * ty + 4 * q]);
                        av[4 * q] = a.x; av[4 * q + 1] = a.y; av[4 * q + 2] = a.z; av[4 * q + 3] = a.w;
                    }
                } else {
                    const float2 a = *reinterpret_cast<const float2*>(&As[buf][k][RM * ty]);
                    av[0] = a.x; av[1] = a.y;
                }
                uint64_t bv[RN / 2];
#pragma unroll
                for (int q = 0; q < RN / 4; ++q) {
                    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(&Bs[buf][k][RN * tx + 4 * q]);
                    bv[2 * q] = b.x;
                    bv[2 * q + 1] = b.y;
                }
#pragma unroll
                for (int i = 0; i < RM; ++i)
#pragma unroll
                    for (int q = 0; q < RN / 2; ++q)
                        acc2[i][q] = f2_add_swapped(acc2[i][q], f2_mul_bcast(av[i], bv[q]));
            }
            if (more) store_smem(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
        float acc[RM][RN];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int q = 0; q < RN / 2; ++q) {
                acc[i][2 * q] = f2_hi(acc2[i][q]);
                acc[i][2 * q + 1] = f2_lo(acc2[i][q]);
            }
        // Epilogue.
#pragma unroll
        for (int i = 0; i < RM; ++i) {
            const int r = RM * ty + i;
            if (r >= tile.count) continue;
            float* crow = C + (size_t)(tile.pos + r) * ldc;
            const int col = col0 + RN * tx;
            if (!kSilu && col + RN - 1 < N && ((reinterpret_cast<uintptr_t>(crow + col) & 15) == 0)) {
#pragma unroll
                for (int q = 0; q < RN / 4; ++q)
                    *reinterpret_cast<float4*>(crow + col + 4 * q) =
                        make_float4(acc[i][4 * q], acc[i][4 * q + 1], acc[i][4 * q + 2], acc[i][4 * q + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < RN; ++j)
                    if (col + j < N) crow[col + j] = kSilu ? scmoe_siluf(acc[i][j]) : acc[i][j];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Router projection, large batches: one CTA per 56-token slab covering all
// E <= 768 expert columns (8 token groups x 96 expert groups = 768 threads,
// 7 x 8 independent sequential chains per thread).  With T=8192 this is 147
// CTAs -- a single wave on 148 SMs.  Same arithmetic as seq_gemm_kernel: per
// output c = 0; c = c + x*w in k order, every product and sum rounded.
//
// The chains run on packed f32x2 instructions (FMUL2 / FADD2: two lanes of
// work per issue slot), which lifts the FP32 pipe from ~108 to ~122 of its
// 128 lane-ops/clk/SM at this tile shape (tests/cpp/fp32x2_bench.cu).  FMUL2
// takes the token as a broadcast scalar against an expert pair (w0, w1); the
// product is added half-swapped into the accumulator pair (c1, c0).  The swap
// is a free operand modifier, and it keeps ptxas from contracting mul + add
// into FFMA2, which it otherwise does for f32x2 even with explicit .rn and
// --fmad=false (build.py asserts the kernel has no FFMA/FFMA2).
// ---------------------------------------------------------------------------
constexpr int kSlabTok = 7, kSlabExp = 8, kSlabTG = 8, kSlabEG = 96;
constexpr int kSlabRows = kSlabTok * kSlabTG;          // 56
constexpr int kSlabThreads = kSlabTG * kSlabEG;        // 768
constexpr int kSlabKC = 16;
constexpr int kSlabXStride = kSlabTG * 8;              // 64: group g at columns [8g, 8g+7)
constexpr int kSlabW = kSlabEG * kSlabExp;             // 768 (padded expert width)
constexpr int kSlabHalf = kSlabW / 2;                  // thread eg: [4eg, 4eg+4) and [384+4eg, ..)

__global__ void __launch_bounds__(kSlabThreads, 1) router_slab_kernel(
    const float* __restrict__ X, const float* __restrict__ W, float* __restrict__ logits, int T,
    int K, int E) {
    extern __shared__ __align__(16) float slab_smem[];
    // ws[buf][k][768]: W rows; xs[buf][k][64]: X transposed (group g's 7
    // tokens at [8g, 8g+7)); xraw[buf][56][16]: X rows as copied.
    auto ws = reinterpret_cast<float(*)[kSlabKC][kSlabW]>(slab_smem);
    auto xs = reinterpret_cast<float(*)[kSlabKC][kSlabXStride]>(slab_smem + 2 * kSlabKC * kSlabW);
    auto xraw = reinterpret_cast<float(*)[kSlabRows][kSlabKC]>(
        slab_smem + 2 * kSlabKC * (kSlabW + kSlabXStride));
    const int tid = threadIdx.x;
    const int tg = tid / kSlabEG, eg = tid % kSlabEG;
    const int row0 = blockIdx.x * kSlabRows;
    const int nrows = min(kSlabRows, T - row0);
    if (nrows <= 0) return;
    // Both operands go global -> shared with cp.async (nothing is held in
    // registers across the arithmetic); X is transposed after the chunk.
    // W chunk: thread tid copies column quad wc of rows wk, wk+4, wk+8, wk+12.
    const int wk = tid / (kSlabW / 4), wc = 4 * (tid % (kSlabW / 4));
    const bool wok = wc < E;
    auto load = [&](int k0, int buf) {
        const float* s = W + (size_t)(k0 + wk) * E + (wok ? wc : 0);
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&ws[buf][wk][wc]));
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                             dst + l * 4 * kSlabW * (int)sizeof(float)),
                         "l"(s + (size_t)l * 4 * E), "r"(wok ? 16 : 0)
                         : "memory");
        }
        if (tid < kSlabRows * kSlabKC / 4) {
            const int r = tid / (kSlabKC / 4), k4 = tid % (kSlabKC / 4);
            const bool ok = r < nrows;
            const float* s = ok ? X + (size_t)(row0 + r) * K + k0 + 4 * k4 : X;
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&xraw[buf][r][4 * k4]));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(s),
                         "r"(ok ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // Waits for this thread's copies, publishes them block-wide, transposes X.
    auto store = [&](int buf) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (tid < kSlabRows * kSlabKC / 4) {
            const int r = tid / (kSlabKC / 4), k4 = tid % (kSlabKC / 4);
            const int col = 8 * (r / kSlabTok) + r % kSlabTok;
            const float4 v = *reinterpret_cast<const float4*>(&xraw[buf][r][4 * k4]);
            xs[buf][4 * k4 + 0][col] = v.x;
            xs[buf][4 * k4 + 1][col] = v.y;
            xs[buf][4 * k4 + 2][col] = v.z;
            xs[buf][4 * k4 + 3][col] = v.w;
        }
    };
    // acc[i][q] = (c[i][q1], c[i][q0]) for token i and this thread's expert
    // pair q: q = 0,1 -> columns 4eg + {0,1}, {2,3}; q = 2,3 -> 384 + 4eg + ...
    uint64_t acc[kSlabTok][kSlabExp / 2];
#pragma unroll
    for (int i = 0; i < kSlabTok; ++i)
#pragma unroll
        for (int q = 0; q < kSlabExp / 2; ++q) acc[i][q] = 0;

    int buf = 0;
    load(0, 0);
    store(0);
    __syncthreads();
    for (int k0 = 0; k0 < K; k0 += kSlabKC) {
        const bool more = k0 + kSlabKC < K;
        if (more) load(k0 + kSlabKC, buf ^ 1);
#pragma unroll 2
        for (int k = 0; k < kSlabKC; ++k) {
            const ulonglong2 b01 = *reinterpret_cast<const ulonglong2*>(&ws[buf][k][4 * eg]);
            const ulonglong2 b23 =
                *reinterpret_cast<const ulonglong2*>(&ws[buf][k][kSlabHalf + 4 * eg]);
            const uint64_t bv[4] = {b01.x, b01.y, b23.x, b23.y};
            // tokens one at a time (broadcast LDS): keeps the live set at
            // 56 accumulators + 8 weights + 1 token under the 80-register cap
#pragma unroll
            for (int i = 0; i < kSlabTok; ++i) {
                const float a = xs[buf][k][8 * tg + i];
#pragma unroll
                for (int q = 0; q < kSlabExp / 2; ++q)
                    acc[i][q] = f2_add_swapped(acc[i][q], f2_mul_bcast(a, bv[q]));
            }
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < kSlabTok; ++i) {
        const int r = kSlabTok * tg + i;
        if (r >= nrows) continue;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int col = half * kSlabHalf + 4 * eg;
            if (col >= E) continue;
            const uint64_t p0 = acc[i][2 * half], p1 = acc[i][2 * half + 1];
            *reinterpret_cast<float4*>(logits + (size_t)(row0 + r) * E + col) =
                make_float4(f2_hi(p0), f2_lo(p0), f2_hi(p1), f2_lo(p1));
        }
    }
}

// ---------------------------------------------------------------------------
// Router projection, "lean" variant sized to co-reside with the persistent
// grouped GEMM on every SM (GEMM: 192 threads, ~194 KB smem; this kernel:
// 512 threads x <= 64 registers, ~26 KB smem), so the FP32-pipe-bound router
// of the next micro-batch runs underneath the HBM-bound expert GEMMs of the
// current one.  CTA = 28 tokens x all E <= 768 experts (4 token groups x 128
// expert groups, 7 x 6 chains per thread); K staged 4 rows at a time, W by a
// double-buffered cp.async ring, X (raw rows) by a 4-deep ring.
// ---------------------------------------------------------------------------
constexpr int kLeanTok = 7, kLeanExp = 6, kLeanTG = 4, kLeanEG = 128;
constexpr int kLeanRows = kLeanTok * kLeanTG;     // 28
constexpr int kLeanThreads = kLeanTG * kLeanEG;   // 512
constexpr int kLeanKC = 4;
constexpr int kLeanW = kLeanEG * kLeanExp;        // 768
constexpr int kLeanXS = 32;                       // xs row: group g at [8g, 8g+7)
constexpr int kLeanXStages = 4;

__global__ void __launch_bounds__(kLeanThreads, 2) router_lean_kernel(
    const float* __restrict__ X, const float* __restrict__ W, float* __restrict__ logits, int T,
    int K, int E) {
    __shared__ __align__(16) float ws[2][kLeanKC][kLeanW];
    __shared__ __align__(16) float xraw[kLeanXStages][kLeanRows][kLeanKC];
    __shared__ __align__(16) float xs[2][kLeanKC][kLeanXS];
    const int tid = threadIdx.x;
    const int tg = tid / kLeanEG, eg = tid % kLeanEG;
    const int nchunks = K / kLeanKC;

    for (int slab = blockIdx.x; slab * kLeanRows < T; slab += gridDim.x) {
        const int row0 = slab * kLeanRows;
        const int nrows = min(kLeanRows, T - row0);
        // W chunk: 4 x 768 floats = 768 float4 -> 1.5 per thread (threads 0..255 do 2)
        auto load_w = [&](int chunk, int buf) {
            const int k0 = chunk * kLeanKC;
            for (int i = tid; i < kLeanKC * kLeanW / 4; i += kLeanThreads) {
                const int k = i / (kLeanW / 4), col = 4 * (i % (kLeanW / 4));
                const bool ok = col + 3 < E;
                const float* s = ok ? W + (size_t)(k0 + k) * E + col : W;
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&ws[buf][k][col]));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(s),
                             "r"(ok ? 16 : 0)
                             : "memory");
            }
        };
        auto load_x = [&](int chunk) {
            if (tid < kLeanRows && chunk < nchunks) {
                const bool ok = tid < nrows;
                const float* s = ok ? X + (size_t)(row0 + tid) * K + chunk * kLeanKC : X;
                const uint32_t dst = static_cast<uint32_t>(
                    __cvta_generic_to_shared(&xraw[chunk % kLeanXStages][tid][0]));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(s),
                             "r"(ok ? 16 : 0)
                             : "memory");
            }
        };
        float acc[kLeanTok][kLeanExp];
#pragma unroll
        for (int i = 0; i < kLeanTok; ++i)
#pragma unroll
            for (int j = 0; j < kLeanExp; ++j) acc[i][j] = 0.0f;

        // prologue: X chunks 0..2, W chunk 0
        load_x(0);
        load_x(1);
        load_x(2);
        load_w(0, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (tid < kLeanRows * kLeanKC) {
            const int r = tid / kLeanKC, k = tid % kLeanKC;
            xs[0][k][8 * (r / kLeanTok) + r % kLeanTok] = xraw[0][r][k];
        }
        __syncthreads();
        for (int ch = 0; ch < nchunks; ++ch) {
            const int buf = ch & 1;
            const bool more = ch + 1 < nchunks;
            // two groups: W(ch+1) (needed next iteration), then X(ch+3); the
            // wait below leaves only the newest group (X(ch+3)) in flight
            if (more) load_w(ch + 1, buf ^ 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            load_x(ch + 3);
            asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
            for (int k = 0; k < kLeanKC; ++k) {
                const float4 a03 = *reinterpret_cast<const float4*>(&xs[buf][k][8 * tg]);
                const float2 a45 = *reinterpret_cast<const float2*>(&xs[buf][k][8 * tg + 4]);
                const float a6 = xs[buf][k][8 * tg + 6];
                const float2 b01 = *reinterpret_cast<const float2*>(&ws[buf][k][kLeanExp * eg]);
                const float2 b23 = *reinterpret_cast<const float2*>(&ws[buf][k][kLeanExp * eg + 2]);
                const float2 b45 = *reinterpret_cast<const float2*>(&ws[buf][k][kLeanExp * eg + 4]);
                const float av[7] = {a03.x, a03.y, a03.z, a03.w, a45.x, a45.y, a6};
                const float bv[6] = {b01.x, b01.y, b23.x, b23.y, b45.x, b45.y};
#pragma unroll
                for (int i = 0; i < kLeanTok; ++i)
#pragma unroll
                    for (int j = 0; j < kLeanExp; ++j)
                        acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
            }
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
            if (more && tid < kLeanRows * kLeanKC) {
                const int r = tid / kLeanKC, k = tid % kLeanKC;
                xs[buf ^ 1][k][8 * (r / kLeanTok) + r % kLeanTok] =
                    xraw[(ch + 1) % kLeanXStages][r][k];
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < kLeanTok; ++i) {
            const int r = kLeanTok * tg + i;
            if (r >= nrows) continue;
            float* dst = logits + (size_t)(row0 + r) * E + kLeanExp * eg;
#pragma unroll
            for (int j = 0; j < kLeanExp; ++j)
                if (kLeanExp * eg + j < E) dst[j] = acc[i][j];
        }
    }
}

bool router_lean_ok(size_t K, size_t E) {
    return E <= (size_t)kLeanW && E % 4 == 0 && K % kLeanKC == 0;
}

void launch_router_lean(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                        size_t K, size_t E) {
    const size_t slabs = ceil_div(T, kLeanRows);
    const int grid = (int)std::min<size_t>(slabs, (size_t)c->num_sms * 2);
    router_lean_kernel<<<grid, kLeanThreads, 0, c->stream>>>(X, W, logits, (int)T, (int)K, (int)E);
    SCMOE_LAUNCH_CHECK(c);
}

// Small batches (config A: 512 tokens x 12 experts): one thread per logit,
// the reference chain c = 0; c = fl(c + fl(x_k * w_k)) in k order (router.hpp:136,
// tensor.hpp:95-112).  A CTA stages W (K x E) and its kSmallTok token rows in
// shared memory once; its E x kSmallTok threads then run their chains out of
// shared memory (x broadcast across a token's experts, W contiguous across
// the experts), k unrolled so the loads run ahead of the add chain.
constexpr int kSmallTok = 8;

__global__ void router_small_kernel(const float* __restrict__ X, const float* __restrict__ W,
                                    float* __restrict__ logits, int T, int K, int E) {
    extern __shared__ float rs_smem[];
    float* ws = rs_smem;            // [K][E]
    float* xs = rs_smem + K * E;    // [kSmallTok][K]
    const int t0 = blockIdx.x * kSmallTok;
    const int nt = min(kSmallTok, T - t0);
    for (int i = threadIdx.x; i < K * E; i += blockDim.x) ws[i] = W[i];
    for (int i = threadIdx.x; i < nt * K; i += blockDim.x) xs[i] = X[(size_t)t0 * K + i];
    __syncthreads();
    const int tl = threadIdx.x / E, e = threadIdx.x % E;
    if (tl >= nt) return;
    const float* x = xs + tl * K;
    float c = 0.f;
    int k = 0;
    for (; k + 8 <= K; k += 8) {
        float xv[8], wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            xv[u] = x[k + u];
            wv[u] = ws[(k + u) * E + e];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) c = __fadd_rn(c, __fmul_rn(xv[u], wv[u]));
    }
    for (; k < K; ++k) c = __fadd_rn(c, __fmul_rn(x[k], ws[k * E + e]));
    logits[(size_t)(t0 + tl) * E + e] = c;
}

static size_t router_small_smem(size_t K, size_t E) { return (K * E + kSmallTok * K) * sizeof(float); }

bool router_small_ok(size_t T, size_t K, size_t E, int num_sms) {
    // one logit per thread pays when the 16-row seq-GEMM tiles would leave most
    // SMs idle (fewer than ~4 tiles per SM); a CTA's E x 8 threads and its
    // staged W (K x E) must stay small
    return E * kSmallTok <= 1024 && router_small_smem(K, E) <= 96 * 1024 &&
           (T + 15) / 16 < (size_t)num_sms * 4;
}

void launch_router_small(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                         size_t K, size_t E) {
    const size_t smem = router_small_smem(K, E);
    SCMOE_CHECK_ARG(smem <= 200 * 1024 && E * kSmallTok <= 1024, SCMOE_ERR_CONFIG,
                    "router: small-batch kernel needs K*E + 8*K floats of shared memory");
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(router_small_kernel), (int)smem,
                            c->device);
    router_small_kernel<<<(unsigned)ceil_div(T, (size_t)kSmallTok), (unsigned)(E * kSmallTok), smem,
                          c->stream>>>(X, W, logits, (int)T, (int)K, (int)E);
    SCMOE_LAUNCH_CHECK(c);
}

bool router_slab_ok(size_t T, size_t K, size_t E, int num_sms) {
    // full-width slab needs E <= 768, E and K multiples of 4 (float4 rows), and
    // enough tokens to fill most SMs (otherwise the 16/64-row tiles spread better)
    return E <= (size_t)kSlabW && E % 4 == 0 && K % kSlabKC == 0 &&
           ceil_div(T, kSlabRows) >= (size_t)num_sms * 3 / 4;
}

void launch_router_slab(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                        size_t K, size_t E) {
    constexpr size_t smem =
        sizeof(float) * 2 * (kSlabKC * (kSlabW + kSlabXStride) + kSlabRows * kSlabKC);
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(router_slab_kernel), (int)smem,
                            c->device);
    router_slab_kernel<<<ceil_div(T, kSlabRows), kSlabThreads, smem, c->stream>>>(
        X, W, logits, (int)T, (int)K, (int)E);
    SCMOE_LAUNCH_CHECK(c);
}

template <int TM, int TN, int RM, int RN, int KC = 32>
static void seq_gemm_dispatch(scmoe_ctx* c, const float* A, size_t lda, const int* a_rows,
                              const float* B, size_t ldb, size_t b_group_stride, float* C,
                              size_t ldc, size_t K, size_t N, int silu, const TokenTile* tiles,
                              const int* n_tiles_dev, size_t max_tiles) {
    constexpr int NT = (TM / RM) * (TN / RN);
    dim3 grid((unsigned)ceil_div(N, TN), (unsigned)std::min<size_t>(max_tiles, 65535));
    if (silu)
        seq_gemm_kernel<TM, TN, RM, RN, true, KC><<<grid, NT, 0, c->stream>>>(
            A, lda, a_rows, B, ldb, b_group_stride, C, ldc, (int)K, (int)N, tiles, n_tiles_dev,
            (int)max_tiles);
    else
        seq_gemm_kernel<TM, TN, RM, RN, false, KC><<<grid, NT, 0, c->stream>>>(
            A, lda, a_rows, B, ldb, b_group_stride, C, ldc, (int)K, (int)N, tiles, n_tiles_dev,
            (int)max_tiles);
    SCMOE_LAUNCH_CHECK(c);
}

int seq_gemm_tile_rows(size_t rows, size_t N, int num_sms) {
    // Large config (64 x 64 tiles, 4x4 per thread) when it gives >= 4 CTAs per
    // SM; otherwise 16-row tiles (2x4 per thread) so small batches (decode)
    // still spread over every SM.
    return ceil_div(rows, 64) * ceil_div(N, 64) >= (size_t)num_sms * 4 ? 64 : 16;
}

void launch_seq_gemm(scmoe_ctx* c, const float* A, size_t lda, const int* a_rows, const float* B,
                     size_t ldb, size_t b_group_stride, float* C, size_t ldc, size_t K, size_t N,
                     int silu, const TokenTile* tiles, const int* n_tiles_dev, size_t max_tiles,
                     int tile_rows) {
    if (max_tiles == 0 || N == 0) return;
    if (tile_rows == 128)  // 128 x 128 tiles, 8 x 8 chains per thread (large GEMMs)
        seq_gemm_dispatch<128, 128, 8, 8, 16>(c, A, lda, a_rows, B, ldb, b_group_stride, C, ldc, K,
                                               N, silu, tiles, n_tiles_dev, max_tiles);
    else if (tile_rows == 64)
        seq_gemm_dispatch<64, 64, 4, 4>(c, A, lda, a_rows, B, ldb, b_group_stride, C, ldc, K, N,
                                        silu, tiles, n_tiles_dev, max_tiles);
    else if (tile_rows == 16)
        seq_gemm_dispatch<16, 64, 2, 4>(c, A, lda, a_rows, B, ldb, b_group_stride, C, ldc, K, N,
                                        silu, tiles, n_tiles_dev, max_tiles);
    else
        SCMOE_THROW(SCMOE_ERR_INTERNAL, "seq_gemm: unsupported tile rows");
}

// ---------------------------------------------------------------------------
// Sequential-k GEMV for a few rows (decode): C[r][n] = sum_k A[r][k] B[k][n]
// with the same chains as seq_gemm_kernel (c = 0; c = c + a*b, both
// rounded, k ascending).  An exact chain cannot be split over k, so the
// parallelism is the N columns: a CTA owns 64 columns (one thread per column,
// R chains each) and streams its [K x 64] slab of B through a 6-stage
// cp.async ring of 64-row chunks (16 KB each), so ~96 KB per CTA is in flight
// while the chains consume shared memory.  A rows are staged once.
// ---------------------------------------------------------------------------
constexpr int kGvCols = 64, kGvRows = 64, kGvStages = 6;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int n = pred ? 16 : 0;  // zero-fill when out of range
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n));
}

template <int R>
__global__ void __launch_bounds__(kGvCols) seq_gemv_kernel(const float* __restrict__ A, size_t lda,
                                                           const float* __restrict__ B, size_t ldb,
                                                           float* __restrict__ C, size_t ldc,
                                                           int K, int N) {
    extern __shared__ __align__(16) float gv_smem[];
    float* ring = gv_smem;                                   // [S][64 rows][64 cols]
    float* xs = gv_smem + kGvStages * kGvRows * kGvCols;     // [R][K]
    const int tid = threadIdx.x, n0 = blockIdx.x * kGvCols, n = n0 + tid;
    for (int i = tid; i < R * K; i += kGvCols) xs[i] = A[(size_t)(i / K) * lda + i % K];
    const int nch = (K + kGvRows - 1) / kGvRows;
    // a chunk = 64 rows x 64 columns = 1024 16-byte pieces, 16 per thread
    const bool vec_ok = ((ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) &&
                        n0 + kGvCols <= N;
    auto issue = [&](int ch) {
        float* dst = ring + (ch % kGvStages) * kGvRows * kGvCols;
        const int k0 = ch * kGvRows;
        if (vec_ok) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int piece = tid + u * kGvCols, row = piece >> 4, c4 = 4 * (piece & 15);
                const bool in = k0 + row < K;
                cp_async16(dst + row * kGvCols + c4, B + (size_t)(in ? k0 + row : 0) * ldb + n0 + c4,
                           in);
            }
        } else {  // ragged column block: scalar loads (synchronous)
            for (int row = 0; row < kGvRows; ++row) {
                const bool in = k0 + row < K && n < N;
                dst[row * kGvCols + tid] = in ? B[(size_t)(k0 + row) * ldb + n] : 0.f;
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    for (int ch = 0; ch < kGvStages - 1; ++ch) {
        if (ch < nch) issue(ch);
        else asm volatile("cp.async.commit_group;");
    }
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    for (int ch = 0; ch < nch; ++ch) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kGvStages - 2));
        __syncthreads();  // chunk ch visible to all; chunk ch-1's slot free
        if (ch + kGvStages - 1 < nch) issue(ch + kGvStages - 1);
        else asm volatile("cp.async.commit_group;");
        const float* w = ring + (ch % kGvStages) * kGvRows * kGvCols + tid;
        const int k0 = ch * kGvRows, kc = min(kGvRows, K - k0);
        if (kc == kGvRows) {
#pragma unroll 16
            for (int k = 0; k < kGvRows; ++k) {
                const float wv = w[k * kGvCols];
#pragma unroll
                for (int r = 0; r < R; ++r)
                    acc[r] = __fadd_rn(acc[r], __fmul_rn(xs[r * K + k0 + k], wv));
            }
        } else {
            for (int k = 0; k < kc; ++k) {
                const float wv = w[k * kGvCols];
#pragma unroll
                for (int r = 0; r < R; ++r)
                    acc[r] = __fadd_rn(acc[r], __fmul_rn(xs[r * K + k0 + k], wv));
            }
        }
    }
    asm volatile("cp.async.wait_group 0;");
    if (n < N) {
#pragma unroll
        for (int r = 0; r < R; ++r) C[(size_t)r * ldc + n] = acc[r];
    }
}

bool launch_seq_gemv(scmoe_ctx* c, const float* A, size_t lda, size_t rows, const float* B,
                     size_t ldb, float* C, size_t ldc, size_t K, size_t N) {
    const size_t smem = (kGvStages * kGvRows * kGvCols + rows * K) * sizeof(float);
    if (rows == 0 || rows > 4 || smem > 200 * 1024) return false;
    const unsigned grid = (unsigned)ceil_div(N, kGvCols);
    auto go = [&](auto kern) {
        ensure_max_dynamic_smem((const void*)kern, 200 * 1024, c->device);
        kern<<<grid, kGvCols, smem, c->stream>>>(A, lda, B, ldb, C, ldc, (int)K, (int)N);
    };
    switch (rows) {
        case 1: go(seq_gemv_kernel<1>); break;
        case 2: go(seq_gemv_kernel<2>); break;
        case 3: go(seq_gemv_kernel<3>); break;
        default: go(seq_gemv_kernel<4>); break;
    }
    SCMOE_LAUNCH_CHECK(c);
    return true;
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

    // glibc-expf table in shared memory: lanes index it divergently, which
    // serialises on the constant cache
    __shared__ uint64_t exp_tab[32];
    if (threadIdx.x < 32) exp_tab[threadIdx.x] = scmoe_exp2f_tab_dev[threadIdx.x];
    for (int j = threadIdx.x; j < E; j += blockDim.x) sbias[j] = bias ? bias[j] : 0.0;
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * 8 + warp;
    if (t >= T) return;
    S* p = rows + (size_t)warp * E;
    unsigned char* taken = taken_all + (size_t)warp * E;
    const S* row = in + (size_t)t * E;

    if constexpr (kFromLogits && std::is_same<S, double>::value) {
        // softmax_rows in S = double (tensor.hpp:174-192): glibc exp port
        double mx = -DBL_MAX;
        bool first = true;
        for (int j = lane; j < E; j += 32) {
            const double v = row[j];
            mx = first ? v : (v > mx ? v : mx);
            first = false;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double other = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = other > mx ? other : mx;
        }
        for (int j = lane; j < E; j += 32) p[j] = scmoe_exp(__dsub_rn(row[j], mx));
        __syncwarp();
        double sum = 0.0;
        if (lane == 0)
            for (int j = 0; j < E; ++j) sum = __dadd_rn(sum, p[j]);
        sum = __shfl_sync(0xffffffffu, sum, 0);
        for (int j = lane; j < E; j += 32) {
            const double q = __ddiv_rn(p[j], sum);
            p[j] = q;
            if (probs_out) probs_out[(size_t)t * E + j] = q;
        }
    } else if constexpr (kFromLogits) {
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
        for (int j = lane; j < E; j += 32) p[j] = scmoe_expf_smem(__fsub_rn(row[j], mx), exp_tab);
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

// ---------------------------------------------------------------------------
// Small batches (config A): the whole front of the layer in one launch --
// rmsnorm (graph.hpp:322-335), router logits (router.hpp:136), softmax and
// biased top-K (tensor.hpp:174-192, router.hpp:90-130) -- for E <= 32 experts.
// A CTA owns kFrontTok tokens: their rows and W sit in shared memory; one
// thread per row runs the sequential sum of squares, every thread scales,
// one thread per logit runs its chain, one warp per token (lane = expert)
// does softmax and selection.  Every step is the arithmetic of the separate
// kernels (rmsnorm_kernel, router_small_kernel, softmax_topk_kernel), so the
// results are identical bit for bit.
// ---------------------------------------------------------------------------
constexpr int kFrontTok = 8;

__global__ void __launch_bounds__(256) front_small_kernel(
    const float* __restrict__ a1, const float* __restrict__ gain, int T, int d, float eps,
    const float* __restrict__ W, int E, int K, int n_ffn, const double* __restrict__ bias,
    float* __restrict__ hmoe, __nv_bfloat16* __restrict__ hb, uint32_t* __restrict__ idx_out,
    double* __restrict__ gates_out, uint32_t* __restrict__ ffn_out) {
    extern __shared__ __align__(16) float fs_smem[];
    float* xs = fs_smem;                       // [kFrontTok][d]
    float* ws = xs + kFrontTok * d;            // [d][E]
    float* lg = ws + d * E;                    // [kFrontTok][32] logits, then probabilities
    float* inv = lg + kFrontTok * 32;          // [kFrontTok]
    __shared__ uint64_t exp_tab[32];
    const int tid = threadIdx.x;
    if (tid < 32) exp_tab[tid] = scmoe_exp2f_tab_dev[tid];
    const int t0 = blockIdx.x * kFrontTok;
    const int nt = min(kFrontTok, T - t0);
    for (int i = tid; i < d * E; i += blockDim.x) ws[i] = W[i];
    for (int i = tid; i < nt * d; i += blockDim.x) xs[i] = a1[(size_t)t0 * d + i];
    __syncthreads();
    // rmsnorm: the reference's sequential sum of squares, one thread per row
    if (tid < nt) {
        const float* x = xs + tid * d;
        float s2 = 0.0f;
#pragma unroll 8
        for (int j = 0; j < d; ++j) s2 = __fadd_rn(s2, __fmul_rn(x[j], x[j]));
        inv[tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(s2, (float)d), eps)));
    }
    __syncthreads();
    for (int i = tid; i < nt * d; i += blockDim.x) {
        const int r = i / d, j = i % d;
        const float v = __fmul_rn(__fmul_rn(xs[i], inv[r]), gain ? gain[j] : 1.0f);
        xs[i] = v;
        hmoe[(size_t)t0 * d + i] = v;
        if (hb) hb[(size_t)t0 * d + i] = __float2bfloat16_rn(v);
    }
    __syncthreads();
    // router logits: one chain per (token, expert), k ascending
    if (tid < nt * E) {
        const int r = tid / E, e = tid % E;
        const float* x = xs + r * d;
        float c = 0.f;
#pragma unroll 8
        for (int k = 0; k < d; ++k) c = __fadd_rn(c, __fmul_rn(x[k], ws[k * E + e]));
        lg[r * 32 + e] = c;
    }
    __syncthreads();
    // softmax + biased top-K: warp w = token w, lane = expert
    const int warp = tid >> 5, lane = tid & 31;
    if (warp >= nt) return;
    const int t = t0 + warp;
    float* row = lg + warp * 32;
    float mx = -FLT_MAX;
    if (lane < E) mx = row[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float other = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = other > mx ? other : mx;
    }
    float p = 0.f;
    if (lane < E) p = scmoe_expf_smem(__fsub_rn(row[lane], mx), exp_tab);
    __syncwarp();
    if (lane < E) row[lane] = p;
    __syncwarp();
    float sum = 0.0f;
    if (lane == 0)
        for (int j = 0; j < E; ++j) sum = __fadd_rn(sum, row[j]);
    sum = __shfl_sync(0xffffffffu, sum, 0);
    const float q = lane < E ? __fdiv_rn(p, sum) : 0.f;
    const double bj = (lane < E && bias) ? bias[lane] : 0.0;
    bool taken = lane >= E;
    uint32_t ffn = 0;
    for (int s = 0; s < K; ++s) {
        double best_s = 0.0;
        int best_i = INT_MAX;
        float best_q = 0.f;
        if (!taken) {
            best_s = __dadd_rn((double)q, bj);
            best_i = lane;
            best_q = q;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, best_s, o);
            const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            const float oq = __shfl_xor_sync(0xffffffffu, best_q, o);
            if (oi != INT_MAX && (best_i == INT_MAX || better(os, oi, best_s, best_i))) {
                best_s = os;
                best_i = oi;
                best_q = oq;
            }
        }
        if (lane == best_i) taken = true;
        if (lane == 0) {
            idx_out[(size_t)t * K + s] = (uint32_t)best_i;
            gates_out[(size_t)t * K + s] = (double)best_q;
        }
        ffn += best_i < n_ffn ? 1u : 0u;
    }
    if (lane == 0) ffn_out[t] = ffn;
}

static size_t front_small_smem(size_t d, size_t E) {
    return (kFrontTok * d + d * E + kFrontTok * 32 + kFrontTok) * sizeof(float);
}

bool front_small_ok(size_t T, size_t d, size_t E, size_t K, int num_sms) {
    return E <= 32 && K <= E && front_small_smem(d, E) <= 96 * 1024 &&
           (T + 15) / 16 < (size_t)num_sms * 4;
}

void launch_front_small(scmoe_ctx* c, const float* a1, const float* gain, size_t T, size_t d,
                        float eps, const float* W, size_t E, size_t K, size_t n_ffn,
                        const double* bias, float* hmoe, __nv_bfloat16* hb, uint32_t* idx,
                        double* gates, uint32_t* ffn_count) {
    if (T == 0) return;
    const size_t smem = front_small_smem(d, E);
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(front_small_kernel), (int)smem,
                            c->device);
    front_small_kernel<<<(unsigned)ceil_div(T, (size_t)kFrontTok), 256, smem, c->stream>>>(
        a1, gain, (int)T, (int)d, eps, W, (int)E, (int)K, (int)n_ffn, bias, hmoe, hb, idx, gates,
        ffn_count);
    SCMOE_LAUNCH_CHECK(c);
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

// ---------------------------------------------------------------------------
// Router projection in S = double (RouterState<double>, router.hpp:136 ->
// tensor.hpp:95-112 in double): per output c = 0; c = c + x*w (separately
// rounded DMUL / DADD) in k order.  64 x 64 CTA tile, 4 x 4 chains per
// thread, K staged 16 rows at a time.  Not on the fp32 hot path.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) router_f64_kernel(const double* __restrict__ X,
                                                         const double* __restrict__ W,
                                                         double* __restrict__ out, int T, int K,
                                                         int E) {
    __shared__ double xs[16][64 + 1];
    __shared__ double wsm[16][64];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int i = threadIdx.x; i < 16 * 64; i += 256) {
            const int kk = i / 64, c = i % 64;
            const int r = row0 + c, k = k0 + kk, e = col0 + c;
            xs[kk][c] = (r < T && k < K) ? X[(size_t)r * K + k] : 0.0;
            wsm[kk][c] = (e < E && k < K) ? W[(size_t)k * E + e] : 0.0;
        }
        __syncthreads();
        const int kn = min(16, K - k0);
        for (int kk = 0; kk < kn; ++kk) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double a = xs[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a, wsm[kk][tx * 4 + j]));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = row0 + ty * 4 + i, e = col0 + tx * 4 + j;
            if (r < T && e < E) out[(size_t)r * E + e] = acc[i][j];
        }
}
void launch_router_f64(scmoe_ctx* c, const double* X, const double* W, double* logits, size_t T,
                       size_t K, size_t E) {
    if (T == 0) return;
    const dim3 grid((unsigned)ceil_div(E, 64), (unsigned)ceil_div(T, 64));
    router_f64_kernel<<<grid, 256, 0, c->stream>>>(X, W, logits, (int)T, (int)K, (int)E);
    SCMOE_LAUNCH_CHECK(c);
}
void launch_softmax_topk_f64(scmoe_ctx* c, const double* logits, size_t T, size_t E, size_t K,
                             size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                             uint32_t* ffn, double* probs) {
    launch_topk_impl<double, true>(c, logits, T, E, K, n_ffn, bias, idx, gates, ffn, probs);
}
// graph.hpp:529-533 in S = double: sign-branched logistic on the exp port;
// graph.hpp:133-135: silu(v) = v * sigmoid(v).
__device__ __forceinline__ double scmoe_silu_f64(double v) {
    double sg;
    if (v >= 0.0) {
        sg = __ddiv_rn(1.0, __dadd_rn(1.0, scmoe_exp(-v)));
    } else {
        const double e = scmoe_exp(v);
        sg = __ddiv_rn(e, __dadd_rn(1.0, e));
    }
    return __dmul_rn(v, sg);
}

// Grouped sequential GEMM in double (mm_into, tensor.hpp:95-112, S = double):
// CTA = one token tile (<= 64 rows of one expert) x 64 output columns.
__global__ void __launch_bounds__(256) seq_gemm_f64_kernel(
    const double* __restrict__ A, int lda, const int* __restrict__ a_rows,
    const double* __restrict__ B, int ldb, size_t b_group_stride, double* __restrict__ C, int ldc,
    int K, int N, int silu, const TokenTile* __restrict__ tiles, const int* __restrict__ n_tiles) {
    if ((int)blockIdx.y >= *n_tiles) return;
    const TokenTile tile = tiles[blockIdx.y];
    __shared__ double xs[16][64 + 1];
    __shared__ double wsm[16][64];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int col0 = blockIdx.x * 64;
    const double* Bg = B + (size_t)tile.e * b_group_stride;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int i = threadIdx.x; i < 16 * 64; i += 256) {
            const int kk = i / 64, cc = i % 64;
            const int k = k0 + kk, col = col0 + cc;
            double xv = 0.0;
            if (cc < tile.count && k < K) {
                const int p = tile.pos + cc;
                xv = A[(size_t)(a_rows ? a_rows[p] : p) * lda + k];
            }
            xs[kk][cc] = xv;
            wsm[kk][cc] = (col < N && k < K) ? Bg[(size_t)k * ldb + col] : 0.0;
        }
        __syncthreads();
        const int kn = min(16, K - k0);
        for (int kk = 0; kk < kn; ++kk) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double a = xs[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a, wsm[kk][tx * 4 + j]));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = ty * 4 + i, col = col0 + tx * 4 + j;
            if (r < tile.count && col < N)
                C[(size_t)(tile.pos + r) * ldc + col] = silu ? scmoe_silu_f64(acc[i][j]) : acc[i][j];
        }
}
void launch_seq_gemm_f64(scmoe_ctx* c, const double* A, size_t lda, const int* a_rows,
                         const double* B, size_t ldb, size_t b_group_stride, double* C,
                         size_t ldc, size_t K, size_t N, int silu, const TokenTile* tiles,
                         const int* n_tiles_dev, size_t max_tiles) {
    if (max_tiles == 0 || N == 0) return;
    const dim3 grid((unsigned)ceil_div(N, 64), (unsigned)std::min<size_t>(max_tiles, 65535));
    seq_gemm_f64_kernel<<<grid, 256, 0, c->stream>>>(A, (int)lda, a_rows, B, (int)ldb,
                                                     b_group_stride, C, (int)ldc, (int)K, (int)N,
                                                     silu, tiles, n_tiles_dev);
    SCMOE_LAUNCH_CHECK(c);
}

__global__ void debug_exp_kernel(const double* __restrict__ in, double* __restrict__ out,
                                 size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = scmoe_exp(in[i]);
}
void launch_debug_exp(scmoe_ctx* c, const double* in, double* out, size_t n) {
    if (n == 0) return;
    debug_exp_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(in, out, n);
    SCMOE_LAUNCH_CHECK(c);
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
