// mla.cu -- multi-head latent attention, forward value (S = float), exact.
//
// blocks.hpp:73-102 (mla_block), :129-181 (mla_infer_step); tensor.hpp:197-224
// (rope_apply); graph.hpp:396-434 (attention).  Every output is produced with
// the reference's operation order and rounding:
//   * projections: sequential-k fp32 chains (seq_gemm_kernel, tensor.hpp:95-112);
//     the projections that read the same input are fused into one GEMM over
//     column-concatenated weights -- output columns are independent, so the
//     bits do not change;
//   * g.scale: one rounded multiply by float(alpha);
//   * rope: a*c - b*s and a*s + b*c, products and sums separately rounded,
//     with (c, s) = float(cos/sin(theta)) from a host table computed with the
//     reference's own expression (libm pow/cos/sin, double);
//   * attention: score = sequential dot over [content | rotary] (rounded mul
//     + add), times the rounded scale; the row max; e = expf(s - max) on the
//     glibc expf port; the normaliser a sequential fp32 sum in key order;
//     w = e / denom; out = sequential sum over keys of w * v.
// Compiled with --fmad=false; packed f32x2 chains use the half-swapped add
// (f32x2.cuh), so nothing is contracted (build.py checks the SASS).
#include <cstdlib>

#include "f32x2.cuh"
#include "internal.cuh"
#include "libm_port.h"

namespace scmoe {

// ---------------------------------------------------------------------------
// Scale + rotary epilogue of a projection output X [rows, ld]:
//   cols [0, n_a) *= alpha_a, [n_a, n_a + n_b) *= alpha_b,
//   cols [rc, rc + heads*hd) rotated per head at pos = pos0 + r % seq_len.
// One thread per (row, item); items are the scaled columns then the pairs.
// ---------------------------------------------------------------------------
__global__ void mla_scale_rope_kernel(float* __restrict__ X, size_t ld, size_t rows, int n_a,
                                      float alpha_a, int n_b, float alpha_b, int rc, int heads,
                                      int hd, const float2* __restrict__ table, size_t pos0,
                                      size_t seq_len) {
    const int half = hd / 2;
    const size_t per_row = (size_t)n_a + n_b + (size_t)heads * half;
    const size_t n = rows * per_row;
    for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < n;
         it += (size_t)gridDim.x * blockDim.x) {
        const size_t r = it / per_row;
        size_t c = it % per_row;
        float* row = X + r * ld;
        if (c < (size_t)n_a) {
            row[c] = __fmul_rn(row[c], alpha_a);
        } else if (c < (size_t)(n_a + n_b)) {
            row[c] = __fmul_rn(row[c], alpha_b);
        } else {
            c -= n_a + n_b;
            const int h = (int)(c / half), p = (int)(c % half);
            const size_t pos = pos0 + r % seq_len;
            const float2 cs = table[pos * half + p];
            float* q = row + rc + h * hd + 2 * p;
            const float a = q[0], b = q[1];
            q[0] = __fsub_rn(__fmul_rn(a, cs.x), __fmul_rn(b, cs.y));
            q[1] = __fadd_rn(__fmul_rn(a, cs.y), __fmul_rn(b, cs.x));
        }
    }
}

constexpr int kMlaKC = 32, kMlaPad = 4, kMlaTN = 64;

// Scores S[i][j] = scale * (sum_t qc_i[t] kc_j[t] + sum_t qr_i[t] kr_j[t]) in
// t order.  CTA tile TM queries x 64 keys, thread tile RM x 4 (f32x2 pairs
// along keys); the dot length is staged through shared memory in chunks of
// 32 taken first from the content halves, then from the rotary halves.
template <int TM, int RM>
__global__ void __launch_bounds__((TM / RM) * 16) mla_scores_kernel(MlaAttnArgs a) {
    constexpr int NT = (TM / RM) * 16;
    __shared__ __align__(16) float As[kMlaKC][TM + kMlaPad];
    __shared__ __align__(16) float Bs[kMlaKC][kMlaTN + kMlaPad];
    const int bh = blockIdx.z, b = bh / a.H, h = bh % a.H;
    const int i0 = blockIdx.y * TM, j0 = blockIdx.x * kMlaTN;
    const int i_last = min(a.nq, i0 + TM) - 1;
    if (j0 > a.q0 + i_last) return;  // tile entirely above the causal diagonal
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const size_t qrow0 = (size_t)b * a.nq, krow0 = (size_t)b * a.nk;

    uint64_t acc2[RM][2];
#pragma unroll
    for (int i = 0; i < RM; ++i) acc2[i][0] = acc2[i][1] = 0;

    for (int seg = 0; seg < 2; ++seg) {
        const int len = seg == 0 ? a.dhc : a.dhr;
        const float* qb = seg == 0 ? a.qc + (size_t)h * a.dhc : a.qr + (size_t)h * a.dhr;
        const float* kb = seg == 0 ? a.kc + (size_t)h * a.dhc : a.kr;
        const size_t ldk = seg == 0 ? a.ldkv : a.ldkr;
        for (int k0 = 0; k0 < len; k0 += kMlaKC) {
            const int kc = min(kMlaKC, len - k0);
            for (int e = tid; e < TM * kMlaKC; e += NT) {
                const int r = e / kMlaKC, k = e % kMlaKC;
                float v = 0.f;
                if (k < kc && i0 + r < a.nq) v = qb[(qrow0 + i0 + r) * a.ldq + k0 + k];
                As[k][r] = v;
            }
            for (int e = tid; e < kMlaTN * kMlaKC; e += NT) {
                const int r = e / kMlaKC, k = e % kMlaKC;
                float v = 0.f;
                if (k < kc && j0 + r < a.nk) v = kb[(krow0 + j0 + r) * ldk + k0 + k];
                Bs[k][r] = v;
            }
            __syncthreads();
            for (int k = 0; k < kc; ++k) {
                float av[RM];
#pragma unroll
                for (int i = 0; i < RM; ++i) av[i] = As[k][RM * ty + i];
                const ulonglong2 bb = *reinterpret_cast<const ulonglong2*>(&Bs[k][4 * tx]);
#pragma unroll
                for (int i = 0; i < RM; ++i) {
                    acc2[i][0] = f2_add_swapped(acc2[i][0], f2_mul_bcast(av[i], bb.x));
                    acc2[i][1] = f2_add_swapped(acc2[i][1], f2_mul_bcast(av[i], bb.y));
                }
            }
            __syncthreads();
        }
    }
    float* att = a.att + (size_t)bh * a.nq * a.nk;
    const int nkt = (a.nk + kMlaTN - 1) / kMlaTN;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
        const int qi = i0 + RM * ty + i;
        const float s[4] = {f2_hi(acc2[i][0]), f2_lo(acc2[i][0]), f2_hi(acc2[i][1]),
                            f2_lo(acc2[i][1])};
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = j0 + 4 * tx + q;
            if (qi < a.nq && j < a.nk && j <= a.q0 + qi) {
                const float v = __fmul_rn(s[q], a.scale);
                att[(size_t)qi * a.nk + j] = v;
                mx = fmaxf(mx, v);
            }
        }
        // this key tile's row max (the 16 threads of a row are lanes of one half-warp)
#pragma unroll
        for (int o = 8; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (tx == 0 && qi < a.nq) a.part_max[((size_t)bh * a.nq + qi) * nkt + blockIdx.x] = mx;
    }
}

// Softmax of the score rows, in place, 32 consecutive rows (b, h, i..i+31)
// per warp; row i has n = q0 + i + 1 keys.
//   max   = max of the scores kernel's per-key-tile maxima (order free);
//   e_j   = expf(s_j - max) and denom = sum of e_j in key order: a 32x32 block
//           is loaded coalesced, transposed through shared memory, and lane l
//           walks row l's 32 keys sequentially (the reference's fp32 sum);
//   w_j   = e_j / denom (rounded division), coalesced, written in place.
__global__ void __launch_bounds__(256, 4) mla_softmax_kernel(float* __restrict__ att,
                                                          const float* __restrict__ part_max,
                                                          int rows_total, int nq, int nk, int q0) {
    __shared__ float tile[8][32][33];
    __shared__ uint64_t exp_tab[32];
    if (threadIdx.x < 32) exp_tab[threadIdx.x] = scmoe_exp2f_tab_dev[threadIdx.x];
    __syncthreads();
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = (blockIdx.x * 8 + wib) * 32;
    if (r0 >= rows_total) return;
    float(*T)[33] = tile[wib];
    const int nkt = (nk + kMlaTN - 1) / kMlaTN;
    const int r = r0 + lane;
    const bool live = r < rows_total;
    const int n = live ? min(nk, q0 + r % nq + 1) : 0;
    float mx = -INFINITY;
    for (int t = 0; t < (n + kMlaTN - 1) / kMlaTN; ++t) mx = fmaxf(mx, part_max[(size_t)r * nkt + t]);
    // rows of the warp may straddle two (b, h) blocks: lengths are per row
    int nmax = 0;
    for (int t = 0; t < 32; ++t) nmax = max(nmax, __shfl_sync(0xffffffffu, n, t));
    float sum = 0.f;
    for (int j0 = 0; j0 < nmax; j0 += 32) {
#pragma unroll
        for (int t0 = 0; t0 < 32; t0 += 16) {
            float v[16];  // 16 coalesced row segments in flight before the transpose
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int nt = __shfl_sync(0xffffffffu, n, t0 + t);
                v[t] = (j0 + lane < nt) ? att[(size_t)(r0 + t0 + t) * nk + j0 + lane] : 0.f;
            }
#pragma unroll
            for (int t = 0; t < 16; ++t) T[t0 + t][lane] = v[t];
        }
        __syncwarp();
        const int m = min(32, n - j0);
        if (m == 32) {
            // 8 independent exponentials at a time (ILP), then the in-order sum
#pragma unroll
            for (int t0 = 0; t0 < 32; t0 += 8) {
                float e[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) e[t] = scmoe_expf_smem(__fsub_rn(T[lane][t0 + t], mx), exp_tab);
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    T[lane][t0 + t] = e[t];
                    sum = __fadd_rn(sum, e[t]);
                }
            }
        } else {
            for (int t = 0; t < m; ++t) {
                const float e = scmoe_expf_smem(__fsub_rn(T[lane][t], mx), exp_tab);
                T[lane][t] = e;
                sum = __fadd_rn(sum, e);
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int nt = __shfl_sync(0xffffffffu, n, t);
            if (j0 + lane < nt) att[(size_t)(r0 + t) * nk + j0 + lane] = T[t][lane];
        }
        __syncwarp();
    }
    // w = e / denom, row by row, 16-byte accesses with 4 in flight per lane
    for (int t = 0; t < 32; ++t) {
        const int rt = r0 + t, nt = __shfl_sync(0xffffffffu, n, t);
        const float den = __shfl_sync(0xffffffffu, sum, t);
        float* row = att + (size_t)rt * nk;
        int j = 0;
        if ((nk & 3) == 0) {
            float4* r4 = reinterpret_cast<float4*>(row);
            const int n4 = nt >> 2;
            for (int q0 = 0; q0 < n4; q0 += 128) {
                float4 w[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = q0 + 32 * u + lane;
                    if (q < n4) w[u] = r4[q];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = q0 + 32 * u + lane;
                    if (q < n4)
                        r4[q] = make_float4(__fdiv_rn(w[u].x, den), __fdiv_rn(w[u].y, den),
                                            __fdiv_rn(w[u].z, den), __fdiv_rn(w[u].w, den));
                }
            }
            j = n4 * 4;
        }
        for (j += lane; j < nt; j += 32) row[j] = __fdiv_rn(row[j], den);
    }
}

// merged[i][h*dhc + p] = sum_{j <= q0+i} w[i][j] * v[j][p], j ascending,
// starting from 0.  CTA tile TM queries x 64 value columns; keys staged in
// chunks of 32.  Chunks that cross the diagonal of some row select instead of
// adding, so a row never sees a key past its own position.
template <int TM, int RM>
__global__ void __launch_bounds__((TM / RM) * 16) mla_pv_kernel(MlaAttnArgs a) {
    constexpr int NT = (TM / RM) * 16;
    __shared__ __align__(16) float As[kMlaKC][TM + kMlaPad];
    __shared__ __align__(16) float Bs[kMlaKC][kMlaTN + kMlaPad];
    const int bh = blockIdx.z, b = bh / a.H, h = bh % a.H;
    const int i0 = blockIdx.y * TM, c0 = blockIdx.x * kMlaTN;
    if (i0 >= a.nq) return;
    const int i_last = min(a.nq, i0 + TM) - 1;
    const int jmax = min(a.nk, a.q0 + i_last + 1);  // keys any row of the tile sees
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const float* att = a.att + (size_t)bh * a.nq * a.nk;
    const float* vb = a.v + (size_t)b * a.nk * a.ldkv + (size_t)h * a.dhc;

    uint64_t acc2[RM][2];
#pragma unroll
    for (int i = 0; i < RM; ++i) acc2[i][0] = acc2[i][1] = 0;
    int lim[RM];  // last key of each thread row
#pragma unroll
    for (int i = 0; i < RM; ++i) lim[i] = a.q0 + i0 + RM * ty + i;

    for (int k0 = 0; k0 < jmax; k0 += kMlaKC) {
        const int kc = min(kMlaKC, jmax - k0);
        for (int e = tid; e < TM * kMlaKC; e += NT) {
            const int r = e / kMlaKC, k = e % kMlaKC;
            float v = 0.f;
            if (k < kc && i0 + r < a.nq && k0 + k <= a.q0 + i0 + r)
                v = att[(size_t)(i0 + r) * a.nk + k0 + k];
            As[k][r] = v;
        }
        for (int e = tid; e < kMlaTN * kMlaKC; e += NT) {
            const int k = e / kMlaTN, cc = e % kMlaTN;
            float v = 0.f;
            if (k < kc && c0 + cc < a.dhc) v = vb[(size_t)(k0 + k) * a.ldkv + c0 + cc];
            Bs[k][cc] = v;
        }
        __syncthreads();
        if (k0 + kc - 1 <= a.q0 + i0) {  // every row of the tile sees the whole chunk
            for (int k = 0; k < kc; ++k) {
                float av[RM];
#pragma unroll
                for (int i = 0; i < RM; ++i) av[i] = As[k][RM * ty + i];
                const ulonglong2 bb = *reinterpret_cast<const ulonglong2*>(&Bs[k][4 * tx]);
#pragma unroll
                for (int i = 0; i < RM; ++i) {
                    acc2[i][0] = f2_add_swapped(acc2[i][0], f2_mul_bcast(av[i], bb.x));
                    acc2[i][1] = f2_add_swapped(acc2[i][1], f2_mul_bcast(av[i], bb.y));
                }
            }
        } else {
            for (int k = 0; k < kc; ++k) {
                float av[RM];
#pragma unroll
                for (int i = 0; i < RM; ++i) av[i] = As[k][RM * ty + i];
                const ulonglong2 bb = *reinterpret_cast<const ulonglong2*>(&Bs[k][4 * tx]);
#pragma unroll
                for (int i = 0; i < RM; ++i) {
                    const bool on = k0 + k <= lim[i];
                    const uint64_t n0 = f2_add_swapped(acc2[i][0], f2_mul_bcast(av[i], bb.x));
                    const uint64_t n1 = f2_add_swapped(acc2[i][1], f2_mul_bcast(av[i], bb.y));
                    acc2[i][0] = on ? n0 : acc2[i][0];
                    acc2[i][1] = on ? n1 : acc2[i][1];
                }
            }
        }
        __syncthreads();
    }
    float* mb = a.merged + (size_t)b * a.nq * a.ldm + (size_t)h * a.dhc;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
        const int qi = i0 + RM * ty + i;
        if (qi >= a.nq) continue;
        const float s[4] = {f2_hi(acc2[i][0]), f2_lo(acc2[i][0]), f2_hi(acc2[i][1]),
                            f2_lo(acc2[i][1])};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = c0 + 4 * tx + q;
            if (col < a.dhc) mb[(size_t)qi * a.ldm + col] = s[q];
        }
    }
}

// ---------------------------------------------------------------------------
// Large-batch variants: 128 x 128 CTA tiles, 8 x 8 chains per thread (256
// threads), chunks of 16 along the dot length staged through shared memory
// with a register double buffer (the next chunk's global loads are in flight
// during the current chunk's arithmetic).  Same per-output operation order as
// the kernels above.
// ---------------------------------------------------------------------------
constexpr int kBT = 128, kBK = 16, kBPad = 4, kBThreads = 256;

// A [128 rows][16 k] chunk from row-major storage (row stride ld), rows
// clipped at n_rows, k clipped at kc; 2 float4 per thread.
struct ChunkRegs {
    float4 v[2];
};
__device__ __forceinline__ void load_rows_chunk(ChunkRegs& R, const float* base, size_t ld,
                                                int n_rows, int kc, int tid) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        const int i = tid + l * kBThreads;
        const int r = i >> 2, kk = 4 * (i & 3);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < n_rows) {
            const float* src = base + (size_t)r * ld + kk;
            if (kk + 3 < kc && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
                v = *reinterpret_cast<const float4*>(src);
            } else {
                if (kk + 0 < kc) v.x = src[0];
                if (kk + 1 < kc) v.y = src[1];
                if (kk + 2 < kc) v.z = src[2];
                if (kk + 3 < kc) v.w = src[3];
            }
        }
        R.v[l] = v;
    }
}
__device__ __forceinline__ void store_rows_chunk_T(const ChunkRegs& R, float (*S)[kBT + kBPad],
                                                   int tid) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        const int i = tid + l * kBThreads;
        const int r = i >> 2, kk = 4 * (i & 3);
        S[kk + 0][r] = R.v[l].x;
        S[kk + 1][r] = R.v[l].y;
        S[kk + 2][r] = R.v[l].z;
        S[kk + 3][r] = R.v[l].w;
    }
}

__device__ __forceinline__ void mma_chunk_8x8(uint64_t (&acc2)[8][4], const float (*As)[kBT + kBPad],
                                              const float (*Bs)[kBT + kBPad], int kc, int ty,
                                              int tx) {
#pragma unroll 4
    for (int k = 0; k < kc; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[k][8 * ty]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[k][8 * ty + 4]);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(&Bs[k][8 * tx]);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(&Bs[k][8 * tx + 4]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const uint64_t bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                acc2[i][q] = f2_add_swapped(acc2[i][q], f2_mul_bcast(av[i], bv[q]));
    }
}

__global__ void __launch_bounds__(kBThreads, 2) mla_scores_big_kernel(MlaAttnArgs a) {
    __shared__ __align__(16) float As[2][kBK][kBT + kBPad];
    __shared__ __align__(16) float Bs[2][kBK][kBT + kBPad];
    const int bh = blockIdx.z, b = bh / a.H, h = bh % a.H;
    const int i0 = blockIdx.y * kBT, j0 = blockIdx.x * kBT;
    const int i_last = min(a.nq, i0 + kBT) - 1;
    if (j0 > a.q0 + i_last) return;  // tile entirely above the causal diagonal
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const float* qc = a.qc + ((size_t)b * a.nq + i0) * a.ldq + (size_t)h * a.dhc;
    const float* qr = a.qr + ((size_t)b * a.nq + i0) * a.ldq + (size_t)h * a.dhr;
    const float* kc = a.kc + ((size_t)b * a.nk + j0) * a.ldkv + (size_t)h * a.dhc;
    const float* kr = a.kr + ((size_t)b * a.nk + j0) * a.ldkr;
    const int nqr = a.nq - i0, nkr = a.nk - j0;
    const int nc_c = (a.dhc + kBK - 1) / kBK, nch = nc_c + (a.dhr + kBK - 1) / kBK;
    auto load = [&](ChunkRegs& RA, ChunkRegs& RB, int ch, int& kcnt) {
        if (ch < nc_c) {
            const int k0 = ch * kBK;
            kcnt = min(kBK, a.dhc - k0);
            load_rows_chunk(RA, qc + k0, a.ldq, nqr, kcnt, tid);
            load_rows_chunk(RB, kc + k0, a.ldkv, nkr, kcnt, tid);
        } else {
            const int k0 = (ch - nc_c) * kBK;
            kcnt = min(kBK, a.dhr - k0);
            load_rows_chunk(RA, qr + k0, a.ldq, nqr, kcnt, tid);
            load_rows_chunk(RB, kr + k0, a.ldkr, nkr, kcnt, tid);
        }
    };
    uint64_t acc2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc2[i][q] = 0;
    ChunkRegs RA, RB;
    int kcur = 0, knext = 0;
    load(RA, RB, 0, kcur);
    store_rows_chunk_T(RA, As[0], tid);
    store_rows_chunk_T(RB, Bs[0], tid);
    __syncthreads();
    for (int ch = 0; ch < nch; ++ch) {
        const int buf = ch & 1;
        const bool more = ch + 1 < nch;
        if (more) load(RA, RB, ch + 1, knext);
        mma_chunk_8x8(acc2, As[buf], Bs[buf], kcur, ty, tx);
        if (more) {
            store_rows_chunk_T(RA, As[buf ^ 1], tid);
            store_rows_chunk_T(RB, Bs[buf ^ 1], tid);
        }
        __syncthreads();
        kcur = knext;
    }
    float* att = a.att + (size_t)bh * a.nq * a.nk;
    const int nkt = (a.nk + kMlaTN - 1) / kMlaTN;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int qi = i0 + 8 * ty + i;
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float pr[2] = {f2_hi(acc2[i][q]), f2_lo(acc2[i][q])};
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = j0 + 8 * tx + 2 * q + u;
                if (qi < a.nq && j < a.nk && j <= a.q0 + qi) {
                    const float v = __fmul_rn(pr[u], a.scale);
                    att[(size_t)qi * a.nk + j] = v;
                    mx = fmaxf(mx, v);
                }
            }
        }
        // row max per 64-key part: threads tx 0-7 hold part 2x, tx 8-15 part 2x+1
#pragma unroll
        for (int o = 4; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int part = 2 * blockIdx.x + (tx >> 3);
        if ((tx & 7) == 0 && qi < a.nq && part < nkt)
            a.part_max[((size_t)bh * a.nq + qi) * nkt + part] = mx;
    }
}

// PV on 128-query x 128-column tiles (d_head_c <= 128 -> one column tile, the
// weights are read once).
__global__ void __launch_bounds__(kBThreads, 2) mla_pv_big_kernel(MlaAttnArgs a) {
    __shared__ __align__(16) float As[2][kBK][kBT + kBPad];
    __shared__ __align__(16) float Bs[2][kBK][kBT + kBPad];
    const int bh = blockIdx.z, b = bh / a.H, h = bh % a.H;
    const int i0 = blockIdx.y * kBT, c0 = blockIdx.x * kBT;
    if (i0 >= a.nq) return;
    const int i_last = min(a.nq, i0 + kBT) - 1;
    const int jmax = min(a.nk, a.q0 + i_last + 1);
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const float* att = a.att + ((size_t)bh * a.nq + i0) * a.nk;
    const float* vb = a.v + (size_t)b * a.nk * a.ldkv + (size_t)h * a.dhc + c0;
    const int ncol = min(kBT, a.dhc - c0), nqr = a.nq - i0;
    // V chunk [16 keys][128 cols]: 2 float4 per thread
    auto load_v = [&](ChunkRegs& R, int k0, int kc) {
#pragma unroll
        for (int l = 0; l < 2; ++l) {
            const int i = tid + l * kBThreads;
            const int k = i >> 5, c4 = 4 * (i & 31);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k < kc) {
                const float* src = vb + (size_t)(k0 + k) * a.ldkv + c4;
                if (c4 + 3 < ncol && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
                    v = *reinterpret_cast<const float4*>(src);
                } else {
                    if (c4 + 0 < ncol) v.x = src[0];
                    if (c4 + 1 < ncol) v.y = src[1];
                    if (c4 + 2 < ncol) v.z = src[2];
                    if (c4 + 3 < ncol) v.w = src[3];
                }
            }
            R.v[l] = v;
        }
    };
    auto store_v = [&](const ChunkRegs& R, float (*S)[kBT + kBPad]) {
#pragma unroll
        for (int l = 0; l < 2; ++l) {
            const int i = tid + l * kBThreads;
            *reinterpret_cast<float4*>(&S[i >> 5][4 * (i & 31)]) = R.v[l];
        }
    };
    uint64_t acc2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc2[i][q] = 0;
    int lim[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) lim[i] = a.q0 + i0 + 8 * ty + i;
    const int nch = (jmax + kBK - 1) / kBK;
    ChunkRegs RA, RB;
    load_rows_chunk(RA, att, a.nk, nqr, min(kBK, jmax), tid);
    load_v(RB, 0, min(kBK, jmax));
    store_rows_chunk_T(RA, As[0], tid);
    store_v(RB, Bs[0]);
    __syncthreads();
    for (int ch = 0; ch < nch; ++ch) {
        const int buf = ch & 1, k0 = ch * kBK, kc = min(kBK, jmax - k0);
        const bool more = ch + 1 < nch;
        if (more) {
            const int k1 = k0 + kBK, kc1 = min(kBK, jmax - k1);
            load_rows_chunk(RA, att + k1, a.nk, nqr, kc1, tid);
            load_v(RB, k1, kc1);
        }
        if (k0 + kc - 1 <= a.q0 + i0) {  // every row of the tile sees the whole chunk
            mma_chunk_8x8(acc2, As[buf], Bs[buf], kc, ty, tx);
        } else {
            for (int k = 0; k < kc; ++k) {
                const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][8 * ty]);
                const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][8 * ty + 4]);
                const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(&Bs[buf][k][8 * tx]);
                const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(&Bs[buf][k][8 * tx + 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const uint64_t bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool on = k0 + k <= lim[i];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t nv = f2_add_swapped(acc2[i][q], f2_mul_bcast(av[i], bv[q]));
                        acc2[i][q] = on ? nv : acc2[i][q];
                    }
                }
            }
        }
        if (more) {
            store_rows_chunk_T(RA, As[buf ^ 1], tid);
            store_v(RB, Bs[buf ^ 1]);
        }
        __syncthreads();
    }
    float* mb = a.merged + ((size_t)b * a.nq + i0) * a.ldm + (size_t)h * a.dhc + c0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = 8 * ty + i;
        if (r >= nqr) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 8 * tx + 2 * q;
            if (col < ncol) mb[(size_t)r * a.ldm + col] = f2_hi(acc2[i][q]);
            if (col + 1 < ncol) mb[(size_t)r * a.ldm + col + 1] = f2_lo(acc2[i][q]);
        }
    }
}

// ---------------------------------------------------------------------------
// Launchers.
// ---------------------------------------------------------------------------
void launch_mla_scale_rope(scmoe_ctx* c, float* X, size_t ld, size_t rows, int n_a, float alpha_a,
                           int n_b, float alpha_b, int rc, int heads, int hd, const float2* table,
                           size_t pos0, size_t seq_len) {
    const size_t n = rows * ((size_t)n_a + n_b + (size_t)heads * (hd / 2));
    if (n == 0) return;
    const int threads = 256;
    const size_t blocks = std::min<size_t>(ceil_div(n, threads), (size_t)c->num_sms * 16);
    mla_scale_rope_kernel<<<(unsigned)blocks, threads, 0, c->stream>>>(
        X, ld, rows, n_a, alpha_a, n_b, alpha_b, rc, heads, hd, table, pos0, seq_len);
    SCMOE_LAUNCH_CHECK(c);
}

// ---------------------------------------------------------------------------
// Decode (one query row per (b, h)): a warp per softmax row and a CTA per
// head for PV -- the lane-per-row and tiled kernels above need many rows.
// Same arithmetic: max (order free), e = expf(s - max) with the normaliser
// summed in key order (each lane adds the chunk's 32 values in order, fed by
// shuffles), w = e / denom; PV chains over keys in order, one per column.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) mla_softmax_warp_kernel(float* __restrict__ att,
                                                               int rows_total, int nq, int nk,
                                                               int q0) {
    __shared__ uint64_t exp_tab[32];
    if (threadIdx.x < 32) exp_tab[threadIdx.x] = scmoe_exp2f_tab_dev[threadIdx.x];
    __syncthreads();
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= rows_total) return;
    const int n = min(nk, q0 + r % nq + 1);
    float* row = att + (size_t)r * nk;
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        float e = 0.f;
        if (j < n) {
            e = scmoe_expf_smem(__fsub_rn(row[j], mx), exp_tab);
            row[j] = e;
        }
        const int m = min(32, n - j0);
        for (int t = 0; t < m; ++t) sum = __fadd_rn(sum, __shfl_sync(0xffffffffu, e, t));
    }
    for (int j = lane; j < n; j += 32) row[j] = __fdiv_rn(row[j], sum);
}

// merged[b][h*dhc + p] = sum_j w[j] * v[j][p]; grid (B*H), dhc threads, the
// weight row staged in shared memory (n <= kPvRowMax).
constexpr int kPvRowMax = 12288;
__global__ void mla_pv_row_kernel(MlaAttnArgs a) {
    extern __shared__ float wrow[];
    const int bh = blockIdx.x, b = bh / a.H, h = bh % a.H;
    const int n = min(a.nk, a.q0 + 1);
    const float* att = a.att + (size_t)bh * a.nk;  // nq == 1
    for (int j = threadIdx.x; j < n; j += blockDim.x) wrow[j] = att[j];
    __syncthreads();
    const int p = threadIdx.x;
    if (p >= a.dhc) return;
    const float* v = a.v + (size_t)b * a.nk * a.ldkv + (size_t)h * a.dhc + p;
    float acc = 0.f;
    int j = 0;
    for (; j + 32 <= n; j += 32) {  // 32 value rows in flight per thread
        float vv[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) vv[u] = v[(size_t)(j + u) * a.ldkv];
#pragma unroll
        for (int u = 0; u < 32; ++u) acc = __fadd_rn(acc, __fmul_rn(wrow[j + u], vv[u]));
    }
    for (; j < n; ++j) acc = __fadd_rn(acc, __fmul_rn(wrow[j], v[(size_t)j * a.ldkv]));
    a.merged[(size_t)b * a.ldm + (size_t)h * a.dhc + p] = acc;
}

// out = a + b (fp32, rounded): the residual adds of build_layer (model.hpp:366, :390, :392).
__global__ void add_f32_kernel(const float4* __restrict__ a, const float4* __restrict__ b,
                               float4* __restrict__ out, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
        const float4 x = a[i], y = b[i];
        out[i] = make_float4(__fadd_rn(x.x, y.x), __fadd_rn(x.y, y.y), __fadd_rn(x.z, y.z),
                             __fadd_rn(x.w, y.w));
    }
}
__global__ void add_f32_tail_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                    float* __restrict__ out, size_t n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = __fadd_rn(a[i], b[i]);
}
void launch_add_f32(scmoe_ctx* c, const float* a, const float* b, size_t n, float* out) {
    if (n == 0) return;
    const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                       reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    const size_t n4 = vec ? n / 4 : 0;
    if (n4) {
        const size_t blocks = std::min<size_t>(ceil_div(n4, 256), (size_t)c->num_sms * 8);
        add_f32_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(
            reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(b),
            reinterpret_cast<float4*>(out), n4);
        SCMOE_LAUNCH_CHECK(c);
    }
    const size_t rem = n - 4 * n4;
    if (rem) {
        add_f32_tail_kernel<<<(unsigned)ceil_div(rem, 256), 256, 0, c->stream>>>(
            a + 4 * n4, b + 4 * n4, out + 4 * n4, rem);
        SCMOE_LAUNCH_CHECK(c);
    }
}

void launch_mla_attention(scmoe_ctx* c, const MlaAttnArgs& a, int batches) {
    const MlaAttnArgs& h = a;
    const unsigned z = (unsigned)(batches * h.H);
    static const bool tiles128 = [] {
        const char* e = getenv("SCMOE_MLA_TILE");
        return !(e && atoi(e) == 64);
    }();
    const bool huge = tiles128 && h.nq >= 128;
    const bool big = h.nq >= 64;
    {
        ProfScope _p(c, "mla_scores");
        if (huge) {
            dim3 grid((unsigned)ceil_div(h.nk, kBT), (unsigned)ceil_div(h.nq, kBT), z);
            mla_scores_big_kernel<<<grid, kBThreads, 0, c->stream>>>(a);
        } else if (big) {
            dim3 grid((unsigned)ceil_div(h.nk, kMlaTN), (unsigned)ceil_div(h.nq, 64), z);
            mla_scores_kernel<64, 4><<<grid, 256, 0, c->stream>>>(a);
        } else {
            dim3 grid((unsigned)ceil_div(h.nk, kMlaTN), (unsigned)ceil_div(h.nq, 16), z);
            mla_scores_kernel<16, 2><<<grid, 128, 0, c->stream>>>(a);
        }
        SCMOE_LAUNCH_CHECK(c);
    }
    const bool decode = h.nq == 1 && h.nk <= kPvRowMax && h.dhc <= 1024;
    if (decode) {
        {
            ProfScope _p(c, "mla_softmax");
            mla_softmax_warp_kernel<<<(unsigned)ceil_div((size_t)z * 32, 256), 256, 0, c->stream>>>(
                h.att, (int)z, 1, h.nk, h.q0);
            SCMOE_LAUNCH_CHECK(c);
        }
        ProfScope _p(c, "mla_pv");
        const size_t smem = (size_t)h.nk * sizeof(float);
        if (smem > 48 * 1024)
            ensure_max_dynamic_smem((const void*)mla_pv_row_kernel, (int)(kPvRowMax * sizeof(float)),
                                    c->device);
        mla_pv_row_kernel<<<z, (unsigned)((h.dhc + 31) / 32 * 32), smem, c->stream>>>(a);
        SCMOE_LAUNCH_CHECK(c);
        return;
    }
    {
        ProfScope _p(c, "mla_softmax");
        const size_t rows = (size_t)z * h.nq;
        mla_softmax_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, c->stream>>>(
            h.att, h.part_max, (int)rows, h.nq, h.nk, h.q0);
        SCMOE_LAUNCH_CHECK(c);
    }
    {
        ProfScope _p(c, "mla_pv");
        if (huge) {
            dim3 grid((unsigned)ceil_div(h.dhc, kBT), (unsigned)ceil_div(h.nq, kBT), z);
            mla_pv_big_kernel<<<grid, kBThreads, 0, c->stream>>>(a);
        } else if (big) {
            dim3 grid((unsigned)ceil_div(h.dhc, kMlaTN), (unsigned)ceil_div(h.nq, 64), z);
            mla_pv_kernel<64, 4><<<grid, 256, 0, c->stream>>>(a);
        } else {
            dim3 grid((unsigned)ceil_div(h.dhc, kMlaTN), (unsigned)ceil_div(h.nq, 16), z);
            mla_pv_kernel<16, 2><<<grid, 128, 0, c->stream>>>(a);
        }
        SCMOE_LAUNCH_CHECK(c);
    }
}

}  // namespace scmoe
