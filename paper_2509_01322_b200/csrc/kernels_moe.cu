// kernels_moe.cu -- permutation / histogram, row gather, combine, routing
// counters, bias controller, and weight preparation.
//
// Permutation follows moe_block (blocks.hpp:349-359): the tokens of expert e
// are listed in ascending token order and slot (t, s) gets its position in
// that list.  On the device the order is made deterministic without sorting:
// each block of 256 tokens builds, per expert, a 256-bit mask of the tokens
// that chose it (atomicOr is order independent), a slot's in-block rank is a
// popcount below its bit, and block offsets come from a scan over blocks.
#include "internal.cuh"
#include "libm_port.h"
#include "sm100_util.cuh"

namespace scmoe {

constexpr int kTB = kPermTokensPerBlock;  // tokens per permutation block
constexpr int kMaskWords = kTB / 32;

// Pass 1: in-block ranks and per-(block, expert) counts for all E experts.
__global__ void __launch_bounds__(kTB) perm_hist_kernel(const uint32_t* __restrict__ idx, int T,
                                                        int K, int E, int* __restrict__ rank_in_block,
                                                        int* __restrict__ block_counts,
                                                        int* __restrict__ dev_status,
                                                        const int* __restrict__ T_dev) {
    extern __shared__ uint32_t masks[];  // [E][kMaskWords]
    if (T_dev) {  // device-side token count (T = capacity): blocks past it have no work
        T = min(T, *T_dev);
        if ((int)blockIdx.x * kTB >= T) return;
    }
    for (int i = threadIdx.x; i < E * kMaskWords; i += blockDim.x) masks[i] = 0;
    __syncthreads();
    const int tl = threadIdx.x;
    const int t = blockIdx.x * kTB + tl;
    const int word = tl >> 5;
    const uint32_t bit = 1u << (tl & 31);
    if (t < T) {
        for (int s = 0; s < K; ++s) {
            const uint32_t e = idx[(size_t)t * K + s];
            if (e >= (uint32_t)E) {
                atomicExch(dev_status, DEV_ERR_INDEX_RANGE);
                continue;
            }
            atomicOr(&masks[e * kMaskWords + word], bit);
        }
    }
    __syncthreads();
    if (t < T) {
        for (int s = 0; s < K; ++s) {
            const uint32_t e = idx[(size_t)t * K + s];
            if (e >= (uint32_t)E) {
                rank_in_block[(size_t)t * K + s] = 0;
                continue;
            }
            const uint32_t* m = masks + e * kMaskWords;
            int r = __popc(m[word] & (bit - 1u));
            for (int w = 0; w < word; ++w) r += __popc(m[w]);
            rank_in_block[(size_t)t * K + s] = r;
        }
    }
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int cnt = 0;
#pragma unroll
        for (int w = 0; w < kMaskWords; ++w) cnt += __popc(masks[e * kMaskWords + w]);
        block_counts[(size_t)blockIdx.x * E + e] = cnt;
    }
}

// Block-wide exclusive scan helper (blockDim.x == 1024).
__device__ int block_exclusive_scan(int v, int* total) {
    __shared__ int warp_sums[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    const int excl = x - v + (warp > 0 ? warp_sums[warp - 1] : 0);
    *total = warp_sums[31];
    __syncthreads();
    return excl;
}

// Pass 2 (one block of 1024 threads): per-expert block offsets, expert
// totals, FFN expert bases (exclusive scan) and the GEMM token-tile list.
__global__ void __launch_bounds__(1024) perm_scan_kernel(int nblk, int E, int n_ffn,
                                                         int tile_rows, int* __restrict__ block_counts,
                                                         int* __restrict__ expert_count,
                                                         int* __restrict__ expert_base,
                                                         TokenTile* __restrict__ tiles,
                                                         int* __restrict__ n_tiles,
                                                         const int* __restrict__ T_dev) {
    if (T_dev) nblk = min(nblk, (*T_dev + kTB - 1) / kTB);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int run = 0;
        for (int b = 0; b < nblk; ++b) {
            const int cnt = block_counts[(size_t)b * E + e];
            block_counts[(size_t)b * E + e] = run;
            run += cnt;
        }
        expert_count[e] = run;
    }
    __syncthreads();
    // Chunked scan over the FFN experts: thread i owns experts [i*per, (i+1)*per).
    const int per = (n_ffn + blockDim.x - 1) / blockDim.x;
    const int e0 = threadIdx.x * per, e1 = min(n_ffn, e0 + per);
    int my_rows = 0, my_tiles = 0;
    for (int e = e0; e < e1; ++e) {
        my_rows += expert_count[e];
        my_tiles += (expert_count[e] + tile_rows - 1) / tile_rows;
    }
    int total_rows, total_tiles;
    int row_base = block_exclusive_scan(my_rows, &total_rows);
    int tile_base = block_exclusive_scan(my_tiles, &total_tiles);
    for (int e = e0; e < e1; ++e) {
        expert_base[e] = row_base;
        const int cnt = expert_count[e];
        const int nt = (cnt + tile_rows - 1) / tile_rows;
        // equal tiles (multiples of 16 rows): 256 tokens -> 2 x 128, not 192 + 64
        const int step = nt > 1 ? min(tile_rows, ((cnt + nt - 1) / nt + 15) & ~15) : tile_rows;
        for (int r = 0, k = 0; r < cnt; r += step, ++k) {
            TokenTile tt;
            tt.e = e;
            tt.pos = row_base + r;
            tt.count = min(step, cnt - r);
            tt.pad = (k << 16) | nt;  // position in the expert's tiles | their count
            tiles[tile_base++] = tt;
        }
        row_base += cnt;
    }
    if (threadIdx.x == 0) {
        expert_base[n_ffn] = total_rows;
        *n_tiles = total_tiles;
    }
}

// Pass 3: slot -> permuted row position, and row -> source token.
__global__ void perm_scatter_kernel(const uint32_t* __restrict__ idx, int T, int K, int E,
                                    int n_ffn, const int* __restrict__ rank_in_block,
                                    const int* __restrict__ block_offsets,
                                    const int* __restrict__ expert_base, int* __restrict__ slot_pos,
                                    int* __restrict__ row_token, const int* __restrict__ T_dev) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (T_dev) T = min(T, *T_dev);
    if (i >= (size_t)T * K) return;
    const int t = (int)(i / K);
    const uint32_t e = idx[i];
    if (e >= (uint32_t)n_ffn) {
        slot_pos[i] = -1;
        return;
    }
    const int b = t / kTB;
    const int pos = expert_base[e] + block_offsets[(size_t)b * E + e] + rank_in_block[i];
    slot_pos[i] = pos;
    row_token[pos] = t;
}

// Pass 1 for bins a token may hit several times (expert-parallel destination
// ranks): slot (t, s) -> bin b gets in-block rank = (slots of bin b in earlier
// tokens of the block) + (earlier slots of token t in bin b); a block scan
// over the 256 tokens per bin replaces the bitmask.  E <= kMaxMultiBins.
constexpr int kMaxMultiBins = 33;

__global__ void __launch_bounds__(kTB) perm_hist_multi_kernel(
    const uint32_t* __restrict__ idx, int T, int K, int E, int* __restrict__ rank_in_block,
    int* __restrict__ block_counts, int* __restrict__ dev_status) {
    __shared__ int warp_tot[kTB / 32];
    const int tl = threadIdx.x;
    const int t = blockIdx.x * kTB + tl;
    const int lane = tl & 31, warp = tl >> 5;
    for (int b = 0; b < E; ++b) {
        int cnt = 0;
        if (t < T)
            for (int s = 0; s < K; ++s) cnt += idx[(size_t)t * K + s] == (uint32_t)b;
        // block exclusive scan of cnt over tokens
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < kTB / 32; ++w) {
            if (w < warp) before += warp_tot[w];
            total += warp_tot[w];
        }
        const int excl = before + incl - cnt;
        if (t < T) {
            int within = 0;
            for (int s = 0; s < K; ++s) {
                const uint32_t e = idx[(size_t)t * K + s];
                if (e == (uint32_t)b) rank_in_block[(size_t)t * K + s] = excl + within++;
            }
        }
        if (tl == 0) block_counts[(size_t)blockIdx.x * E + b] = total;
        __syncthreads();
    }
    if (t < T)
        for (int s = 0; s < K; ++s)
            if (idx[(size_t)t * K + s] >= (uint32_t)E) {
                atomicExch(dev_status, DEV_ERR_INDEX_RANGE);
                rank_in_block[(size_t)t * K + s] = 0;
            }
}

// Small batches (T <= 1024 tokens, E <= 64 experts): the three passes in one
// CTA of 1024 threads (one token each), the same results -- per-expert token
// bitmask ranks (tokens ascending, blocks.hpp:349-359), expert counts, FFN
// bases, equal-width token tiles, slot positions and row tokens.
constexpr int kSmallPermT = 1024, kSmallPermE = 64;

__global__ void __launch_bounds__(1024) perm_small_kernel(
    const uint32_t* __restrict__ idx, int T, int K, int E, int n_ffn, int tile_rows,
    int* __restrict__ expert_count, int* __restrict__ expert_base, TokenTile* __restrict__ tiles,
    int* __restrict__ n_tiles, int* __restrict__ slot_pos, int* __restrict__ row_token,
    int* __restrict__ dev_status) {
    constexpr int W = kSmallPermT / 32;
    __shared__ uint32_t masks[kSmallPermE * W];
    __shared__ int cnt_s[kSmallPermE], base_s[kSmallPermE + 1];
    const int t = threadIdx.x, word = t >> 5;
    const uint32_t bit = 1u << (t & 31);
    for (int i = t; i < E * W; i += blockDim.x) masks[i] = 0;
    __syncthreads();
    if (t < T)
        for (int s = 0; s < K; ++s) {
            const uint32_t e = idx[(size_t)t * K + s];
            if (e >= (uint32_t)E) {
                atomicExch(dev_status, DEV_ERR_INDEX_RANGE);
                continue;
            }
            atomicOr(&masks[e * W + word], bit);
        }
    __syncthreads();
    for (int e = t; e < E; e += blockDim.x) {
        int n = 0;
        for (int w = 0; w < W; ++w) n += __popc(masks[e * W + w]);
        cnt_s[e] = n;
        expert_count[e] = n;
    }
    __syncthreads();
    if (t == 0) {  // FFN bases and the tile list (n_ffn <= 64: serial is cheap)
        int row = 0, nt_all = 0;
        for (int e = 0; e < n_ffn; ++e) {
            base_s[e] = row;
            expert_base[e] = row;
            const int cnt = cnt_s[e];
            const int nt = (cnt + tile_rows - 1) / tile_rows;
            const int step = nt > 1 ? min(tile_rows, ((cnt + nt - 1) / nt + 15) & ~15) : tile_rows;
            for (int r = 0, k = 0; r < cnt; r += step, ++k)
                tiles[nt_all++] = TokenTile{e, row + r, min(step, cnt - r), (k << 16) | nt};
            row += cnt;
        }
        base_s[n_ffn] = row;
        expert_base[n_ffn] = row;
        *n_tiles = nt_all;
    }
    __syncthreads();
    if (t < T)
        for (int s = 0; s < K; ++s) {
            const size_t i = (size_t)t * K + s;
            const uint32_t e = idx[i];
            if (e >= (uint32_t)n_ffn) {
                slot_pos[i] = -1;
                continue;
            }
            const uint32_t* m = masks + e * W;
            int r = __popc(m[word] & (bit - 1u));
            for (int w = 0; w < word; ++w) r += __popc(m[w]);
            const int pos = base_s[e] + r;
            slot_pos[i] = pos;
            row_token[pos] = t;
        }
}

PermResult launch_permute(scmoe_ctx* c, const uint32_t* idx, size_t T, size_t K, size_t n_ffn,
                          size_t E, int tile_rows, bool multi, const int* T_dev) {
    Workspace& ws = c->ws;
    if (multi) SCMOE_CHECK_ARG(E <= kMaxMultiBins, SCMOE_ERR_CONFIG, "permute: too many bins");
    const size_t nblk = ceil_div(std::max<size_t>(T, 1), kTB);
    PermResult pr;
    int* rank = ws.rank_in_block.get<int>(T * K);
    int* bcounts = ws.block_counts.get<int>(nblk * E);
    pr.expert_count = ws.expert_count.get<int>(E);
    pr.expert_base = ws.expert_base.get<int>(n_ffn + 1);
    pr.slot_pos = ws.slot_pos.get<int>(T * K);
    pr.row_token = ws.row_token.get<int>(T * K);
    pr.max_tiles = ceil_div(T * K, tile_rows) + n_ffn;
    pr.tiles = ws.tiles.get<TokenTile>(pr.max_tiles);
    pr.n_tiles = ws.n_tiles.get<int>(1);
    if (!multi && !T_dev && T > 0 && T <= (size_t)kSmallPermT && E <= (size_t)kSmallPermE) {
        perm_small_kernel<<<1, kSmallPermT, 0, c->stream>>>(
            idx, (int)T, (int)K, (int)E, (int)n_ffn, tile_rows, pr.expert_count, pr.expert_base,
            pr.tiles, pr.n_tiles, pr.slot_pos, pr.row_token, c->dev_status);
        SCMOE_LAUNCH_CHECK(c);
        return pr;
    }
    const size_t smem = E * kMaskWords * sizeof(uint32_t);
    SCMOE_CHECK_ARG(smem <= 200 * 1024, SCMOE_ERR_CONFIG, "permute: too many experts");
    if (smem > 48 * 1024)
        SCMOE_CUDA(cudaFuncSetAttribute(perm_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    SCMOE_CHECK_ARG(!(multi && T_dev), SCMOE_ERR_INTERNAL, "permute: device count needs single bins");
    if (T > 0 && multi) {
        perm_hist_multi_kernel<<<nblk, kTB, 0, c->stream>>>(idx, (int)T, (int)K, (int)E, rank,
                                                            bcounts, c->dev_status);
        SCMOE_LAUNCH_CHECK(c);
    } else if (T > 0) {
        perm_hist_kernel<<<nblk, kTB, smem, c->stream>>>(idx, (int)T, (int)K, (int)E, rank, bcounts,
                                                         c->dev_status, T_dev);
        SCMOE_LAUNCH_CHECK(c);
    } else {
        SCMOE_CUDA(cudaMemsetAsync(bcounts, 0, nblk * E * sizeof(int), c->stream));
    }
    perm_scan_kernel<<<1, 1024, 0, c->stream>>>((int)nblk, (int)E, (int)n_ffn, tile_rows, bcounts,
                                                pr.expert_count, pr.expert_base, pr.tiles,
                                                pr.n_tiles, T_dev);
    SCMOE_LAUNCH_CHECK(c);
    if (T > 0) {
        perm_scatter_kernel<<<ceil_div(T * K, 256), 256, 0, c->stream>>>(
            idx, (int)T, (int)K, (int)E, (int)n_ffn, rank, bcounts, pr.expert_base, pr.slot_pos,
            pr.row_token, T_dev);
        SCMOE_LAUNCH_CHECK(c);
    }
    return pr;
}

// Row gather into the permuted order: dst[pos] = src[row_token[pos]] (bf16,
// 16-byte vectors; one warp per row).  Rows past the total are skipped.
__global__ void gather_bf16_kernel(const __nv_bfloat16* __restrict__ src, int d,
                                   const int* __restrict__ row_token,
                                   const int* __restrict__ total_rows, int max_rows,
                                   __nv_bfloat16* __restrict__ dst) {
    const int total = *total_rows;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int vec = d / 8;
    for (int pos = warp; pos < total && pos < max_rows; pos += nwarps) {
        const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)row_token[pos] * d);
        uint4* o = reinterpret_cast<uint4*>(dst + (size_t)pos * d);
        for (int v = lane; v < vec; v += 32) o[v] = s[v];
    }
}

void launch_gather_bf16(scmoe_ctx* c, const __nv_bfloat16* src, size_t d, const int* row_token,
                        const int* expert_base, size_t n_ffn, size_t max_rows,
                        __nv_bfloat16* dst) {
    if (max_rows == 0) return;
    SCMOE_CHECK_ARG(d % 8 == 0, SCMOE_ERR_DIMENSION, "gather: d must be a multiple of 8");
    const int blocks = c->num_sms * 8;
    gather_bf16_kernel<<<blocks, 256, 0, c->stream>>>(src, (int)d, row_token, expert_base + n_ffn,
                                                      (int)max_rows, dst);
    SCMOE_LAUNCH_CHECK(c);
}

// ---------------------------------------------------------------------------
// Combine -- moe_combine forward (blocks.hpp:226-274) + residual
// (model.hpp:400).  One block per token, threads over columns.  For slots in
// rank order: FFN out += (g_ffn*w)*y[pos]; zero zero_w += w; then
// out += (g_zero*zero_w)*x when zero_w != 0; finally out = residual + out.
// w = (float)gate / denom with denom = 1 or the rank-order gate sum.
// ---------------------------------------------------------------------------
template <typename Y>
__device__ __forceinline__ float load_y(const Y* p);
template <>
__device__ __forceinline__ float load_y<float>(const float* p) {
    return *p;
}
template <>
__device__ __forceinline__ float load_y<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}

constexpr int kMaxK = 64;

template <typename Y>
__global__ void __launch_bounds__(256) combine_kernel(
    const float* __restrict__ x, const Y* __restrict__ y, const uint32_t* __restrict__ idx,
    const double* __restrict__ gates, const int* __restrict__ slot_pos, int d, int K, int n_ffn,
    float gamma_ffn, float gamma_zero, int renorm, const float* __restrict__ residual,
    float* __restrict__ out) {
    __shared__ float coeff[kMaxK];
    __shared__ int rowpos[kMaxK];
    __shared__ int nffn, use_zero;
    __shared__ float zcoeff;
    const int t = blockIdx.x;
    if (threadIdx.x == 0) {
        float denom = 1.0f;
        if (renorm) {
            float s = 0.0f;
            for (int sl = 0; sl < K; ++sl) s = __fadd_rn(s, (float)gates[(size_t)t * K + sl]);
            denom = s;
        }
        float zero_w = 0.0f;
        int n = 0;
        for (int sl = 0; sl < K; ++sl) {
            const uint32_t e = idx[(size_t)t * K + sl];
            const float w = __fdiv_rn((float)gates[(size_t)t * K + sl], denom);
            if (e < (uint32_t)n_ffn) {
                coeff[n] = __fmul_rn(gamma_ffn, w);
                rowpos[n] = slot_pos[(size_t)t * K + sl];
                ++n;
            } else {
                zero_w = __fadd_rn(zero_w, w);
            }
        }
        nffn = n;
        // zero_w == 0 skips the identity term entirely (blocks.hpp:266)
        use_zero = zero_w != 0.0f;
        zcoeff = __fmul_rn(gamma_zero, zero_w);
    }
    __syncthreads();
    const int n = nffn;
    const float zc = zcoeff;
    const bool uz = use_zero != 0;
    const float* xr = x + (size_t)t * d;
    float* orow = out + (size_t)t * d;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        float acc = 0.0f;
        for (int s = 0; s < n; ++s)
            acc = __fadd_rn(acc, __fmul_rn(coeff[s], load_y(y + (size_t)rowpos[s] * d + j)));
        if (uz) acc = __fadd_rn(acc, __fmul_rn(zc, xr[j]));
        if (residual) acc = __fadd_rn(residual[(size_t)t * d + j], acc);
        orow[j] = acc;
    }
}

template <typename Y>
static void launch_combine_impl(scmoe_ctx* c, const float* x, const Y* y, const uint32_t* idx,
                                const double* gates, const int* slot_pos, size_t T, size_t d,
                                size_t K, size_t n_ffn, float gamma_ffn, float gamma_zero,
                                int renorm, const float* residual, float* out) {
    if (T == 0) return;
    SCMOE_CHECK_ARG(K <= kMaxK, SCMOE_ERR_CONFIG, "combine: top_k too large");
    combine_kernel<Y><<<T, 256, 0, c->stream>>>(x, y, idx, gates, slot_pos, (int)d, (int)K,
                                                (int)n_ffn, gamma_ffn, gamma_zero, renorm,
                                                residual, out);
    SCMOE_LAUNCH_CHECK(c);
}

// moe_combine forward in S = double (blocks.hpp:226-274), same order as the
// fp32 kernel: w = gate / denom, FFN out += (g_ffn*w)*y, zero_w += w, then the
// identity term and the residual.
__global__ void __launch_bounds__(256) combine_f64_kernel(
    const double* __restrict__ x, const double* __restrict__ y, const uint32_t* __restrict__ idx,
    const double* __restrict__ gates, const int* __restrict__ slot_pos, int d, int K, int n_ffn,
    double gamma_ffn, double gamma_zero, int renorm, const double* __restrict__ residual,
    double* __restrict__ out) {
    __shared__ double coeff[kMaxK];
    __shared__ int rowpos[kMaxK];
    __shared__ int nffn, use_zero;
    __shared__ double zcoeff;
    const int t = blockIdx.x;
    if (threadIdx.x == 0) {
        double denom = 1.0;
        if (renorm) {
            double s = 0.0;
            for (int sl = 0; sl < K; ++sl) s = __dadd_rn(s, gates[(size_t)t * K + sl]);
            denom = s;
        }
        double zero_w = 0.0;
        int n = 0;
        for (int sl = 0; sl < K; ++sl) {
            const uint32_t e = idx[(size_t)t * K + sl];
            const double w = __ddiv_rn(gates[(size_t)t * K + sl], denom);
            if (e < (uint32_t)n_ffn) {
                coeff[n] = __dmul_rn(gamma_ffn, w);
                rowpos[n] = slot_pos[(size_t)t * K + sl];
                ++n;
            } else {
                zero_w = __dadd_rn(zero_w, w);
            }
        }
        nffn = n;
        use_zero = zero_w != 0.0;
        zcoeff = __dmul_rn(gamma_zero, zero_w);
    }
    __syncthreads();
    const int n = nffn;
    const double zc = zcoeff;
    const bool uz = use_zero != 0;
    const double* xr = x + (size_t)t * d;
    double* orow = out + (size_t)t * d;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < n; ++s)
            acc = __dadd_rn(acc, __dmul_rn(coeff[s], y[(size_t)rowpos[s] * d + j]));
        if (uz) acc = __dadd_rn(acc, __dmul_rn(zc, xr[j]));
        if (residual) acc = __dadd_rn(residual[(size_t)t * d + j], acc);
        orow[j] = acc;
    }
}
void launch_combine_f64(scmoe_ctx* c, const double* x, const double* y, const uint32_t* idx,
                        const double* gates, const int* slot_pos, size_t T, size_t d, size_t K,
                        size_t n_ffn, double gamma_ffn, double gamma_zero, int renorm,
                        const double* residual, double* out) {
    if (T == 0) return;
    SCMOE_CHECK_ARG(K <= kMaxK, SCMOE_ERR_CONFIG, "combine: top_k too large");
    combine_f64_kernel<<<T, 256, 0, c->stream>>>(x, y, idx, gates, slot_pos, (int)d, (int)K,
                                                 (int)n_ffn, gamma_ffn, gamma_zero, renorm,
                                                 residual, out);
    SCMOE_LAUNCH_CHECK(c);
}

void launch_combine_f32(scmoe_ctx* c, const float* x, const float* y, const uint32_t* idx,
                        const double* gates, const int* slot_pos, size_t T, size_t d, size_t K,
                        size_t n_ffn, float gamma_ffn, float gamma_zero, int renorm,
                        const float* residual, float* out) {
    launch_combine_impl<float>(c, x, y, idx, gates, slot_pos, T, d, K, n_ffn, gamma_ffn,
                               gamma_zero, renorm, residual, out);
}
// bf16 expert rows, 8 columns per thread per step (16-byte Y loads, 2x float4
// for x / residual / out).  Same per-element operation order as above.
__global__ void __launch_bounds__(256) combine_bf16_vec8_kernel(
    const float* __restrict__ x, const __nv_bfloat16* __restrict__ y,
    const uint32_t* __restrict__ idx, const double* __restrict__ gates,
    const int* __restrict__ slot_pos, int d, int K, int n_ffn, float gamma_ffn, float gamma_zero,
    int renorm, const float* __restrict__ residual, float* __restrict__ out) {
    __shared__ float coeff[kMaxK];
    __shared__ int rowpos[kMaxK];
    __shared__ int nffn, use_zero;
    __shared__ float zcoeff;
    const int t = blockIdx.x;
    if (threadIdx.x == 0) {
        float denom = 1.0f;
        if (renorm) {
            float s = 0.0f;
            for (int sl = 0; sl < K; ++sl) s = __fadd_rn(s, (float)gates[(size_t)t * K + sl]);
            denom = s;
        }
        float zero_w = 0.0f;
        int n = 0;
        for (int sl = 0; sl < K; ++sl) {
            const uint32_t e = idx[(size_t)t * K + sl];
            const float w = __fdiv_rn((float)gates[(size_t)t * K + sl], denom);
            if (e < (uint32_t)n_ffn) {
                coeff[n] = __fmul_rn(gamma_ffn, w);
                rowpos[n] = slot_pos[(size_t)t * K + sl];
                ++n;
            } else {
                zero_w = __fadd_rn(zero_w, w);
            }
        }
        nffn = n;
        use_zero = zero_w != 0.0f;
        zcoeff = __fmul_rn(gamma_zero, zero_w);
    }
    __syncthreads();
    const int n = nffn;
    const float zc = zcoeff;
    const bool uz = use_zero != 0;
    const int d8 = d / 8;
    for (int v = threadIdx.x; v < d8; v += blockDim.x) {
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
        for (int s = 0; s < n; ++s) {
            const uint4 raw = reinterpret_cast<const uint4*>(y + (size_t)rowpos[s] * d)[v];
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(h[q]);
                acc[2 * q] = __fadd_rn(acc[2 * q], __fmul_rn(coeff[s], f.x));
                acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], __fmul_rn(coeff[s], f.y));
            }
        }
        if (uz) {
            const float4* xr = reinterpret_cast<const float4*>(x + (size_t)t * d) + 2 * v;
            const float4 a = xr[0], b = xr[1];
            const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(zc, xv[q]));
        }
        if (residual) {
            const float4* rr = reinterpret_cast<const float4*>(residual + (size_t)t * d) + 2 * v;
            const float4 a = rr[0], b = rr[1];
            const float rv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(rv[q], acc[q]);
        }
        float4* o = reinterpret_cast<float4*>(out + (size_t)t * d) + 2 * v;
        o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

void launch_combine_bf16(scmoe_ctx* c, const float* x, const __nv_bfloat16* y,
                         const uint32_t* idx, const double* gates, const int* slot_pos, size_t T,
                         size_t d, size_t K, size_t n_ffn, float gamma_ffn, float gamma_zero,
                         int renorm, const float* residual, float* out) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) |
                           reinterpret_cast<uintptr_t>(residual) | reinterpret_cast<uintptr_t>(y)) &
                          15) == 0;
    if (d % 8 == 0 && aligned && T > 0) {
        SCMOE_CHECK_ARG(K <= kMaxK, SCMOE_ERR_CONFIG, "combine: top_k too large");
        combine_bf16_vec8_kernel<<<T, 256, 0, c->stream>>>(x, y, idx, gates, slot_pos, (int)d,
                                                           (int)K, (int)n_ffn, gamma_ffn,
                                                           gamma_zero, renorm, residual, out);
        SCMOE_LAUNCH_CHECK(c);
        return;
    }
    launch_combine_impl<__nv_bfloat16>(c, x, y, idx, gates, slot_pos, T, d, K, n_ffn, gamma_ffn,
                                       gamma_zero, renorm, residual, out);
}

// ---------------------------------------------------------------------------
// Index validation (blocks.hpp:375-377) and counters (router.hpp:144-150).
// ---------------------------------------------------------------------------
__global__ void check_indices_kernel(const uint32_t* __restrict__ idx, size_t n, uint32_t E,
                                     int* __restrict__ dev_status) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && idx[i] >= E) atomicExch(dev_status, DEV_ERR_INDEX_RANGE);
}

void launch_check_indices(scmoe_ctx* c, const uint32_t* idx, size_t n, size_t E) {
    if (n == 0) return;
    check_indices_kernel<<<ceil_div(n, 256), 256, 0, c->stream>>>(idx, n, (uint32_t)E,
                                                                 c->dev_status);
    SCMOE_LAUNCH_CHECK(c);
}

__global__ void accumulate_kernel(const uint32_t* __restrict__ idx, size_t n, uint32_t E,
                                  unsigned long long* __restrict__ routed,
                                  int* __restrict__ dev_status) {
    extern __shared__ unsigned int hist[];
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
    __syncthreads();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t e = idx[i];
        if (e < E)
            atomicAdd(&hist[e], 1u);
        else
            atomicExch(dev_status, DEV_ERR_INDEX_RANGE);
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x)
        if (hist[e]) atomicAdd(&routed[e], (unsigned long long)hist[e]);
}

// RoutingDecision::mean_ffn / std_ffn (router.hpp:73-86): sequential double
// sums in token order (the order fixes the rounding of the second one), one
// thread -- T dependent adds, ~30 us at T = 8192.
__global__ void ffn_moments_kernel(const uint32_t* __restrict__ cnt, size_t T,
                                   double* __restrict__ out) {
    double m = 0.0, sd = 0.0;
    if (T) {
        double s = 0.0;
        for (size_t t = 0; t < T; ++t) s = __dadd_rn(s, (double)cnt[t]);
        m = __ddiv_rn(s, (double)T);
        double s2 = 0.0;
        for (size_t t = 0; t < T; ++t) {
            const double dlt = __dsub_rn((double)cnt[t], m);
            s2 = __dadd_rn(s2, __dmul_rn(dlt, dlt));
        }
        sd = __dsqrt_rn(__ddiv_rn(s2, (double)T));
    }
    out[0] = m;
    out[1] = sd;
}
void launch_ffn_moments(scmoe_ctx* c, const uint32_t* cnt, size_t T, double* out) {
    ffn_moments_kernel<<<1, 1, 0, c->stream>>>(cnt, T, out);
    SCMOE_LAUNCH_CHECK(c);
}

void launch_accumulate(scmoe_ctx* c, const uint32_t* idx, size_t n, size_t E, uint64_t* routed) {
    if (n == 0) return;
    const int blocks = (int)std::min<size_t>(ceil_div(n, 1024), (size_t)c->num_sms * 2);
    accumulate_kernel<<<blocks, 1024, E * sizeof(unsigned int), c->stream>>>(
        idx, n, (uint32_t)E, reinterpret_cast<unsigned long long*>(routed), c->dev_status);
    SCMOE_LAUNCH_CHECK(c);
}

// bias_update (router.hpp:155-176), double arithmetic with explicit rounding
// so nothing is contracted: load = T_i / (K*T_all); delta = mu*(target-load);
// b += delta; counters reset.  Counter coverage is validated first.
__global__ void bias_update_kernel(int n_ffn, int E, int top_k, int k_expected, double mu,
                                   unsigned long long tokens_seen, double* __restrict__ b,
                                   unsigned long long* __restrict__ routed,
                                   double* __restrict__ delta, int* __restrict__ dev_status,
                                   const unsigned long long* __restrict__ seen_dev) {
    __shared__ unsigned long long total;
    if (seen_dev) {  // tokens_seen summed over the ranks on the device (expert parallelism)
        tokens_seen = *seen_dev;
        if (tokens_seen == 0) {  // router.hpp:157
            if (threadIdx.x == 0) atomicExch(dev_status, DEV_ERR_EMPTY);
            return;
        }
    }
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int i = 0; i < E; ++i) s += routed[i];
        total = s;
    }
    __syncthreads();
    if (total != (unsigned long long)top_k * tokens_seen) {
        if (threadIdx.x == 0) atomicExch(dev_status, DEV_ERR_COUNTERS);
        return;
    }
    const double t_all = (double)tokens_seen;
    const double target = __ddiv_rn((double)k_expected, __dmul_rn((double)top_k, (double)n_ffn));
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
        double dl = 0.0;
        if (i < n_ffn) {
            const double load = __ddiv_rn((double)routed[i], __dmul_rn((double)top_k, t_all));
            dl = __dmul_rn(mu, __dsub_rn(target, load));
            b[i] = __dadd_rn(b[i], dl);
        }
        if (delta) delta[i] = dl;
        routed[i] = 0;
    }
}

void launch_bias_update(scmoe_ctx* c, scmoe_router* r, double* delta_dev,
                        const uint64_t* routed, const uint64_t* seen_dev) {
    bias_update_kernel<<<1, 256, 0, c->stream>>>((int)r->n_ffn, (int)r->E(), (int)r->top_k,
                                                 (int)r->k_expected, r->mu,
                                                 (unsigned long long)r->tokens_seen, r->b,
                                                 reinterpret_cast<unsigned long long*>(
                                                     const_cast<uint64_t*>(routed ? routed : r->routed)),
                                                 delta_dev, c->dev_status,
                                                 reinterpret_cast<const unsigned long long*>(seen_dev));
    SCMOE_LAUNCH_CHECK(c);
}

// ---------------------------------------------------------------------------
// Synthetic weights: seeded_init Uniform (rng.hpp:89-94) on the device,
// bitwise equal to the host: u = ((h >> 11) + 1) * 2^-53 is exact, then
// (2u - 1) * half_width with separately rounded double ops.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t d_mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}
__device__ __forceinline__ float d_uniform_init(uint64_t seed_mix, uint64_t ctr, double hw) {
    const uint64_t h = d_mix64(seed_mix ^ d_mix64(ctr + 0xbf58476d1ce4e5b9ULL));
    const double u = __dmul_rn((double)(h >> 11) + 1.0, 0x1.0p-53);
    return (float)__dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), hw);
}

__global__ void uniform_init_kernel(uint64_t seed_mix, uint64_t first, size_t n, double hw,
                                    float* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = d_uniform_init(seed_mix, first + i, hw);
}

static uint64_t host_mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

void launch_uniform_init(scmoe_ctx* c, uint64_t seed, uint64_t first, size_t n, double half_width,
                         float* out) {
    if (n == 0) return;
    const uint64_t seed_mix = host_mix64(seed + 0x9e3779b97f4a7c15ULL);
    uniform_init_kernel<<<c->num_sms * 16, 256, 0, c->stream>>>(seed_mix, first, n, half_width, out);
    SCMOE_LAUNCH_CHECK(c);
}

// Uniform init of a [rows, cols] row-major matrix, written transposed as
// bf16 [cols, rows] (the K-major layout the tcgen05 GEMM reads).
__global__ void uniform_init_bf16_t_kernel(uint64_t seed_mix, int rows, int cols, double hw,
                                           __nv_bfloat16* __restrict__ out_t) {
    __shared__ float tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, cc = c0 + threadIdx.x;
        if (r < rows && cc < cols)
            tile[i][threadIdx.x] = d_uniform_init(seed_mix, (uint64_t)r * cols + cc, hw);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int cc = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && cc < cols)
            out_t[wblk_index(cc, r, rows)] = __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
}

void launch_uniform_init_bf16_t(scmoe_ctx* c, uint64_t seed, size_t rows, size_t cols,
                                double half_width, __nv_bfloat16* out_t) {
    const uint64_t seed_mix = host_mix64(seed + 0x9e3779b97f4a7c15ULL);
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
    uniform_init_bf16_t_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(seed_mix, (int)rows, (int)cols,
                                                                   half_width, out_t);
    SCMOE_LAUNCH_CHECK(c);
}

__global__ void f32_to_bf16_t_kernel(const float* __restrict__ src, int rows, int cols,
                                     __nv_bfloat16* __restrict__ dst_t, int n_a, float alpha_a,
                                     int n_b, float alpha_b) {
    __shared__ float tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, cc = c0 + threadIdx.x;
        if (r < rows && cc < cols) tile[i][threadIdx.x] = src[(size_t)r * cols + cc];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int cc = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && cc < cols) {
            // optional column scales (folded output scalings): [0, n_a) by
            // alpha_a, [n_a, n_a + n_b) by alpha_b
            const float sc = cc < n_a ? alpha_a : (cc < n_a + n_b ? alpha_b : 1.f);
            dst_t[wblk_index(cc, r, rows)] = __float2bfloat16_rn(tile[threadIdx.x][i] * sc);
        }
    }
}

void launch_f32_to_bf16_t(scmoe_ctx* c, const float* src, size_t rows, size_t cols,
                          __nv_bfloat16* dst_t, int n_a, float alpha_a, int n_b, float alpha_b) {
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
    f32_to_bf16_t_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(src, (int)rows, (int)cols, dst_t,
                                                               n_a, alpha_a, n_b, alpha_b);
    SCMOE_LAUNCH_CHECK(c);
}

__global__ void cast_bf16_kernel(const float* __restrict__ src, size_t n,
                                 __nv_bfloat16* __restrict__ dst) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

void launch_cast_bf16(scmoe_ctx* c, const float* src, size_t n, __nv_bfloat16* dst) {
    if (n == 0) return;
    cast_bf16_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(src, n, dst);
    SCMOE_LAUNCH_CHECK(c);
}

// One group, consecutive row tiles (router projection, router.hpp:136).
__global__ void row_tiles_kernel(int rows, int tile_rows, TokenTile* __restrict__ tiles,
                                 int* __restrict__ n_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = (rows + tile_rows - 1) / tile_rows;
    if (i < n) tiles[i] = TokenTile{0, i * tile_rows, min(tile_rows, rows - i * tile_rows), 0};
    if (i == 0 && n_out) *n_out = n;
}

void launch_row_tiles(scmoe_ctx* c, size_t rows, int tile_rows, TokenTile* tiles, int* n_out) {
    const size_t n = ceil_div(rows, tile_rows);
    if (n == 0) return;
    row_tiles_kernel<<<ceil_div(n, 256), 256, 0, c->stream>>>((int)rows, tile_rows, tiles, n_out);
    SCMOE_LAUNCH_CHECK(c);
}

// out = a + float(y) (fp32 add, round to nearest): the dense branch's
// residual dd = a1 + ffn(rmsnorm(a1)) (model.hpp:390-391).
__global__ void add_bf16_residual_kernel(const float* __restrict__ a,
                                         const __nv_bfloat16* __restrict__ y, size_t n8,
                                         float* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 yv = reinterpret_cast<const uint4*>(y)[i];
        const float4 a0 = reinterpret_cast<const float4*>(a)[2 * i];
        const float4 a1 = reinterpret_cast<const float4*>(a)[2 * i + 1];
        const __nv_bfloat162* yb = reinterpret_cast<const __nv_bfloat162*>(&yv);
        const float2 y0 = __bfloat1622float2(yb[0]), y1 = __bfloat1622float2(yb[1]);
        const float2 y2 = __bfloat1622float2(yb[2]), y3 = __bfloat1622float2(yb[3]);
        reinterpret_cast<float4*>(out)[2 * i] =
            make_float4(__fadd_rn(a0.x, y0.x), __fadd_rn(a0.y, y0.y), __fadd_rn(a0.z, y1.x),
                        __fadd_rn(a0.w, y1.y));
        reinterpret_cast<float4*>(out)[2 * i + 1] =
            make_float4(__fadd_rn(a1.x, y2.x), __fadd_rn(a1.y, y2.y), __fadd_rn(a1.z, y3.x),
                        __fadd_rn(a1.w, y3.y));
    }
}

void launch_add_bf16_residual(scmoe_ctx* c, const float* a, const __nv_bfloat16* y, size_t n,
                              float* out) {
    SCMOE_CHECK_ARG(n % 8 == 0, SCMOE_ERR_DIMENSION, "residual add: size must be a multiple of 8");
    if (n == 0) return;
    const size_t n8 = n / 8;
    const int blocks = (int)std::min<size_t>(ceil_div(n8, 256), (size_t)c->num_sms * 8);
    add_bf16_residual_kernel<<<blocks, 256, 0, c->stream>>>(a, y, n8, out);
    SCMOE_LAUNCH_CHECK(c);
}

// ---------------------------------------------------------------------------
// Expert-parallel helpers.
// ---------------------------------------------------------------------------
// Destination "bin" of every slot: owning rank of an FFN expert, `world` for
// a zero expert (never sent).
__global__ void ep_bins_kernel(const uint32_t* __restrict__ idx, size_t n, uint32_t n_ffn,
                               uint32_t per_rank, uint32_t world, uint32_t* __restrict__ bins) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const uint32_t e = idx[i];
        bins[i] = e < n_ffn ? e / per_rank : world;
    }
}

void launch_ep_bins(scmoe_ctx* c, const uint32_t* idx, size_t n, size_t n_ffn, size_t per_rank,
                    int world, uint32_t* bins) {
    if (n == 0) return;
    ep_bins_kernel<<<ceil_div(n, 256), 256, 0, c->stream>>>(idx, n, (uint32_t)n_ffn,
                                                           (uint32_t)per_rank, (uint32_t)world, bins);
    SCMOE_LAUNCH_CHECK(c);
}

// send_expert[slot_pos[i]] = idx[i] for every sent slot.
__global__ void ep_send_expert_kernel(const uint32_t* __restrict__ idx,
                                      const int* __restrict__ slot_pos, size_t n,
                                      int* __restrict__ send_expert) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && slot_pos[i] >= 0) send_expert[slot_pos[i]] = (int)idx[i];
}

void launch_ep_send_expert(scmoe_ctx* c, const uint32_t* idx, const int* slot_pos, size_t n,
                           int* send_expert) {
    if (n == 0) return;
    ep_send_expert_kernel<<<ceil_div(n, 256), 256, 0, c->stream>>>(idx, slot_pos, n, send_expert);
    SCMOE_LAUNCH_CHECK(c);
}

// moe_block's permutation in the reference's own terms (blocks.hpp:349-359):
// slot_row[t*K+s] = position of token t in expert e's ascending token list
// (slot_pos minus the expert's base row), -1 for a zero expert.
__global__ void slot_rows_kernel(const uint32_t* __restrict__ idx, const int* __restrict__ slot_pos,
                                 const int* __restrict__ expert_base, size_t n, int n_ffn,
                                 int* __restrict__ slot_row) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t e = idx[i];
    slot_row[i] = e < (uint32_t)n_ffn ? slot_pos[i] - expert_base[e] : -1;
}

void launch_slot_rows(scmoe_ctx* c, const uint32_t* idx, const int* slot_pos,
                      const int* expert_base, size_t n, int n_ffn, int* slot_row) {
    if (n == 0) return;
    slot_rows_kernel<<<ceil_div(n, 256), 256, 0, c->stream>>>(idx, slot_pos, expert_base, n, n_ffn,
                                                              slot_row);
    SCMOE_LAUNCH_CHECK(c);
}

// Received rows' global expert ids -> this rank's local ids (range-checked).
__global__ void ep_localize_kernel(const int* __restrict__ row_expert, size_t n, int offset,
                                   int n_local, uint32_t* __restrict__ local,
                                   int* __restrict__ dev_status, const int* __restrict__ n_dev) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n_dev) n = min(n, (size_t)max(*n_dev, 0));
    if (i >= n) return;
    const int e = row_expert[i] - offset;
    if (e < 0 || e >= n_local) {
        atomicExch(dev_status, DEV_ERR_INDEX_RANGE);
        local[i] = 0;
    } else {
        local[i] = (uint32_t)e;
    }
}

void launch_ep_localize(scmoe_ctx* c, const int* row_expert, size_t n, int offset, int n_local,
                        uint32_t* local, const int* n_dev) {
    if (n == 0) return;
    ep_localize_kernel<<<ceil_div(n, 256), 256, 0, c->stream>>>(row_expert, n, offset, n_local,
                                                               local, c->dev_status, n_dev);
    SCMOE_LAUNCH_CHECK(c);
}

// dst[i] = src[rows[i]], bf16 rows of width d (one warp per row, 16-byte vectors).
__global__ void gather_rows_bf16_kernel(const __nv_bfloat16* __restrict__ src, int d,
                                        const int* __restrict__ rows, size_t n_rows,
                                        __nv_bfloat16* __restrict__ dst) {
    const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
    const int vec = d / 8;
    for (size_t r = warp; r < n_rows; r += nwarps) {
        const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)rows[r] * d);
        uint4* o = reinterpret_cast<uint4*>(dst + r * d);
        for (int v = lane; v < vec; v += 32) o[v] = s[v];
    }
}

// Expert-parallel dispatch straight into the destination ranks' receive
// buffers (symmetric memory mapped over NVLink): one warp per send row, 16-byte
// stores (512 B per warp instruction); lane 0 also stores the row's expert id.
__global__ void ep_put_rows_kernel(const __nv_bfloat16* __restrict__ src, int d,
                                   const int* __restrict__ send_token,
                                   const int* __restrict__ send_expert, int n_send,
                                   const int* __restrict__ send_start,
                                   const int64_t* __restrict__ dst_offset,
                                   const uint64_t* __restrict__ peer_rows,
                                   const uint64_t* __restrict__ peer_expert, int G,
                                   int64_t cap_dst, int* __restrict__ dev_status) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int vec = d / 8;
    n_send = min(n_send, send_start[G]);  // the plan's count (device side)
    for (int j = warp; j < n_send; j += nwarps) {
        int dst = 0;
        while (dst + 1 < G && send_start[dst + 1] <= j) ++dst;
        const int64_t pos = dst_offset[dst] + (j - send_start[dst]);
        if (pos >= cap_dst) {  // receiver capacity exceeded: latched, row dropped
            if (lane == 0) atomicExch(dev_status, DEV_ERR_CAPACITY);
            continue;
        }
        const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)send_token[j] * d);
        uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(peer_rows[dst]) +
                                            (size_t)pos * d);
        // four loads in flight per lane before the (NVLink) stores
        int v = lane;
        for (; v + 96 < vec; v += 128) {
            const uint4 q0 = s[v], q1 = s[v + 32], q2 = s[v + 64], q3 = s[v + 96];
            o[v] = q0;
            o[v + 32] = q1;
            o[v + 64] = q2;
            o[v + 96] = q3;
        }
        for (; v < vec; v += 32) o[v] = s[v];
        if (lane == 0) reinterpret_cast<int*>(peer_expert[dst])[pos] = send_expert[j];
    }
}
// Same dispatch with the copy engine: per warp, lane 0 moves whole rows by
// bulk async copies -- local row -> shared memory (mbarrier completion) ->
// peer row over NVLink -- with two row buffers per warp, so the transfers
// are single large transactions instead of 16-byte stores.
constexpr int kPutWarps = 4;
__global__ void __launch_bounds__(kPutWarps * 32) ep_put_rows_bulk_kernel(
    const __nv_bfloat16* __restrict__ src, int d, const int* __restrict__ send_token,
    const int* __restrict__ send_expert, int n_send, const int* __restrict__ send_start,
    const int64_t* __restrict__ dst_offset, const uint64_t* __restrict__ peer_rows,
    const uint64_t* __restrict__ peer_expert, int G, int64_t cap_dst, int* __restrict__ dev_status) {
    extern __shared__ __align__(128) unsigned char put_smem[];
    __shared__ uint64_t bars[kPutWarps][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t row_bytes = (uint32_t)d * 2;
    unsigned char* buf = put_smem + (size_t)warp * 2 * row_bytes;
    if (lane == 0) {
        mbar_init(&bars[warp][0], 1);
        mbar_init(&bars[warp][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (lane != 0) return;
    const int gw = blockIdx.x * kPutWarps + warp, nw = gridDim.x * kPutWarps;
    uint32_t phase[2] = {0, 0};
    int it = 0;
    n_send = min(n_send, send_start[G]);
    for (int j = gw; j < n_send; j += nw, ++it) {
        const int b = it & 1;
        unsigned char* sb = buf + b * row_bytes;
        // the bulk store that last read this buffer (two rows ago) has read it
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        int dst = 0;
        while (dst + 1 < G && send_start[dst + 1] <= j) ++dst;
        const int64_t pos = dst_offset[dst] + (j - send_start[dst]);
        if (pos >= cap_dst) {
            atomicExch(dev_status, DEV_ERR_CAPACITY);
            continue;
        }
        mbar_expect_tx(&bars[warp][b], row_bytes);
        asm volatile(
            "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(smem_u32(sb)),
            "l"(reinterpret_cast<uint64_t>(src + (size_t)send_token[j] * d)), "r"(row_bytes),
            "r"(smem_u32(&bars[warp][b]))
            : "memory");
        mbar_wait(&bars[warp][b], phase[b]);
        phase[b] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<uint64_t>(reinterpret_cast<__nv_bfloat16*>(peer_rows[dst]) +
                                                    (size_t)pos * d)),
                     "r"(smem_u32(sb)), "r"(row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        reinterpret_cast<int*>(peer_expert[dst])[pos] = send_expert[j];
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

void launch_ep_put_rows(scmoe_ctx* c, const __nv_bfloat16* src, size_t d, const int* send_token,
                        const int* send_expert, size_t n_send, const int* send_start,
                        const int64_t* dst_offset, const uint64_t* peer_rows,
                        const uint64_t* peer_expert, int G, int64_t cap_dst) {
    if (n_send == 0) return;
    SCMOE_CHECK_ARG(d % 8 == 0, SCMOE_ERR_DIMENSION, "ep_put_rows: d must be a multiple of 8");
    // the warp-store kernel is the default: same NVLink rate as the bulk-copy
    // one (1.11 ms for 604 MB at EP x4) and no shared memory, so it can share
    // an SM with the expert GEMM of the previous batch (SCMOE_PUT_BULK=1)
    static const bool bulk = getenv("SCMOE_PUT_BULK") != nullptr;
    const size_t smem = (size_t)kPutWarps * 2 * d * 2;
    if (bulk && smem <= 200 * 1024) {
        ensure_max_dynamic_smem(reinterpret_cast<const void*>(ep_put_rows_bulk_kernel), (int)smem,
                                c->device);
        ep_put_rows_bulk_kernel<<<c->num_sms * 2, kPutWarps * 32, smem, c->stream>>>(
            src, (int)d, send_token, send_expert, (int)n_send, send_start, dst_offset, peer_rows,
            peer_expert, G, cap_dst, c->dev_status);
    } else {
        const int blocks = c->num_sms * 4;
        ep_put_rows_kernel<<<blocks, 256, 0, c->stream>>>(src, (int)d, send_token, send_expert,
                                                          (int)n_send, send_start, dst_offset,
                                                          peer_rows, peer_expert, G, cap_dst,
                                                          c->dev_status);
    }
    SCMOE_LAUNCH_CHECK(c);
}

void launch_gather_rows_bf16(scmoe_ctx* c, const __nv_bfloat16* src, size_t d, const int* rows,
                             size_t n_rows, __nv_bfloat16* dst) {
    if (n_rows == 0) return;
    SCMOE_CHECK_ARG(d % 8 == 0, SCMOE_ERR_DIMENSION, "gather: d must be a multiple of 8");
    const int blocks = (int)std::min<size_t>(ceil_div(n_rows, 8), (size_t)c->num_sms * 8);
    gather_rows_bf16_kernel<<<blocks, 256, 0, c->stream>>>(src, (int)d, rows, n_rows, dst);
    SCMOE_LAUNCH_CHECK(c);
}

}  // namespace scmoe
