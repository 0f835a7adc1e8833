// mla_tc.cu -- multi-head latent attention forward (blocks.hpp:73-102) on the
// tensor cores: bf16 operands, fp32 accumulation, the same tcgen05 grouped
// GEMM as the experts for every contraction.  Tolerance path (rel-L2 <= 2e-2
// vs the exact oracle, tests/test_gpu_mla.py); the exact fp32 path (mla.cu)
// stays the bitwise reference implementation.
//
//   P1  = [cq | ckv | kr] = bf16(h) W_h        (one GEMM, W_h = [w_dq|w_dkv|w_kr])
//         cq *= alpha_q, ckv *= alpha_kv, rope(kr)            (bf16 epilogue kernel)
//   Q   = [qc | qr] = cq W_q, rope(qr)         (X = P1's cq columns by TMA stride)
//   KV  = [kc | vv] = ckv W_kv
//   per (sequence b, head h), as grouped-GEMM "experts" (one per (b, h)):
//     S   = [qc|qr] [kc|kr]^T                  (keys on the M side, K-blocked)
//     P   = softmax(scale * S) causal          (rows written straight into the
//                                               K-blocked layout PV reads as W)
//     O^T = V^T-rows x P                       (O^T[c][q] = sum_k P[q][k] V[k][c])
//   out = fp32(merged(O) W_o)
// Every GEMM is D[rows][m] = sum_k W[m][k] X[rows][k] with W in the blocked
// K-major layout (internal.cuh wblk_index), M padded to a multiple of 256 and
// K to a multiple of 64 with zeros; sequence lengths are padded to 256 keys.
#include <cmath>
#include <cstdlib>

#include "internal.cuh"
#include "tcgen05_util.cuh"

namespace scmoe {

namespace {

size_t pad_to(size_t x, size_t m) { return (x + m - 1) / m * m; }

// Qrows[(bh*L + q)][t] = [qc_h | rope(qr_h) | 0] of token b*L + q;
// Kblk[bh] (blocked, Lp x Dk) row key = [kc_h | rope(kr) | 0] of token b*L + key
// (0 past L).  The rotary halves are rotated here (pair (2p, 2p+1) by the
// angle of position q and frequency p, rope table [pos][dhr/2] of (cos, sin)),
// so the projections need no separate rope pass.  Index math in 32 bits (the
// host checks BH * Lp * Dk < 2^31).
__device__ __forceinline__ void rope_pair(float& a, float& b, float2 cs) {
    const float x = a * cs.x - b * cs.y, y = a * cs.y + b * cs.x;
    a = x;
    b = y;
}
__global__ void mla_pack_qk_kernel(const __nv_bfloat16* __restrict__ Q, size_t ldq,
                                   const __nv_bfloat16* __restrict__ KV, size_t ldkv,
                                   const __nv_bfloat16* __restrict__ P1, size_t ldp1, int kr_col,
                                   int BH, int H, int L, int Lp, int dhc, int dhr, int Dk,
                                   const float2* __restrict__ rope,
                                   __nv_bfloat16* __restrict__ Qrows,
                                   __nv_bfloat16* __restrict__ Kblk) {
    const int n = BH * Lp * Dk;
    const __nv_bfloat16 zero = __float2bfloat16_rn(0.f);
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n; it += gridDim.x * blockDim.x) {
        const int t = it % Dk;
        const int row = it / Dk;
        const int j = row % Lp;
        const int bh = row / Lp, b = bh / H, h = bh % H;
        const size_t tok = (size_t)b * L + j;
        __nv_bfloat16 kv = zero, qv = zero;
        if (j < L) {
            if (t < dhc) {
                kv = KV[tok * ldkv + (size_t)h * dhc + t];
                qv = Q[tok * ldq + (size_t)h * dhc + t];
            } else if (t < dhc + dhr) {
                const int e = t - dhc, e0 = e & ~1;
                const float2 cs = rope[(size_t)j * (dhr / 2) + e0 / 2];
                const __nv_bfloat16* kp = P1 + tok * ldp1 + kr_col + e0;
                const __nv_bfloat16* qp = Q + tok * ldq + (size_t)H * dhc + (size_t)h * dhr + e0;
                float ka = __bfloat162float(kp[0]), kb = __bfloat162float(kp[1]);
                float qa = __bfloat162float(qp[0]), qb = __bfloat162float(qp[1]);
                rope_pair(ka, kb, cs);
                rope_pair(qa, qb, cs);
                kv = __float2bfloat16_rn(e & 1 ? kb : ka);
                qv = __float2bfloat16_rn(e & 1 ? qb : qa);
            }
            Qrows[((size_t)bh * L + j) * Dk + t] = qv;
        }
        Kblk[(size_t)bh * Lp * Dk + wblk_index(j, t, Dk)] = kv;
    }
}

// Same, 8 consecutive t (16 bytes) per thread: needs dhc % 8 == dhr % 8 == 0.
__global__ void mla_pack_qk8_kernel(const __nv_bfloat16* __restrict__ Q, size_t ldq,
                                    const __nv_bfloat16* __restrict__ KV, size_t ldkv,
                                    const __nv_bfloat16* __restrict__ P1, size_t ldp1, int kr_col,
                                    int BH, int H, int L, int Lp, int dhc, int dhr, int Dk,
                                    const float2* __restrict__ rope,
                                    __nv_bfloat16* __restrict__ Qrows,
                                    __nv_bfloat16* __restrict__ Kblk) {
    const int Dk8 = Dk / 8;
    const int n = BH * Lp * Dk8;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n; it += gridDim.x * blockDim.x) {
        const int t = (it % Dk8) * 8;
        const int row = it / Dk8;
        const int j = row % Lp;
        const int bh = row / Lp, b = bh / H, h = bh % H;
        const size_t tok = (size_t)b * L + j;
        uint4 kv = make_uint4(0, 0, 0, 0), qv = make_uint4(0, 0, 0, 0);
        if (j < L) {
            if (t < dhc) {
                kv = *reinterpret_cast<const uint4*>(KV + tok * ldkv + (size_t)h * dhc + t);
                qv = *reinterpret_cast<const uint4*>(Q + tok * ldq + (size_t)h * dhc + t);
            } else if (t < dhc + dhr) {
                kv = *reinterpret_cast<const uint4*>(P1 + tok * ldp1 + kr_col + (t - dhc));
                qv = *reinterpret_cast<const uint4*>(Q + tok * ldq + (size_t)H * dhc +
                                                     (size_t)h * dhr + (t - dhc));
                const float2* cs = rope + (size_t)j * (dhr / 2) + (t - dhc) / 2;
                __nv_bfloat162* k2 = reinterpret_cast<__nv_bfloat162*>(&kv);
                __nv_bfloat162* q2 = reinterpret_cast<__nv_bfloat162*>(&qv);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 c = cs[u];
                    float ka = __low2float(k2[u]), kb = __high2float(k2[u]);
                    float qa = __low2float(q2[u]), qb = __high2float(q2[u]);
                    rope_pair(ka, kb, c);
                    rope_pair(qa, qb, c);
                    k2[u] = __floats2bfloat162_rn(ka, kb);
                    q2[u] = __floats2bfloat162_rn(qa, qb);
                }
            }
            *reinterpret_cast<uint4*>(Qrows + ((size_t)bh * L + j) * Dk + t) = qv;
        }
        *reinterpret_cast<uint4*>(Kblk + (size_t)bh * Lp * Dk + wblk_index(j, t, Dk)) = kv;
    }
}

// Vt[(bh*dhc + c)][key] = vv_h[c] of token b*L + key (0 past L): 32x32 tile transpose.
__global__ void mla_pack_vt_kernel(const __nv_bfloat16* __restrict__ KV, size_t ldkv, int H,
                                   int L, int Lp, int dhc, __nv_bfloat16* __restrict__ Vt) {
    __shared__ float tile[32][33];
    const int bh = blockIdx.z, b = bh / H, h = bh % H;
    const int k0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int key = k0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] =
            key < L && c < dhc
                ? __bfloat162float(KV[((size_t)b * L + key) * ldkv + (size_t)H * dhc +
                                      (size_t)h * dhc + c])
                : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, key = k0 + threadIdx.x;
        if (c < dhc && key < Lp)
            Vt[((size_t)bh * dhc + c) * Lp + key] = __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
}

// Causal softmax of scale * S (graph.hpp:396-434 semantics: query i sees keys
// j <= i), one warp per (bh, query row), 8 keys (16 bytes) per lane access;
// the probabilities are written in the blocked K-major layout the PV GEMM
// reads as its W operand.  Keys past the end of q's 256-row block are never
// read (the PV GEMM's causal K bound), so only the diagonal block's tail gets
// zeros; padding rows q >= L get zeros (their outputs are discarded).
__global__ void mla_softmax_bf16_kernel(const __nv_bfloat16* __restrict__ S, int BH, int L, int Lp,
                                        float scale, __nv_bfloat16* __restrict__ Pblk) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= BH * Lp) return;
    const int bh = warp / Lp, q = warp % Lp;
    __nv_bfloat16* P = Pblk + (size_t)bh * Lp * Lp;
    const int jend = min(Lp, ((q >> 8) + 1) << 8);  // multiple of 256
    if (q >= L) {
        for (int j = lane * 8; j < jend; j += 256)
            *reinterpret_cast<uint4*>(P + wblk_index(q, j, Lp)) = make_uint4(0, 0, 0, 0);
        return;
    }
    const __nv_bfloat16* s = S + ((size_t)bh * L + q) * Lp;
    float mx = -INFINITY, sum = 0.f;
    for (int j0 = lane * 8; j0 <= q; j0 += 256) {  // online max / sum per lane
        const uint4 raw = *reinterpret_cast<const uint4*>(s + j0);
        const __nv_bfloat16* v8 = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (j0 + u > q) break;
            const float v = __bfloat162float(v8[u]) * scale;
            if (v > mx) {
                sum = sum * __expf(mx - v) + 1.f;
                mx = v;
            } else {
                sum += __expf(v - mx);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
        const float mn = fmaxf(mx, m2);
        sum = (mx == -INFINITY ? 0.f : sum * __expf(mx - mn)) +
              (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
        mx = mn;
    }
    const float inv = 1.f / sum;
    for (int j0 = lane * 8; j0 < jend; j0 += 256) {
        uint4 outv = make_uint4(0, 0, 0, 0);
        if (j0 <= q) {
            const uint4 raw = *reinterpret_cast<const uint4*>(s + j0);
            const __nv_bfloat16* v8 = reinterpret_cast<const __nv_bfloat16*>(&raw);
            __nv_bfloat16* o8 = reinterpret_cast<__nv_bfloat16*>(&outv);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                o8[u] = j0 + u <= q
                            ? __float2bfloat16_rn(__expf(__bfloat162float(v8[u]) * scale - mx) * inv)
                            : __float2bfloat16_rn(0.f);
        }
        *reinterpret_cast<uint4*>(P + wblk_index(q, j0, Lp)) = outv;
    }
}


// ---------------------------------------------------------------------------
// Fused causal attention (default): one CTA per (sequence b, head h) x 128
// queries, one pass over the key tiles j <= diagonal on the tensor cores:
// S_j = Q K_j^T into TMEM (double buffered, S_{j+1} computed under the
// softmax of tile j), P = exp2(S scale - m_ref) written as bf16 into a
// 128B-swizzled K-major smem tile, O += P V_j accumulated in TMEM.  The
// reference max m_ref moves only when a tile's row max exceeds it by more
// than 8 (exp2 domain), and only then are O (in TMEM, between two P.V MMAs)
// and l rescaled -- after the first tiles the max has settled.  O / l goes
// straight to the merged rows; S and P never touch HBM.  Warp roles: 0 Q + K
// TMA producer, 1 MMA issuer (one lane), 2 V^T producer, 3-10 softmax (two
// warps per TMEM lane quadrant, 64 keys of every tile each, one query row per
// thread).
// ---------------------------------------------------------------------------
// 2^x on the SFU alone (no range fix-up: arguments are <= 0 or -inf here)
__device__ __forceinline__ float ex2_fast(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void st_shared_v4(unsigned char* p, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}

constexpr int FA_BQ = 128, FA_BKEY = 128, FA_KBMAX = 3, FA_DVMAX = 128;
constexpr int FA_BLK = 128 * 64 * 2;  // one [128 rows][64 cols] bf16 SW128 block (16 KB)
constexpr int FA_SWARPS = 8;          // softmax warps: 2 per TMEM lane quadrant (64 keys each)
constexpr int FA_THREADS = (3 + FA_SWARPS) * 32;
constexpr size_t FA_SMEM = 1024 + FA_KBMAX * FA_BLK /*Q*/ + 2 * FA_KBMAX * FA_BLK /*K ring*/ +
                           2 * FA_DVMAX * 128 /*V^T: 2 key halves*/ + 2 * FA_BLK /*P*/ +
                           6 * FA_BQ * 4 /*row stats*/ + 256;

struct FaArgs {
    int BH, H, L, Lp, nqt, KB, dv;
    float scale_log2;
    __nv_bfloat16* merged;
    size_t ldm;
};

// warps: 0 Q + K producer, 1 MMA issuer, 2 V producer, 3..10 softmax (warp w
// owns TMEM lane quadrant w % 4 and key half (w - 3) / 4 of every tile)
__global__ void __launch_bounds__(FA_THREADS, 1)
    mla_flash_kernel(const __grid_constant__ CUtensorMap map_q,
                     const __grid_constant__ CUtensorMap map_k,
                     const __grid_constant__ CUtensorMap map_v, const FaArgs a) {
    extern __shared__ __align__(1024) unsigned char fa_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(fa_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* Qs = sm;
    unsigned char* Ks = Qs + FA_KBMAX * FA_BLK;             // [2][KB blocks]
    unsigned char* Vs = Ks + 2 * FA_KBMAX * FA_BLK;         // [2 halves][dv rows][128 B]
    unsigned char* Ps = Vs + 2 * FA_DVMAX * 128;            // [2 blocks][128 rows][128 B]
    float* stat_m = reinterpret_cast<float*>(Ps + 2 * FA_BLK);  // [2 halves][128 rows]
    float* stat_l = stat_m + 4 * FA_BQ;  // stat_m: [2 halves][2 tile parities][128 rows]
    uint64_t* bars = reinterpret_cast<uint64_t*>(stat_l + 2 * FA_BQ);
    uint64_t *q_full = bars, *k_full = bars + 1, *k_empty = bars + 3, *v_full = bars + 5,
             *v_empty = bars + 6, *s_full = bars + 7, *s_empty = bars + 9, *p_full = bars + 11,
             *p_empty = bars + 12, *o_full = bars + 13;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    // CTAs of one (b, h) are consecutive, so the ~148 resident ones span only a
    // few heads and their K / V^T tiles stay in L2 (head-strided order thrashed
    // it: 7 GB of DRAM reads per MLA); heaviest query tile first within a head
    const int t = a.nqt - 1 - (int)(blockIdx.x % a.nqt);
    const int bh = (int)(blockIdx.x / a.nqt);
    const int q0 = t * FA_BQ;
    const int nj = t + 1;
    const int KB = a.KB, dv = a.dv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], FA_SWARPS);
        }
        mbar_init(v_full, 1);
        mbar_init(v_empty, 1);
        mbar_init(p_full, FA_SWARPS);
        mbar_init(p_empty, 1);
        mbar_init(o_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;  // S0 cols [0,128), S1 [128,256), O [256, 256 + dv)

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            mbar_expect_tx(q_full, (uint32_t)(KB * FA_BLK));
            for (int kb = 0; kb < KB; ++kb)
                tma_load_2d(&map_q, q_full, Qs + kb * FA_BLK, kb * 64, bh * a.L + q0, pol);
            const int krow0 = bh * (a.Lp * KB);  // K blocked layout: rows of 64 elements
            int ks = 0;
            uint32_t kph = 0;
            for (int j = 0; j < nj; ++j) {
                mbar_wait(&k_empty[ks], kph ^ 1);
                mbar_expect_tx(&k_full[ks], (uint32_t)(KB * FA_BLK));
                for (int kb = 0; kb < KB; ++kb)
                    tma_load_2d(&map_k, &k_full[ks], Ks + (ks * FA_KBMAX + kb) * FA_BLK, 0,
                                krow0 + (j * KB + kb) * 128, pol);
                if (++ks == 2) {
                    ks = 0;
                    kph ^= 1;
                }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {  // V^T tiles of the second pass, their own ring
            const uint64_t pol = policy_evict_last();
            uint32_t vph = 0;
            for (int j = 0; j < nj; ++j) {
                mbar_wait(v_empty, vph ^ 1);
                mbar_expect_tx(v_full, (uint32_t)(dv * 256));
                tma_load_2d(&map_v, v_full, Vs, j * FA_BKEY, bh * dv, pol);
                tma_load_2d(&map_v, v_full, Vs + dv * 128, j * FA_BKEY + 64, bh * dv, pol);
                vph ^= 1;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id_s = tc::idesc_bf16(128, FA_BKEY), id_o = tc::idesc_bf16(128, dv);
            int ks = 0, sb = 0;
            uint32_t kph = 0, sph = 0, pph = 0, vph = 0;
            auto issue_s = [&]() {
                mbar_wait(&k_full[ks], kph);
                mbar_wait(&s_empty[sb], sph ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = 0; kb < KB; ++kb)
                    for (int k = 0; k < 4; ++k)
                        tc::mma(tmem + sb * FA_BKEY,
                                tc::desc_sw128(smem_u32(Qs + kb * FA_BLK) + k * 32),
                                tc::desc_sw128(smem_u32(Ks + (ks * FA_KBMAX + kb) * FA_BLK) + k * 32),
                                id_s, (kb | k) != 0);
                tc::commit(&k_empty[ks]);
                tc::commit(&s_full[sb]);
                if (++ks == 2) {
                    ks = 0;
                    kph ^= 1;
                }
                if (++sb == 2) {
                    sb = 0;
                    sph ^= 1;
                }
            };
            mbar_wait(q_full, 0);
            issue_s();  // S_0 ahead
            for (int j = 0; j < nj; ++j) {
                if (j + 1 < nj) issue_s();  // S_{j+1} under the softmax of tile j
                mbar_wait(p_full, pph);
                mbar_wait(v_full, vph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int b = 0; b < 2; ++b)
                    for (int k = 0; k < 4; ++k)
                        tc::mma(tmem + 2 * FA_BKEY, tc::desc_sw128(smem_u32(Ps + b * FA_BLK) + k * 32),
                                tc::desc_sw128(smem_u32(Vs + b * dv * 128) + k * 32), id_o,
                                (j | b | k) != 0);
                tc::commit(p_empty);
                tc::commit(v_empty);
                pph ^= 1;
                vph ^= 1;
            }
            tc::commit(o_full);
        }
    } else {
        const int sw = warp - 3;            // 0..7
        const int quad = warp & 3;           // TMEM lanes this warp may access
        const int half = sw >> 2;            // key half [half*64, half*64 + 64) of each tile
        const int r = quad * 32 + lane;      // query row = TMEM lane
        const int q = q0 + r;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        // m_ref: the row's reference max (exp2 domain) the probabilities of
        // every tile so far are relative to; both key halves hold the same
        // value.  It moves only when a tile's max exceeds it by > 8 (P <= 256:
        // exact enough in bf16 / fp32), and then O and l are rescaled.
        float m_ref = -INFINITY, l = 0.f;
        int sb = 0;
        uint32_t sph = 0, pph = 0;
        uint32_t v[2][32];
        const int pair_bar = 2 + quad;  // named barrier of the two warps sharing these rows
        for (int j = 0; j < nj; ++j) {
            mbar_wait(&s_full[sb], sph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            tc::ld32(tmem + lane_off + sb * FA_BKEY + (half * 2) * 32, v[0]);
            tc::ld32(tmem + lane_off + sb * FA_BKEY + (half * 2 + 1) * 32, v[1]);
            tc::ld_wait();
            // S buffer free as soon as it is in registers
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            if (++sb == 2) {
                sb = 0;
                sph ^= 1;
            }
            const int key0 = j * FA_BKEY + half * 64;
            const bool diag = key0 + 63 > q;  // only the diagonal tile is masked
            if (diag) {  // keys past the query: -inf (p = 0)
#pragma unroll
                for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (key0 + cc * 32 + i > q) v[cc][i] = __float_as_uint(-INFINITY);
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(v[cc][i]));
            float cm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
            // the row max over both halves (scale_log2 > 0 commutes with max)
            const uint32_t xm = smem_u32(stat_m + (j & 1) * FA_BQ);  // [half][parity][row]
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(xm + (uint32_t)(half * 2 * FA_BQ + r) * 4),
                         "f"(cm)
                         : "memory");
            asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
            float cm2;
            asm volatile("ld.shared.f32 %0, [%1];"
                         : "=f"(cm2)
                         : "r"(xm + (uint32_t)((half ^ 1) * 2 * FA_BQ + r) * 4)
                         : "memory");
            cm = fmaxf(cm, cm2) * a.scale_log2;
            float alpha = 1.f;
            const bool move = cm > m_ref + 8.f;  // also true on the first tile (-inf)
            if (move) {
                alpha = ex2_fast(m_ref - cm);  // 0 on the first tile
                l *= alpha;
                m_ref = cm;
            }
            const float nm = -m_ref;
            uint32_t pw[2][16];
            float add[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int i2 = 0; i2 < 16; ++i2) {
                    const float p0 = ex2_fast(fmaf(__uint_as_float(v[cc][2 * i2]), a.scale_log2, nm));
                    const float p1 =
                        ex2_fast(fmaf(__uint_as_float(v[cc][2 * i2 + 1]), a.scale_log2, nm));
                    add[(i2 & 1) * 2] += p0;
                    add[(i2 & 1) * 2 + 1] += p1;
                    const __nv_bfloat162 pk = __floats2bfloat162_rn(p0, p1);
                    pw[cc][i2] = *reinterpret_cast<const uint32_t*>(&pk);
                }
            l += (add[0] + add[1]) + (add[2] + add[3]);
            // P.V of tile j-1 has completed once the P buffer is free; O is then
            // quiescent and may be rescaled in place (rare: the max settles)
            mbar_wait(p_empty, pph ^ 1);
            if (move && j > 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int c = half; c < dv / 32; c += 2) {
                    uint32_t o[32];
                    tc::ld32(tmem + lane_off + 2 * FA_BKEY + c * 32, o);
                    tc::ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tc::st32(tmem + lane_off + 2 * FA_BKEY + c * 32, o);
                }
                tc::st_wait();
            }
            unsigned char* rowp = Ps + half * FA_BLK + r * 128;  // block `half`
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int chunk = cc * 4 + u;
                    st_shared_v4(rowp + ((chunk ^ (r & 7)) << 4), pw[cc][4 * u], pw[cc][4 * u + 1],
                                 pw[cc][4 * u + 2], pw[cc][4 * u + 3]);
                }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
            pph ^= 1;
        }
        // the row normaliser: both halves' partial sums share m_ref
        stat_l[half * FA_BQ + r] = l;
        asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
        l += stat_l[(half ^ 1) * FA_BQ + r];
        mbar_wait(o_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float inv = 1.f / l;
        const int b = bh / a.H, h = bh % a.H;
        __nv_bfloat16* dst = a.merged + ((size_t)b * a.L + q) * a.ldm + (size_t)h * dv;
        for (int c = half; c < dv / 32; c += 2) {
            tc::ld32(tmem + lane_off + 2 * FA_BKEY + c * 32, v[0]);
            tc::ld_wait();
            if (q < a.L) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t w[4];
#pragma unroll
                    for (int h2 = 0; h2 < 4; ++h2) {
                        const int i0 = u * 8 + h2 * 2;
                        const __nv_bfloat162 pk = __floats2bfloat162_rn(
                            __uint_as_float(v[0][i0]) * inv, __uint_as_float(v[0][i0 + 1]) * inv);
                        w[h2] = *reinterpret_cast<const uint32_t*>(&pk);
                    }
                    *reinterpret_cast<uint4*>(dst + c * 32 + u * 8) = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// Fused causal attention, two query tiles per CTA (default): tiles tA = 2u and
// tB = 2u + 1 of one (sequence, head) share every 128-key K and V^T tile they
// both need (loaded once), and their softmax warp groups ping-pong with the
// tensor core: while group A turns S_A(j) into probabilities, the MMA lane
// runs S_B(j); while group B works, P_A(j) V_j and S_A(j+1).  Each softmax
// thread owns one full query row of its tile (no cross-warp exchange); P is
// written back as bf16 pairs into the S columns of TMEM and consumed from
// there by the P.V MMA (A operand in tensor memory), so P touches neither
// shared memory nor HBM.  TMEM: S_A [0,128), S_B [128,256), O_A
// [256,256+dv), O_B [384,384+dv).  The tensor pipe executes one thread's MMAs
// in order and every commit tracks all earlier MMAs: when S_X(j) has landed,
// P_X(j-1) V_{j-1} has too, so O_X may be rescaled in place (lazy, only when
// the row max moves by > 8 in the exp2 domain) without a barrier.  Shared
// memory: Q_A, Q_B (96 KB), 2 K stages (96 KB), one V^T tile (32 KB).
// Warps: 0 Q + K producer, 1 MMA lane, 2 V^T producer, 3-6 softmax of tile A,
// 7-10 softmax of tile B.  Measured (clock64 timeline of one CTA, LongCat
// widths): ~4.6 k cycles per key tile for both query tiles against 2.56 k of
// tensor work at the dense-MMA floor; the Q.K^T MMAs (both operands in shared
// memory, 8 KB per 64-cycle MMA) run ~40 % above the floor, and the softmax
// of one tile (128 exponentials per thread) takes ~1.6 k cycles.  Tried and
// slower: 64-key tiles with double-buffered S and V (1.10 vs 0.81 ms: twice
// the MMA issues and handshakes); a quarter of the exponentials on the FMA
// pipe (polynomial 2^x; no gain, the SFU is not the limiter).
// ---------------------------------------------------------------------------
constexpr int F2_THREADS = 11 * 32;
constexpr size_t F2_SMEM = 1024 + 2 * FA_KBMAX * FA_BLK /*Q_A, Q_B*/ +
                           2 * FA_KBMAX * FA_BLK /*K ring*/ + 2 * FA_DVMAX * 128 /*V^T*/ + 256;

__global__ void __launch_bounds__(F2_THREADS, 1)
    mla_flash2_kernel(const __grid_constant__ CUtensorMap map_q,
                      const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v, const FaArgs a) {
    extern __shared__ __align__(1024) unsigned char f2_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(f2_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* Qs = sm;                          // [tile X][KB blocks]
    unsigned char* Ks = Qs + 2 * FA_KBMAX * FA_BLK;  // [stage][KB blocks]
    unsigned char* Vs = Ks + 2 * FA_KBMAX * FA_BLK;  // [key half][dv rows][128 B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(Vs + 2 * FA_DVMAX * 128);
    uint64_t *q_full = bars, *k_full = bars + 1, *k_empty = bars + 3, *v_full = bars + 5,
             *v_empty = bars + 6, *s_full = bars + 7, *p_full = bars + 9, *o_done = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

    // heaviest pair of query tiles first within a head; the CTAs of one head
    // are consecutive so its K / V^T tiles stay in L2
    const int npairs = (a.nqt + 1) >> 1;
    const int u = npairs - 1 - (int)(blockIdx.x % npairs);
    const int bh = (int)(blockIdx.x / npairs);
    const int tA = 2 * u, tB = 2 * u + 1;
    const bool hasB = tB < a.nqt;
    const int nj = hasB ? tB + 1 : tA + 1;  // key tiles the pair needs
    const int KB = a.KB, dv = a.dv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&o_done[i], 1);
        }
        mbar_init(v_full, 1);
        mbar_init(v_empty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            const int nq = hasB ? 2 : 1;
            mbar_expect_tx(q_full, (uint32_t)(nq * KB * FA_BLK));
            for (int x = 0; x < nq; ++x)
                for (int kb = 0; kb < KB; ++kb)
                    tma_load_2d(&map_q, q_full, Qs + (x * FA_KBMAX + kb) * FA_BLK, kb * 64,
                                bh * a.L + (tA + x) * FA_BQ, pol);
            const int krow0 = bh * (a.Lp * KB);  // K blocked layout: rows of 64 elements
            int ks = 0;
            uint32_t kph = 0;
            for (int j = 0; j < nj; ++j) {
                mbar_wait(&k_empty[ks], kph ^ 1);
                mbar_expect_tx(&k_full[ks], (uint32_t)(KB * FA_BLK));
                for (int kb = 0; kb < KB; ++kb)
                    tma_load_2d(&map_k, &k_full[ks], Ks + (ks * FA_KBMAX + kb) * FA_BLK, 0,
                                krow0 + (j * KB + kb) * 128, pol);
                if (++ks == 2) {
                    ks = 0;
                    kph ^= 1;
                }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            uint32_t vph = 0;
            for (int j = 0; j < nj; ++j) {
                mbar_wait(v_empty, vph ^ 1);
                mbar_expect_tx(v_full, (uint32_t)(dv * 256));
                tma_load_2d(&map_v, v_full, Vs, j * FA_BKEY, bh * dv, pol);
                tma_load_2d(&map_v, v_full, Vs + dv * 128, j * FA_BKEY + 64, bh * dv, pol);
                vph ^= 1;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id_s = tc::idesc_bf16(128, FA_BKEY), id_o = tc::idesc_bf16(128, dv);
            const uint64_t qd0 = tc::desc_sw128(smem_u32(Qs)), kd0 = tc::desc_sw128(smem_u32(Ks)),
                           vd0 = tc::desc_sw128(smem_u32(Vs));
            int ks = 0;
            uint32_t kph = 0, vph = 0, pph[2] = {0, 0};
            // S_X = Q_X K^T of the K tile in stage ks
            auto issue_s = [&](int x) {
                for (int kb = 0; kb < KB; ++kb)
                    tc::mma_k4(tmem + x * 128, qd0 + (uint64_t)(((x * FA_KBMAX + kb) * FA_BLK) >> 4),
                               kd0 + (uint64_t)(((ks * FA_KBMAX + kb) * FA_BLK) >> 4), id_s, kb != 0);
                tc::commit(&s_full[x]);
            };
            // O_X (+)= P_X V_j, P_X = bf16 pairs in the S_X columns
            auto issue_pv = [&](int x, int j) {
                mbar_wait(&p_full[x], pph[x]);
                pph[x] ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int h = 0; h < 2; ++h)  // the two 64-key halves of V^T
                    tc::mma_ts_k4(tmem + 256 + x * 128, tmem + x * 128 + h * 32,
                                  vd0 + (uint64_t)((h * dv * 128) >> 4), id_o, (j | h) != 0);
                if (j == (x ? tB : tA)) tc::commit(&o_done[x]);  // the tile's last P.V
            };
            auto next_k = [&]() {
                tc::commit(&k_empty[ks]);
                if (++ks == 2) {
                    ks = 0;
                    kph ^= 1;
                }
            };
            mbar_wait(q_full, 0);
            mbar_wait(&k_full[ks], kph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            issue_s(0);
            if (hasB) issue_s(1);
            next_k();
            for (int j = 0; j < nj; ++j) {
                mbar_wait(v_full, vph);
                vph ^= 1;
                const bool more = j + 1 < nj;
                if (j <= tA) issue_pv(0, j);
                if (more) {
                    mbar_wait(&k_full[ks], kph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (j + 1 <= tA) issue_s(0);
                }
                if (hasB) issue_pv(1, j);
                tc::commit(v_empty);  // V_{j+1} streams in under S_B(j+1)
                if (more) {
                    if (hasB) issue_s(1);
                    next_k();
                }
            }
        }
    } else {
        const int x = (warp - 3) >> 2;  // 0: tile A, 1: tile B
        if (x == 0 || hasB) {
            const int quad = warp & 3;  // TMEM lanes this warp may access
            const int r = quad * 32 + lane;
            const int tx = x ? tB : tA;
            const int q = tx * FA_BQ + r;
            const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
            const uint32_t s_col = tmem + lane_off + x * 128;
            const uint32_t o_col = tmem + lane_off + 256 + x * 128;
            float m_ref = -INFINITY, l = 0.f;
            uint32_t sph = 0;
            uint32_t v[4][32];
            for (int j = 0; j <= tx; ++j) {
                mbar_wait(&s_full[x], sph);
                sph ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 4; ++c) tc::ld32(s_col + c * 32, v[c]);
                tc::ld_wait();
                if (j == tx) {  // the diagonal tile: keys past the query get p = 0
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (c * 32 + i > r) v[c][i] = __float_as_uint(-INFINITY);
                }
                float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(v[c][i]));
                const float cm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * a.scale_log2;
                float alpha = 1.f;
                const bool move = cm > m_ref + 8.f;  // true on the first tile (m_ref = -inf)
                if (move) {
                    alpha = ex2_fast(m_ref - cm);
                    l *= alpha;
                    m_ref = cm;
                }
                const float nm = -m_ref;
                float add[4] = {0.f, 0.f, 0.f, 0.f};
                // P word w = bf16(s[2w]) | bf16(s[2w+1]) << 16, packed in place
#pragma unroll
                for (int w = 0; w < 64; ++w) {
                    const float s0 = __uint_as_float(v[(2 * w) >> 5][(2 * w) & 31]);
                    const float s1 = __uint_as_float(v[(2 * w + 1) >> 5][(2 * w + 1) & 31]);
                    const float p0 = ex2_fast(fmaf(s0, a.scale_log2, nm));
                    const float p1 = ex2_fast(fmaf(s1, a.scale_log2, nm));
                    add[(w & 1) * 2] += p0;
                    add[(w & 1) * 2 + 1] += p1;
                    const __nv_bfloat162 pk = __floats2bfloat162_rn(p0, p1);
                    v[w >> 5][w & 31] = *reinterpret_cast<const uint32_t*>(&pk);
                }
                l += (add[0] + add[1]) + (add[2] + add[3]);
                if (move && j > 0) {  // O_X is quiescent: P_X(j-1) V landed before S_X(j)
                    for (int c = 0; c < dv / 32; ++c) {
                        uint32_t o[32];
                        tc::ld32(o_col + c * 32, o);
                        tc::ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                        tc::st32(o_col + c * 32, o);
                    }
                }
                tc::st32(s_col, v[0]);
                tc::st32(s_col + 32, v[1]);
                tc::st_wait();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[x]);
            }
            mbar_wait(&o_done[x], 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const float inv = 1.f / l;
            const int bb = bh / a.H, h = bh % a.H;
            __nv_bfloat16* dst = a.merged + ((size_t)bb * a.L + q) * a.ldm + (size_t)h * dv;
            for (int c = 0; c < dv / 32; ++c) {
                tc::ld32(o_col + c * 32, v[0]);
                tc::ld_wait();
                if (q < a.L) {
#pragma unroll
                    for (int u8 = 0; u8 < 4; ++u8) {
                        uint32_t w4[4];
#pragma unroll
                        for (int h2 = 0; h2 < 4; ++h2) {
                            const int i0 = u8 * 8 + h2 * 2;
                            const __nv_bfloat162 pk = __floats2bfloat162_rn(
                                __uint_as_float(v[0][i0]) * inv, __uint_as_float(v[0][i0 + 1]) * inv);
                            w4[h2] = *reinterpret_cast<const uint32_t*>(&pk);
                        }
                        *reinterpret_cast<uint4*>(dst + c * 32 + u8 * 8) =
                            make_uint4(w4[0], w4[1], w4[2], w4[3]);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// merged[(b*L + q)][h*dhc + c] = Ot[(bh*dhc + c)][q]: 32x32 tile transpose.
__global__ void mla_unpack_o_kernel(const __nv_bfloat16* __restrict__ Ot, int H, int L, int Lp,
                                    int dhc, __nv_bfloat16* __restrict__ merged) {
    __shared__ float tile[32][33];
    const int bh = blockIdx.z, b = bh / H, h = bh % H;
    const int q0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, q = q0 + threadIdx.x;
        tile[i][threadIdx.x] =
            c < dhc && q < L ? __bfloat162float(Ot[((size_t)bh * dhc + c) * Lp + q]) : 0.f;
    }
    __syncthreads();
    const size_t ldm = (size_t)H * dhc;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int q = q0 + i, c = c0 + threadIdx.x;
        if (q < L && c < dhc)
            merged[((size_t)b * L + q) * ldm + (size_t)h * dhc + c] =
                __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
}

// groups x ceil(rows_per_group / tile) token tiles, expert-major (pad = index
// in the group << 16 | tiles per group, for the GEMM's sibling scheduling).
__global__ void uniform_tiles_kernel(int groups, int rows_per_group, int tile,
                                     TokenTile* __restrict__ tiles, int* __restrict__ n_out) {
    const int nt = (rows_per_group + tile - 1) / tile;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < groups * nt) {
        const int g = i / nt, k = i % nt;
        tiles[i] = TokenTile{g, g * rows_per_group + k * tile, min(tile, rows_per_group - k * tile),
                             (k << 16) | nt};
    }
    if (i == 0) *n_out = groups * nt;
}

// out[r][j] = float(O[r][j]) (+ residual[r][j]), O with row stride ldo.
__global__ void mla_out_f32_kernel(const __nv_bfloat16* __restrict__ O, size_t ldo, size_t rows,
                                   size_t d, float* __restrict__ out) {
    const size_t n = rows * d;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = __bfloat162float(O[(i / d) * ldo + i % d]);
}

TokenTile* uniform_tiles(scmoe_ctx* c, DevBuf& buf, int groups, int rows_per_group, int tile,
                         size_t* max_tiles, int** n_dev) {
    const size_t nt = (size_t)groups * ceil_div((size_t)rows_per_group, (size_t)tile);
    TokenTile* t = buf.get<TokenTile>(nt + 1);
    *n_dev = reinterpret_cast<int*>(t + nt);
    *max_tiles = nt;
    uniform_tiles_kernel<<<ceil_div(std::max<size_t>(nt, 1), 256), 256, 0, c->stream>>>(
        groups, rows_per_group, tile, t, *n_dev);
    SCMOE_LAUNCH_CHECK(c);
    return t;
}

int gs(scmoe_ctx* c, size_t n) {
    return (int)std::min<size_t>(ceil_div(std::max<size_t>(n, 1), 256), (size_t)c->num_sms * 16);
}

}  // namespace

// bf16 blocked weights from the fp32 device weights (re-done when a weight changed).
void mla_prepare_tc(scmoe_ctx* c, scmoe_mla* m) {
    if (!m->tc_dirty) return;
    const size_t H = m->H;
    const size_t Ks[4] = {m->d, m->dq, m->dkv, H * m->dhc};
    const size_t Ns[4] = {m->n1(), m->n2(), m->n3(), m->d};
    const float* src[4] = {m->w_h, m->w_q, m->w_kv, m->w_o};
    for (int i = 0; i < 4; ++i) {
        const size_t M = pad_to(Ns[i], 256);
        m->tc_M[i] = M;
        if (!m->tc_w[i]) SCMOE_CUDA(cudaMalloc(&m->tc_w[i], M * Ks[i] * sizeof(__nv_bfloat16)));
        SCMOE_CUDA(cudaMemsetAsync(m->tc_w[i], 0, M * Ks[i] * sizeof(__nv_bfloat16), c->stream));
        // src [K][N] row-major -> blocked W[m = n][k]
        // the latent scalings (cq * alpha_q, ckv * alpha_kv) fold into W_h's columns
        if (i == 0)
            launch_f32_to_bf16_t(c, src[i], Ks[i], Ns[i], m->tc_w[i], (int)m->dq, m->alpha_q,
                                 (int)m->dkv, m->alpha_kv);
        else
            launch_f32_to_bf16_t(c, src[i], Ks[i], Ns[i], m->tc_w[i]);
    }
    m->tc_dirty = false;
}

void mla_forward_tc(scmoe_ctx* c, scmoe_mla* m, const float* h, size_t rows, size_t L,
                    const float2* rope, float* out) {
    mla_prepare_tc(c, m);
    Workspace& ws = c->ws;
    const size_t d = m->d, dq = m->dq, dkv = m->dkv, H = m->H, dhc = m->dhc, dhr = m->dhr;
    const size_t B = rows / L, BH = B * H;
    const size_t M1 = m->tc_M[0], M2 = m->tc_M[1], M3 = m->tc_M[2], M4 = m->tc_M[3];
    const size_t Lp = pad_to(L, 256), Dk = pad_to(dhc + dhr, 64);
    if (BH * Lp * Dk >= (size_t(1) << 31))
        SCMOE_THROW(SCMOE_ERR_CONFIG, "mla: tensor-core path limited to B*H*L*(dhc+dhr) < 2^31");
    const int TR = grouped_gemm_tile_rows_large();
    __nv_bfloat16* xb = ws.mtc_x.get<__nv_bfloat16>(rows * d);
    __nv_bfloat16* p1 = ws.mtc_p1.get<__nv_bfloat16>(rows * M1);
    __nv_bfloat16* qb = ws.mtc_q.get<__nv_bfloat16>(rows * M2);
    __nv_bfloat16* kv = ws.mtc_kv.get<__nv_bfloat16>(rows * M3);
    __nv_bfloat16* qrows = ws.mtc_qr.get<__nv_bfloat16>(BH * L * Dk);
    __nv_bfloat16* kblk = ws.mtc_kb.get<__nv_bfloat16>(BH * Lp * Dk);
    __nv_bfloat16* vt = ws.mtc_vt.get<__nv_bfloat16>(BH * dhc * Lp);
    __nv_bfloat16* mg = ws.mtc_mg.get<__nv_bfloat16>(rows * H * dhc);
    __nv_bfloat16* ob = ws.mtc_o.get<__nv_bfloat16>(rows * M4);
    size_t mt_rows = 0, mt_s = 0, mt_pv = 0;
    int *n_rows = nullptr, *n_s = nullptr, *n_pv = nullptr;
    TokenTile* t_rows = uniform_tiles(c, ws.mtc_t0, 1, (int)rows, TR, &mt_rows, &n_rows);
    TokenTile* t_s = uniform_tiles(c, ws.mtc_t1, (int)BH, (int)L, TR, &mt_s, &n_s);
    TokenTile* t_pv = uniform_tiles(c, ws.mtc_t2, (int)BH, (int)dhc, TR, &mt_pv, &n_pv);
    {
        ProfScope _p(c, "mla_tc_proj_h");
        launch_cast_bf16(c, h, rows * d, xb);
        // alpha_q / alpha_kv are folded into W_h; rope is applied by the packing
        launch_grouped_gemm_bf16(c, m->tc_w[0], 1, M1, d, xb, rows, nullptr, p1, 0, t_rows, n_rows,
                                 mt_rows, TR);
    }
    {
        ProfScope _p(c, "mla_tc_proj_q");
        launch_grouped_gemm_bf16(c, m->tc_w[1], 1, M2, dq, p1, rows, nullptr, qb, 0, t_rows, n_rows,
                                 mt_rows, TR, nullptr, nullptr, M1);
    }
    {
        ProfScope _p(c, "mla_tc_proj_kv");
        launch_grouped_gemm_bf16(c, m->tc_w[2], 1, M3, dkv, p1 + dq, rows, nullptr, kv, 0, t_rows,
                                 n_rows, mt_rows, TR, nullptr, nullptr, M1);
    }
    {
        ProfScope _p(c, "mla_tc_pack");
        // 16-byte accesses need 8-element aligned sources: dhc, dhr, dq + dkv, the
        // row strides and the kr column
        if (dhc % 8 == 0 && dhr % 8 == 0 && (dq + dkv) % 8 == 0)
            mla_pack_qk8_kernel<<<gs(c, BH * Lp * Dk / 8), 256, 0, c->stream>>>(
                qb, M2, kv, M3, p1, M1, (int)(dq + dkv), (int)BH, (int)H, (int)L, (int)Lp,
                (int)dhc, (int)dhr, (int)Dk, rope, qrows, kblk);
        else
            mla_pack_qk_kernel<<<gs(c, BH * Lp * Dk), 256, 0, c->stream>>>(
                qb, M2, kv, M3, p1, M1, (int)(dq + dkv), (int)BH, (int)H, (int)L, (int)Lp,
                (int)dhc, (int)dhr, (int)Dk, rope, qrows, kblk);
        SCMOE_LAUNCH_CHECK(c);
    }
    static const bool fused = [] {
        const char* e = getenv("SCMOE_MLA_ATTN");
        return !(e && std::string(e) == "gemm");
    }();
    if (fused && Dk <= 64 * FA_KBMAX && dhc % 32 == 0 && dhc <= FA_DVMAX) {
        ProfScope _p(c, "mla_tc_attention");
        mla_pack_vt_kernel<<<dim3((unsigned)ceil_div(dhc, 32), (unsigned)(Lp / 32), (unsigned)BH),
                             dim3(32, 8), 0, c->stream>>>(kv, M3, (int)H, (int)L, (int)Lp,
                                                          (int)dhc, vt);
        SCMOE_LAUNCH_CHECK(c);
        const CUtensorMap mq = make_tma_map_2d(qrows, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, BH * L, Dk,
                                               128, 64, CU_TENSOR_MAP_SWIZZLE_128B);
        const CUtensorMap mk = make_tma_map_2d(kblk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                               BH * Lp * Dk / 64, 64, 128, 64,
                                               CU_TENSOR_MAP_SWIZZLE_128B);
        const CUtensorMap mv = make_tma_map_2d(vt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, BH * dhc, Lp,
                                               (uint32_t)dhc, 64, CU_TENSOR_MAP_SWIZZLE_128B);
        FaArgs fa;
        fa.BH = (int)BH;
        fa.H = (int)H;
        fa.L = (int)L;
        fa.Lp = (int)Lp;
        fa.nqt = (int)ceil_div(L, (size_t)FA_BQ);
        fa.KB = (int)(Dk / 64);
        fa.dv = (int)dhc;
        fa.scale_log2 = m->att_scale * 1.4426950408889634f;
        fa.merged = mg;
        fa.ldm = H * dhc;
        static const bool one_tile = [] {
            const char* e = getenv("SCMOE_MLA_ATTN");
            return e && std::string(e) == "flash1";
        }();
        if (one_tile) {
            ensure_max_dynamic_smem(reinterpret_cast<const void*>(mla_flash_kernel), (int)FA_SMEM,
                                    c->device);
            mla_flash_kernel<<<(unsigned)(BH * fa.nqt), FA_THREADS, FA_SMEM, c->stream>>>(mq, mk,
                                                                                          mv, fa);
        } else {
            ensure_max_dynamic_smem(reinterpret_cast<const void*>(mla_flash2_kernel), (int)F2_SMEM,
                                    c->device);
            mla_flash2_kernel<<<(unsigned)(BH * ((fa.nqt + 1) / 2)), F2_THREADS, F2_SMEM,
                                c->stream>>>(mq, mk, mv, fa);
        }
        SCMOE_LAUNCH_CHECK(c);
    } else {
    // the unfused path materialises S and P (BH x Lp^2 each: GBs at long L)
    __nv_bfloat16* S = ws.mtc_s.get<__nv_bfloat16>(BH * L * Lp);
    __nv_bfloat16* P = ws.mtc_p.get<__nv_bfloat16>(BH * Lp * Lp);
    __nv_bfloat16* ot = ws.mtc_ot.get<__nv_bfloat16>(BH * dhc * Lp);
    {
        ProfScope _p(c, "mla_tc_scores");
        // causal: key blocks above a query tile's last query are skipped
        launch_grouped_gemm_bf16(c, kblk, BH, Lp, Dk, qrows, BH * L, nullptr, S, 0, t_s, n_s, mt_s,
                                 TR, nullptr, nullptr, 0, (int)L, 0);
    }
    {
        ProfScope _p(c, "mla_tc_softmax");
        const size_t warps = BH * Lp;
        mla_softmax_bf16_kernel<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, c->stream>>>(
            S, (int)BH, (int)L, (int)Lp, m->att_scale, P);
        SCMOE_LAUNCH_CHECK(c);
    }
    {
        ProfScope _p(c, "mla_tc_pv");
        mla_pack_vt_kernel<<<dim3((unsigned)ceil_div(dhc, 32), (unsigned)(Lp / 32), (unsigned)BH),
                             dim3(32, 8), 0, c->stream>>>(kv, M3, (int)H, (int)L, (int)Lp,
                                                          (int)dhc, vt);
        SCMOE_LAUNCH_CHECK(c);
        // causal: query block mb reduces over keys < (mb + 1) * 256 only
        launch_grouped_gemm_bf16(c, P, BH, Lp, Lp, vt, BH * dhc, nullptr, ot, 0, t_pv, n_pv, mt_pv,
                                 TR, nullptr, nullptr, 0, 0, 1);
        mla_unpack_o_kernel<<<dim3((unsigned)ceil_div(dhc, 32), (unsigned)(Lp / 32), (unsigned)BH),
                              dim3(32, 8), 0, c->stream>>>(ot, (int)H, (int)L, (int)Lp, (int)dhc,
                                                           mg);
        SCMOE_LAUNCH_CHECK(c);
    }
    }
    ProfScope _p(c, "mla_tc_proj_o");
    launch_grouped_gemm_bf16(c, m->tc_w[3], 1, M4, H * dhc, mg, rows, nullptr, ob, 0, t_rows,
                             n_rows, mt_rows, TR);
    mla_out_f32_kernel<<<gs(c, rows * d), 256, 0, c->stream>>>(ob, M4, rows, d, out);
    SCMOE_LAUNCH_CHECK(c);
}

}  // namespace scmoe
