// internal.cuh -- shared state and helpers of libscmoe (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/scmoe.h"

// ---------------------------------------------------------------------------
// Status plumbing.  The C ABI maps the reference's exceptions to codes
// (common.hpp:11-33); ScmoeError carries one through the C++ implementation.
// ---------------------------------------------------------------------------
struct ScmoeError {
    int code;
    std::string msg;
};

#define SCMOE_THROW(code, msg) throw ScmoeError{(code), (msg)}
#define SCMOE_CHECK_ARG(cond, code, msg) \
    do {                                 \
        if (!(cond)) SCMOE_THROW(code, msg); \
    } while (0)
#define SCMOE_CUDA(expr)                                                                      \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            SCMOE_THROW(SCMOE_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
    } while (0)

// Device-side latched errors (written by kernels that validate data).
enum : int {
    DEV_OK = 0,
    DEV_ERR_INDEX_RANGE = 1,
    DEV_ERR_COUNTERS = 2,
    DEV_ERR_EMPTY = 3,    // bias_update on an empty batch (router.hpp:157), device-side seen
    DEV_ERR_CAPACITY = 4, // expert-parallel receive buffer capacity exceeded
    DEV_ERR_TIMEOUT = 5   // expert-parallel peer barrier timed out (a rank did not arrive)
};

// ---------------------------------------------------------------------------
// Grow-only device workspace.
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    template <typename T>
    T* get(size_t n) {
        size_t need = n * sizeof(T);
        if (need == 0) need = 16;
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            bytes = 0;
            // round up to 2 MiB so repeated growth is rare
            size_t cap = (need + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
            SCMOE_CUDA(cudaMalloc(&p, cap));
            bytes = cap;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct Workspace {
    DevBuf logits, probs, hmoe, hmoe_bf16, idx, gates, ffn_count;
    DevBuf rank_in_block, block_counts, expert_count, expert_base, slot_pos, row_token;
    DevBuf tiles, n_tiles, xp, h, y, in_copy, out_copy, misc, tiles_router, ep_bins, ep_local,
        ep_y;
    // dense shortcut FFN (scmoe_dense_ffn): own buffers, so it can run on
    // another stream beside the MoE branch
    DevBuf dn_x, dn_h, dn_y, dn_tiles;
    // MLA (mla.cu): projections, scores/weights, merged heads, row tiles
    DevBuf mla_p1, mla_q, mla_kv, mla_att, mla_m, mla_tiles;
    // full ScMoE layer (scmoe_layer_full_forward): normed input, MLA output, a1, dd, a3
    DevBuf full_n, full_m, full_a1, full_dd, full_a3;
    // tensor-core MLA (mla_tc.cu)
    DevBuf mtc_x, mtc_p1, mtc_q, mtc_kv, mtc_qr, mtc_kb, mtc_s, mtc_p, mtc_vt, mtc_ot, mtc_mg,
        mtc_o, mtc_t0, mtc_t1, mtc_t2;
    unsigned char pr_blob[64] = {};  // permutation result carried from moe_front to moe_back
    void release_all() {
        DevBuf* all[] = {&logits, &probs, &hmoe, &hmoe_bf16, &idx, &gates, &ffn_count,
                         &rank_in_block, &block_counts, &expert_count, &expert_base, &slot_pos,
                         &row_token, &tiles, &n_tiles, &xp, &h, &y, &in_copy, &out_copy, &misc,
                         &tiles_router, &ep_bins, &ep_local, &ep_y, &dn_x, &dn_h, &dn_y,
                         &dn_tiles, &mla_p1, &mla_q, &mla_kv, &mla_att, &mla_m, &mla_tiles, &full_n, &full_m, &full_a1,
                         &full_dd, &full_a3, &mtc_x, &mtc_p1, &mtc_q, &mtc_kv, &mtc_qr, &mtc_kb,
                         &mtc_s, &mtc_p, &mtc_vt, &mtc_ot, &mtc_mg, &mtc_o, &mtc_t0, &mtc_t1,
                         &mtc_t2};
        for (DevBuf* b : all) b->release();
    }
};

// Optional per-kernel timing: CUDA events recorded on the launching stream
// around each named stage (scmoe_profile_* in the ABI).
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
struct ProfAgg {
    std::string name;
    double ms = 0.0;
    uint64_t count = 0;
};
struct Profiler {
    bool on = false;
    std::vector<ProfRec> recs;
    size_t used = 0;
    std::vector<ProfAgg> agg;
    struct Span {
        std::string name;
        double start_ms, end_ms;  // relative to the first record of the flush
    };
    std::vector<Span> spans;
};

struct HostStage {
    DevBuf bufs[12];
};

struct scmoe_ctx {
    HostStage stage;  // host-tier (_host) staging buffers
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string last_error;
    int* dev_status = nullptr;  // latched device-side error
    uint64_t launches = 0;
    Workspace ws;
    Profiler prof;
    bool gemm1_gather = false;  // GEMM1 B operand via TMA gather4 (SCMOE_GEMM1_GATHER=1)
    // router projection kernel: 0 auto, 1 slab (56 tokens x E, 1 CTA/SM),
    // 2 lean (co-resides with the GEMM), 3 tiled (64/16-row tiles), 4 tma (slab
    // tile fed by TMA, the large-batch default); SCMOE_ROUTER
    int router_variant = 0;
    // SM budget (CTAs) of the persistent router / grouped GEMM kernels; 0 = all
    // (SCMOE_ROUTER_SMS / SCMOE_GEMM_SMS, or the overlapped schedule's split)
    int router_sms = 0, gemm_sms = 0;
    bool overlapped = false;    // inside a pipelined multi-batch call
    // this context's grouped GEMMs run beside the co-resident router of another
    // stream: pick the smaller-footprint ring for 256-token tiles
    bool corun_gemm = false;
    // pipelined multi-batch execution (scmoe_layer_forward_batches)
    cudaStream_t s_front = nullptr, s_back = nullptr;
    cudaEvent_t ev_front[2] = {nullptr, nullptr}, ev_back[2] = {nullptr, nullptr};
    cudaEvent_t ev_join = nullptr;
    Workspace ws_alt;
    // host-batch pipeline (scmoe_layer_forward_host_batches): copy streams,
    // per-slot events and double-buffered device I/O
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_in_a1[2] = {nullptr, nullptr};  // host tier: a1 landed (a3 may follow)
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
                ev_out[2] = {nullptr, nullptr};
    DevBuf io[2][7];
    // full-layer overlap: the MoE branch's stream and its events
    cudaStream_t s_moe = nullptr;
    cudaEvent_t ev_full[3] = {nullptr, nullptr, nullptr};
};

// RAII stage timer; a no-op unless profiling is enabled on the context.
struct ProfScope {
    scmoe_ctx* c;
    size_t i = SIZE_MAX;
    ProfScope(scmoe_ctx* ctx, const char* name) : c(ctx) {
        if (!c->prof.on) return;
        Profiler& p = c->prof;
        if (p.used == p.recs.size()) {
            ProfRec r{name, nullptr, nullptr};
            cudaEventCreate(&r.a);
            cudaEventCreate(&r.b);
            p.recs.push_back(r);
        }
        i = p.used++;
        p.recs[i].name = name;
        cudaEventRecord(p.recs[i].a, c->stream);
    }
    ~ProfScope() {
        if (i != SIZE_MAX) cudaEventRecord(c->prof.recs[i].b, c->stream);
    }
};

struct scmoe_router {
    size_t d = 0, n_ffn = 0, n_zero = 0, top_k = 0, k_expected = 0;
    double mu = 0.0, mu_decay = 1.0;
    uint64_t tokens_seen = 0;  // host mirror of RouterState::tokens_seen
    float* w = nullptr;         // [d, E] fp32
    double* b = nullptr;        // [E]
    uint64_t* routed = nullptr; // [E]
    size_t E() const { return n_ffn + n_zero; }
};

struct scmoe_bank {
    size_t n = 0, d = 0, inter = 0, m = 1;
    int precision = SCMOE_PREC_F32_EXACT;
    int gamma_mode = SCMOE_GAMMA_FFN_ONLY;
    float* w_in32 = nullptr;          // [n][d][inter]   (F32_EXACT)
    float* w_out32 = nullptr;         // [n][inter][d]
    __nv_bfloat16* w1t = nullptr;     // [n][inter][d]   (BF16, K-major for GEMM1)
    __nv_bfloat16* w2t = nullptr;     // [n][d][inter]   (BF16, K-major for GEMM2)
    double* w_in64 = nullptr;         // [n][d][inter]   (F64_EXACT)
    double* w_out64 = nullptr;        // [n][inter][d]
    double gamma_ffn() const { return gamma_mode == SCMOE_GAMMA_OFF ? 1.0 : (double)m; }
    double gamma_zero() const { return gamma_mode == SCMOE_GAMMA_ALL ? (double)m : 1.0; }
};

// Blocked K-major layout of one expert's bf16 weight matrix W[M][K] (the
// tcgen05 GEMM's A operand): 128-row x 64-column tiles stored contiguously,
// tile (m/128, k/64) at ((m/128) * K/64 + k/64) * 8192 elements, row-major
// inside (128 B rows).  Every TMA box the GEMM loads is then one contiguous
// 16 KB read.  Requires M % 128 == 0 and K % 64 == 0.
__host__ __device__ __forceinline__ size_t wblk_index(size_t m, size_t k, size_t K) {
    return (((m >> 7) * (K >> 6) + (k >> 6)) << 13) + ((m & 127) << 6) + (k & 63);
}

// One GEMM work tile: rows [pos, pos+count) of expert `e` in the permuted order.
struct TokenTile {
    int e, pos, count, pad;
};

// ---------------------------------------------------------------------------
// Kernel launchers (defined in the .cu files).
// ---------------------------------------------------------------------------
namespace scmoe {

constexpr int kPermTokensPerBlock = 256;

void launch_rmsnorm(scmoe_ctx* c, const float* x, const float* gain, size_t rows, size_t d,
                    float eps, float* out, __nv_bfloat16* out_bf16);
// C[rows, n] = A[rows, k] B[k, n], sequential k (router.hpp:136 / tensor.hpp:95-112).
void launch_seq_gemm(scmoe_ctx* c, const float* A, size_t lda, const int* a_rows,
                     const float* B, size_t ldb, size_t b_group_stride, float* C, size_t ldc,
                     size_t K, size_t N, int silu, const TokenTile* tiles, const int* n_tiles_dev,
                     size_t max_tiles, int tile_rows);
int seq_gemm_tile_rows(size_t rows, size_t N, int num_sms);
// Sequential-k GEMV for rows <= 4 (false: not applicable, nothing launched).
bool launch_seq_gemv(scmoe_ctx* c, const float* A, size_t lda, size_t rows, const float* B,
                     size_t ldb, float* C, size_t ldc, size_t K, size_t N);
// Router projection with one CTA per 56-token slab x all experts (E <= 768).
// Same tile as the slab kernel, operands by TMA into an mbarrier ring.
// RouterState<double>: projection and softmax/top-K in double.
void launch_router_f64(scmoe_ctx* c, const double* X, const double* W, double* logits, size_t T,
                       size_t K, size_t E);
void launch_softmax_topk_f64(scmoe_ctx* c, const double* logits, size_t T, size_t E, size_t K,
                             size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                             uint32_t* ffn, double* probs);
// moe_forward<double>: grouped sequential GEMM in double over token tiles
// (rows a_rows[pos + r] of A, or A rows pos + r), optional SiLU, and the
// double combine.
void launch_seq_gemm_f64(scmoe_ctx* c, const double* A, size_t lda, const int* a_rows,
                         const double* B, size_t ldb, size_t b_group_stride, double* C,
                         size_t ldc, size_t K, size_t N, int silu, const TokenTile* tiles,
                         const int* n_tiles_dev, size_t max_tiles);
void launch_combine_f64(scmoe_ctx* c, const double* x, const double* y, const uint32_t* idx,
                        const double* gates, const int* slot_pos, size_t T, size_t d, size_t K,
                        size_t n_ffn, double gamma_ffn, double gamma_zero, int renorm,
                        const double* residual, double* out);
void launch_debug_exp(scmoe_ctx* c, const double* in, double* out, size_t n);
bool router_tma_ok(size_t T, size_t K, size_t E, int num_sms);
void launch_router_tma(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                       size_t K, size_t E);
// Small-footprint persistent TMA router that co-resides with the grouped GEMM.
bool router_corun_ok(size_t T, size_t K, size_t E);
void launch_router_corun(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                         size_t K, size_t E);
bool router_slab_ok(size_t T, size_t K, size_t E, int num_sms);
// Router projection sized to co-reside with the grouped GEMM (28-token slabs).
bool router_lean_ok(size_t K, size_t E);
bool router_small_ok(size_t T, size_t K, size_t E, int num_sms);
bool front_small_ok(size_t T, size_t d, size_t E, size_t K, int num_sms);
void launch_front_small(scmoe_ctx* c, const float* a1, const float* gain, size_t T, size_t d,
                        float eps, const float* W, size_t E, size_t K, size_t n_ffn,
                        const double* bias, float* hmoe, __nv_bfloat16* hb, uint32_t* idx,
                        double* gates, uint32_t* ffn_count);
void launch_router_small(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                         size_t K, size_t E);
void launch_router_lean(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                        size_t K, size_t E);
void launch_router_slab(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                        size_t K, size_t E);
void launch_softmax_topk(scmoe_ctx* c, const float* logits, size_t T, size_t E, size_t K,
                         size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                         uint32_t* ffn_count, float* probs_out);
void launch_topk_from_probs_f32(scmoe_ctx* c, const float* probs, size_t T, size_t E, size_t K,
                                size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                                uint32_t* ffn_count);
void launch_topk_from_probs_f64(scmoe_ctx* c, const double* probs, size_t T, size_t E, size_t K,
                                size_t n_ffn, const double* bias, uint32_t* idx, double* gates,
                                uint32_t* ffn_count);

struct PermResult {
    int* slot_pos;      // [T*K], -1 for zero experts
    int* row_token;     // [T*K] upper bound; first total entries valid
    int* expert_base;   // [n_ffn+1]
    int* expert_count;  // [E]
    TokenTile* tiles;   // [max_tiles]
    int* n_tiles;       // device scalar
    size_t max_tiles;
};
// multi: a token may hit the same bin in several slots (EP destination ranks);
// otherwise each token hits an expert at most once (top-K of distinct experts).
// T_dev: the token count lives on the device (T is then the capacity the
// grids and buffers are sized for; expert-parallel receive side).
PermResult launch_permute(scmoe_ctx* c, const uint32_t* idx, size_t T, size_t K, size_t n_ffn,
                          size_t E, int tile_rows, bool multi = false,
                          const int* T_dev = nullptr);
void launch_gather_bf16(scmoe_ctx* c, const __nv_bfloat16* src, size_t d, const int* row_token,
                        const int* expert_base, size_t n_ffn, size_t max_rows,
                        __nv_bfloat16* dst);
void launch_combine_f32(scmoe_ctx* c, const float* x, const float* y, const uint32_t* idx,
                        const double* gates, const int* slot_pos, size_t T, size_t d, size_t K,
                        size_t n_ffn, float gamma_ffn, float gamma_zero, int renorm,
                        const float* residual, float* out);
void launch_combine_bf16(scmoe_ctx* c, const float* x, const __nv_bfloat16* y,
                         const uint32_t* idx, const double* gates, const int* slot_pos, size_t T,
                         size_t d, size_t K, size_t n_ffn, float gamma_ffn, float gamma_zero,
                         int renorm, const float* residual, float* out);
void launch_check_indices(scmoe_ctx* c, const uint32_t* idx, size_t n, size_t E);
void launch_ffn_moments(scmoe_ctx* c, const uint32_t* cnt, size_t T, double* out);
void launch_accumulate(scmoe_ctx* c, const uint32_t* idx, size_t n, size_t E, uint64_t* routed);
// routed / seen_dev (optional): counters and tokens_seen already on the device
// (summed over the expert-parallel ranks); default: the router's own counters
// and its host mirror of tokens_seen.
void launch_bias_update(scmoe_ctx* c, scmoe_router* r, double* delta_dev,
                        const uint64_t* routed = nullptr, const uint64_t* seen_dev = nullptr);
void launch_uniform_init(scmoe_ctx* c, uint64_t seed, uint64_t first, size_t n,
                         double half_width, float* out);
void launch_uniform_init_bf16_t(scmoe_ctx* c, uint64_t seed, size_t rows, size_t cols,
                                double half_width, __nv_bfloat16* out_t);
void launch_debug_expf(scmoe_ctx* c, const float* in, float* out, size_t n);
void launch_debug_expf_range(scmoe_ctx* c, uint32_t first, float* out, size_t n);
void launch_cast_bf16(scmoe_ctx* c, const float* src, size_t n, __nv_bfloat16* dst);
void launch_row_tiles(scmoe_ctx* c, size_t rows, int tile_rows, TokenTile* tiles,
                      int* n_out = nullptr);
void launch_add_bf16_residual(scmoe_ctx* c, const float* a, const __nv_bfloat16* y, size_t n,
                              float* out);
void launch_f32_to_bf16_t(scmoe_ctx* c, const float* src, size_t rows, size_t cols,
                          __nv_bfloat16* dst_t, int n_a = 0, float alpha_a = 1.f, int n_b = 0,
                          float alpha_b = 1.f);

// tcgen05 grouped GEMM (gemm_sm100.cu).  D^T = W x X^T per expert tile:
//   out[pos, m] = epi( sum_k W[e][m][k] * X[pos][k] ),  epi = silu or identity,
// W: [n][M][K] bf16 (K-major), X: [rows][K] bf16, out: [rows][M] bf16.
// expert parallelism helpers (kernels_moe.cu)
void launch_ep_bins(scmoe_ctx* c, const uint32_t* idx, size_t n, size_t n_ffn, size_t per_rank,
                    int world, uint32_t* bins);
void launch_ep_send_expert(scmoe_ctx* c, const uint32_t* idx, const int* slot_pos, size_t n,
                           int* send_expert);
void launch_slot_rows(scmoe_ctx* c, const uint32_t* idx, const int* slot_pos,
                      const int* expert_base, size_t n, int n_ffn, int* slot_row);
void launch_ep_localize(scmoe_ctx* c, const int* row_expert, size_t n, int offset, int n_local,
                        uint32_t* local, const int* n_dev = nullptr);
void launch_gather_rows_bf16(scmoe_ctx* c, const __nv_bfloat16* src, size_t d, const int* rows,
                             size_t n_rows, __nv_bfloat16* dst);

// Expert FFN on rows that each carry one (global) expert id (capi.cu); with
// R_dev the count is read on the device and R is the capacity.
void moe_rows_impl(scmoe_ctx* c, scmoe_bank* b, const void* x_bf16, const int* row_expert,
                   int expert_offset, size_t R, void* y_bf16, const uint64_t* row_dst,
                   const int* R_dev);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to the device context, and callers may drive several
// devices from one process or thread.  Thread-safe.
void ensure_max_dynamic_smem(const void* kernel, int bytes, int device);

int grouped_gemm_tile_rows();        // 192: single-GPU prefill (router co-residency)
int grouped_gemm_tile_rows_large();  // 256: expert-parallel shards, dense FFN
void launch_grouped_gemm_bf16(scmoe_ctx* c, const __nv_bfloat16* W, size_t n_experts,
                              size_t M, size_t K, const __nv_bfloat16* X, size_t x_rows,
                              const int* x_row_ids, __nv_bfloat16* out, int silu,
                              const TokenTile* tiles,
                              const int* n_tiles_dev, size_t max_tiles, int tile_rows,
                              const uint64_t* row_dst = nullptr, const int* row_ids = nullptr,
                              size_t x_ld = 0, int causal_rows = 0, int causal_k = 0);
// Expert-parallel dispatch over peer memory: send row j (rows sorted by
// destination rank, send_start[G+1]) -> peer_rows[d] row dst_offset[d] + j - send_start[d].
void launch_ep_put_rows(scmoe_ctx* c, const __nv_bfloat16* src, size_t d, const int* send_token,
                        const int* send_expert, size_t n_send, const int* send_start,
                        const int64_t* dst_offset, const uint64_t* peer_rows,
                        const uint64_t* peer_expert, int G, int64_t cap_dst = INT64_MAX);

// ---- MLA (mla.cu) ----
// Attention operands of the (sequence b, head h) pairs.  Rows of sequence b
// start at b * nq (queries) and b * nk (keys); query i sits at absolute
// position q0 + i and sees keys j <= q0 + i.
struct MlaAttnArgs {
    const float* qc;  // query content [rows, ldq] (+ h*dhc)
    const float* qr;  // query rotary  [rows, ldq] (+ h*dhr)
    size_t ldq;
    const float* kc;  // key content [keys, ldkv] (+ h*dhc)
    const float* v;   // values      [keys, ldkv] (+ h*dhc)
    size_t ldkv;
    const float* kr;  // rotary key shared by the heads [keys, ldkr]
    size_t ldkr;
    float* att;       // [B][H][nq][nk] scores -> softmax weights, in place
    float* part_max;  // [B][H][nq][ceil(nk/64)] per-key-tile row maxima
    float* merged;    // [B*nq, ldm] (+ h*dhc)
    size_t ldm;
    int H, dhc, dhr, nq, nk, q0;
    float scale;
};
void launch_mla_scale_rope(scmoe_ctx* c, float* X, size_t ld, size_t rows, int n_a, float alpha_a,
                           int n_b, float alpha_b, int rc, int heads, int hd, const float2* table,
                           size_t pos0, size_t seq_len);
void launch_mla_attention(scmoe_ctx* c, const MlaAttnArgs& a, int batches);
void launch_add_f32(scmoe_ctx* c, const float* a, const float* b, size_t n, float* out);
// tensor-core MLA forward (mla_tc.cu); rope = the (cos, sin) table of m
void mla_forward_tc(scmoe_ctx* c, scmoe_mla* m, const float* h, size_t rows, size_t seq_len,
                    const float2* rope, float* out);

}  // namespace scmoe

// MlaParams<float> (blocks.hpp:38-58) resident on the device.  The projections
// that share an input are stored column-concatenated so each runs as one GEMM:
//   w_h  [d,   dq + dkv + dhr] = [w_dq | w_dkv | w_kr]
//   w_q  [dq,  H*dhc + H*dhr]  = [w_uq | w_qr]
//   w_kv [dkv, 2*H*dhc]        = [w_uk | w_uv]
//   w_o  [H*dhc, d]
struct scmoe_mla {
    size_t d = 0, dq = 0, dkv = 0, H = 0, dhc = 0, dhr = 0;
    double rope_base = 1.0e6;
    int variance_alignment = 1;
    float alpha_q = 1.f, alpha_kv = 1.f, att_scale = 1.f;
    float *w_h = nullptr, *w_q = nullptr, *w_kv = nullptr, *w_o = nullptr;
    float2* rope = nullptr;  // (cos, sin) [rope_rows][dhr/2]
    size_t rope_rows = 0;
    // forward precision: SCMOE_PREC_F32_EXACT (bitwise, mla.cu) or SCMOE_PREC_BF16
    // (tensor cores, mla_tc.cu); the bf16 blocked weights [w_h | w_q | w_kv | w_o]
    // (rows padded to 256) are rebuilt from the fp32 ones after a weight change
    int precision = SCMOE_PREC_F32_EXACT;
    bool tc_dirty = true;
    __nv_bfloat16* tc_w[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t tc_M[4] = {0, 0, 0, 0};
    size_t n1() const { return dq + dkv + dhr; }
    size_t n2() const { return H * (dhc + dhr); }
    size_t n3() const { return 2 * H * dhc; }
};

// MlaCache (blocks.hpp:106-112) plus the expanded content keys / values of
// the cached rows (kc = c_kv W_uk and vv = c_kv W_uv are row-wise, so caching
// them is bitwise the reference's per-step re-expansion).
struct scmoe_mla_cache {
    size_t len = 0, cap = 0;
    float* c_kv = nullptr;  // [cap, dkv]
    float* k_r = nullptr;   // [cap, dhr] (rotated)
    float* kv = nullptr;    // [cap, 2*H*dhc] = [kc | vv]
};

#define SCMOE_LAUNCH_CHECK(c)                                                               \
    do {                                                                                    \
        (c)->launches++;                                                                    \
        cudaError_t _e = cudaGetLastError();                                                \
        if (_e != cudaSuccess)                                                              \
            SCMOE_THROW(SCMOE_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

static inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }
