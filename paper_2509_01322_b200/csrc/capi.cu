// capi.cu -- the extern "C" boundary (include/scmoe.h).
//
// Host-side validation reproduces the reference's checks and exception types
// (router.hpp:45-61, :112, :157-162; blocks.hpp:237-238, :348, :375-377);
// all numeric work is done by the CUDA kernels.  There is no CPU compute
// path: without a device every entry point fails with SCMOE_ERR_CUDA.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

using namespace scmoe;

namespace scmoe {
// Raises a kernel's dynamic shared-memory limit on this device to at least
// `bytes` (remembering the largest value set, so a later, larger request for
// the same kernel raises it again).
void ensure_max_dynamic_smem(const void* kernel, int bytes, int device) {
    struct Set {
        const void* kernel;
        int device, bytes;
    };
    static std::mutex mu;
    static std::vector<Set> done;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& s : done)
        if (s.kernel == kernel && s.device == device) {
            if (bytes <= s.bytes) return;
            SCMOE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            bytes));
            s.bytes = bytes;
            return;
        }
    SCMOE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.push_back(Set{kernel, device, bytes});
}
}  // namespace scmoe

namespace {

template <typename F>
int guarded(scmoe_ctx* c, F&& f) {
    try {
        f();
        if (c) c->last_error.clear();
        return SCMOE_OK;
    } catch (const ScmoeError& e) {
        if (c) c->last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        if (c) c->last_error = e.what();
        return SCMOE_ERR_INTERNAL;
    }
}

// Host-tier staging buffers (distinct from the kernel workspace), owned by the
// context so that destroying it never depends on thread/static teardown order.
using Stage = HostStage;
Stage& stage_of(scmoe_ctx* c) { return c->stage; }

template <typename T>
T* upload(scmoe_ctx* c, DevBuf& b, const T* host, size_t n) {
    T* d = b.get<T>(n);
    if (n) SCMOE_CUDA(cudaMemcpyAsync(d, host, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    return d;
}
template <typename T>
void download(scmoe_ctx* c, T* host, const T* dev, size_t n) {
    if (n) SCMOE_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
}

// Blocking fills/copies for state set-up.  They go through the context's
// stream: its streams are non-blocking, so a legacy-stream cudaMemset or a
// pageable cudaMemcpy (which may return before its DMA lands) is NOT ordered
// before the next kernel on them.
void stream_zero(scmoe_ctx* c, void* p, size_t bytes) {
    SCMOE_CUDA(cudaMemsetAsync(p, 0, bytes, c->stream));
    SCMOE_CUDA(cudaStreamSynchronize(c->stream));
}
void stream_copy(scmoe_ctx* c, void* dst, const void* src, size_t bytes) {
    SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    if (bytes) SCMOE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
    SCMOE_CUDA(cudaStreamSynchronize(c->stream));
}

void sync_and_check(scmoe_ctx* c) {
    SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    int st = 0;
    SCMOE_CUDA(cudaMemcpy(&st, c->dev_status, sizeof(int), cudaMemcpyDeviceToHost));
    if (st != DEV_OK) {
        stream_zero(c, c->dev_status, sizeof(int));
        if (st == DEV_ERR_INDEX_RANGE) SCMOE_THROW(SCMOE_ERR_STATE, "moe_forward: expert index out of range");
        if (st == DEV_ERR_COUNTERS)
            SCMOE_THROW(SCMOE_ERR_STATE, "bias_update: counters do not cover top_k slots per token");
        if (st == DEV_ERR_EMPTY) SCMOE_THROW(SCMOE_ERR_STATE, "bias_update: empty batch");
        if (st == DEV_ERR_CAPACITY)
            SCMOE_THROW(SCMOE_ERR_STATE, "ep: receive buffer capacity exceeded (rows dropped)");
        if (st == DEV_ERR_TIMEOUT) SCMOE_THROW(SCMOE_ERR_CUDA, "ep: peer barrier timed out");
        SCMOE_THROW(SCMOE_ERR_INTERNAL, "device reported an unknown error");
    }
}

void validate_router(size_t n_ffn, size_t n_zero, size_t top_k, size_t k_expected, double mu) {
    // RouterState::validate, router.hpp:50-61 (in its order)
    const size_t e = n_ffn + n_zero;
    if (top_k > e) SCMOE_THROW(SCMOE_ERR_CONFIG, "router: top_k exceeds expert count");
    if (k_expected < 1 || k_expected > top_k)
        SCMOE_THROW(SCMOE_ERR_CONFIG, "router: need 1 <= k_expected <= top_k");
    if (n_zero > 0 && k_expected >= top_k)
        SCMOE_THROW(SCMOE_ERR_CONFIG, "router: k_expected must be < top_k when zero experts exist");
    if (n_zero < top_k - k_expected)
        SCMOE_THROW(SCMOE_ERR_CONFIG, "router: too few zero experts to absorb top_k - k_expected slack");
    if (mu < 0.0) SCMOE_THROW(SCMOE_ERR_CONFIG, "router: mu must be >= 0");
}

void require_ctx(scmoe_ctx* c) {
    if (!c) throw ScmoeError{SCMOE_ERR_PARAMETER, "null context"};
    SCMOE_CUDA(cudaSetDevice(c->device));
}

int tile_rows_for(const scmoe_ctx* c, const scmoe_bank* b, size_t T, size_t K) {
    // single-GPU bf16 path: 192-token tiles (or SCMOE_TILE_ROWS=128 / 256)
    static const int v = [] {
        const char* e = getenv("SCMOE_TILE_ROWS");
        const int x = e ? atoi(e) : 192;
        return x == 128 || x == 256 ? x : 192;
    }();
    if (b->precision == SCMOE_PREC_BF16) return v;
    // exact fp32: 64-row tiles when they give every SM >= 4 CTAs, else 16-row
    // tiles so a small batch (config A: ~85 rows per expert) spreads over the
    // SMs instead of running 48 long CTAs (the chains, hence the bits, do not
    // depend on the tiling)
    return seq_gemm_tile_rows(T * K, b->inter, c->num_sms);
}

// The MoE block is split into a front half (permutation, and the row gather
// of the bf16 operand) and a back half (expert GEMMs, combine) so a pipelined
// caller can run the front of batch i+1 beside the back of batch i.  The
// permutation result travels between the halves inside the workspace.
void moe_front(scmoe_ctx* c, scmoe_bank* b, const float* x, const __nv_bfloat16* x_bf16,
               size_t T, const uint32_t* idx, size_t K, size_t n_zero) {
    const size_t n_ffn = b->n, d = b->d, E = n_ffn + n_zero;
    SCMOE_CHECK_ARG(K >= 1 && K <= 64, SCMOE_ERR_CONFIG, "moe_forward: top_k must be in [1, 64]");
    Workspace& ws = c->ws;
    PermResult pr;
    {
        ProfScope _p(c, "permute");
        pr = launch_permute(c, idx, T, K, n_ffn, E, tile_rows_for(c, b, T, K));
    }
    static_assert(sizeof(PermResult) <= sizeof(ws.pr_blob), "perm blob");
    memcpy(ws.pr_blob, &pr, sizeof(pr));
    if (b->precision == SCMOE_PREC_BF16) {
        __nv_bfloat16* xb = const_cast<__nv_bfloat16*>(x_bf16);
        if (!xb) {
            // Caller passed fp32 only: make the bf16 GEMM operand copy once.
            xb = ws.hmoe_bf16.get<__nv_bfloat16>(T * d);
            launch_cast_bf16(c, x, T * d, xb);
        }
        if (!c->gemm1_gather) {
            __nv_bfloat16* xp = ws.xp.get<__nv_bfloat16>(T * K * d + 1);
            ProfScope _p(c, "gather");
            launch_gather_bf16(c, xb, d, pr.row_token, pr.expert_base, n_ffn, T * K, xp);
        }
    }
}

// phase: 0 = expert FFN + combine, 1 = expert FFN only, 2 = combine only
// (the full layer runs the FFN before its residual a3 exists).
void moe_back(scmoe_ctx* c, scmoe_bank* b, const float* x, size_t T, const uint32_t* idx,
              const double* gates, size_t K, int renorm, const float* residual, float* out,
              int phase = 0) {
    const size_t n_ffn = b->n, d = b->d, I = b->inter;
    Workspace& ws = c->ws;
    PermResult pr;
    memcpy(&pr, ws.pr_blob, sizeof(pr));
    const float gf = (float)b->gamma_ffn(), gz = (float)b->gamma_zero();
    const bool ffn = phase != 2, comb = phase != 1;
    if (b->precision == SCMOE_PREC_F32_EXACT) {
        float* h = ws.h.get<float>(T * K * I + 1);
        float* y = ws.y.get<float>(T * K * d + 1);
        if (ffn) {
            {
                ProfScope _p(c, "expert_gemm1_f32");
                launch_seq_gemm(c, x, d, pr.row_token, b->w_in32, I, d * I, h, I, d, I, /*silu=*/1,
                                pr.tiles, pr.n_tiles, pr.max_tiles, tile_rows_for(c, b, T, K));
            }
            ProfScope _p(c, "expert_gemm2_f32");
            launch_seq_gemm(c, h, I, nullptr, b->w_out32, d, I * d, y, d, I, d, /*silu=*/0,
                            pr.tiles, pr.n_tiles, pr.max_tiles, tile_rows_for(c, b, T, K));
        }
        if (comb) {
            ProfScope _p(c, "combine");
            launch_combine_f32(c, x, y, idx, gates, pr.slot_pos, T, d, K, n_ffn, gf, gz, renorm,
                               residual, out);
        }
    } else {
        __nv_bfloat16* h = ws.h.get<__nv_bfloat16>(T * K * I + 1);
        __nv_bfloat16* y = ws.y.get<__nv_bfloat16>(T * K * d + 1);
        if (ffn) {
            if (c->gemm1_gather) {
                // GEMM1 gathers its token rows straight from x (cp.async row gather).
                ProfScope _p(c, "gemm1_tcgen05");
                launch_grouped_gemm_bf16(c, b->w1t, n_ffn, I, d,
                                         ws.hmoe_bf16.get<__nv_bfloat16>(T * d), T, pr.row_token,
                                         h, /*silu=*/1, pr.tiles, pr.n_tiles, pr.max_tiles,
                                         tile_rows_for(c, b, T, K));
            } else {
                ProfScope _p(c, "gemm1_tcgen05");
                launch_grouped_gemm_bf16(c, b->w1t, n_ffn, I, d,
                                         ws.xp.get<__nv_bfloat16>(T * K * d + 1), T * K, nullptr,
                                         h, /*silu=*/1, pr.tiles, pr.n_tiles, pr.max_tiles,
                                         tile_rows_for(c, b, T, K));
            }
            ProfScope _p(c, "gemm2_tcgen05");
            launch_grouped_gemm_bf16(c, b->w2t, n_ffn, d, I, h, T * K, nullptr, y, /*silu=*/0,
                                     pr.tiles, pr.n_tiles, pr.max_tiles, tile_rows_for(c, b, T, K));
        }
        if (comb) {
            ProfScope _p(c, "combine");
            launch_combine_bf16(c, x, y, idx, gates, pr.slot_pos, T, d, K, n_ffn, gf, gz, renorm,
                                residual, out);
        }
    }
}

// moe_forward on device pointers; x is the MoE input (hmoe), used by the
// expert FFN and by the zero-expert identity term.
void moe_forward_dev(scmoe_ctx* c, scmoe_bank* b, const float* x, const __nv_bfloat16* x_bf16,
                     size_t T, const uint32_t* idx, const double* gates, size_t K, size_t n_zero,
                     int renorm, const float* residual, float* out) {
    moe_front(c, b, x, x_bf16, T, idx, K, n_zero);
    moe_back(c, b, x, T, idx, gates, K, renorm, residual, out);
}

// router.hpp:136 logits = mm(x, W_r).  Kernel choice: the full-width slab
// kernel (1 CTA/SM, single wave) when the batch fills the GPU; the lean
// kernel inside pipelined calls (it co-resides with the grouped GEMM); one
// thread per logit for small batches (config A); the 64/16-row tiled kernel
// otherwise (E > 768).
void route_logits(scmoe_ctx* c, scmoe_router* r, const float* x, size_t T, float* logits) {
    const size_t E = r->E();
    int v = c->router_variant;
    if (v == 2 && !router_lean_ok(r->d, E)) v = 0;
    if (v == 1 && !router_slab_ok(T, r->d, E, 0)) v = 0;
    if (v == 4 && !router_tma_ok(T, r->d, E, 0)) v = 0;
    if (v == 5 && !router_corun_ok(T, r->d, E)) v = 0;
    if (v == 6 && !router_small_ok(0, r->d, E, c->num_sms)) v = 0;
    if (v == 0) {
        if (c->overlapped && router_corun_ok(T, r->d, E) && T >= 512)
            v = 5;
        else if (router_tma_ok(T, r->d, E, c->num_sms))
            v = 4;
        else if (router_small_ok(T, r->d, E, c->num_sms))
            v = 6;
        else
            v = 3;
    }
    ProfScope _p(c, "router_gemm");
    if (v == 5) {
        launch_router_corun(c, x, r->w, logits, T, r->d, E);
    } else if (v == 4) {
        launch_router_tma(c, x, r->w, logits, T, r->d, E);
    } else if (v == 1) {
        launch_router_slab(c, x, r->w, logits, T, r->d, E);
    } else if (v == 2) {
        launch_router_lean(c, x, r->w, logits, T, r->d, E);
    } else if (v == 6) {
        launch_router_small(c, x, r->w, logits, T, r->d, E);
    } else {
        const int tr = seq_gemm_tile_rows(T, E, c->num_sms);
        const size_t ntile = ceil_div(T, tr);
        TokenTile* td = c->ws.tiles_router.get<TokenTile>(ntile);
        launch_row_tiles(c, T, tr, td);
        launch_seq_gemm(c, x, r->d, nullptr, r->w, E, 0, logits, E, r->d, E, 0, td, nullptr, ntile,
                        tr);
    }
}

// Front half of the ScMoE MoE branch (model.hpp:394-397): rmsnorm, router,
// softmax + top-K, permutation (+ gather).
void layer_front(scmoe_ctx* c, scmoe_router* r, scmoe_bank* b, const float* a1, const float* gain,
                 size_t T, uint32_t* idx, double* gates, uint32_t* ffn_count) {
    const size_t d = r->d, E = r->E(), K = r->top_k;
    Workspace& ws = c->ws;
    float* hmoe = ws.hmoe.get<float>(T * d);
    __nv_bfloat16* hb =
        b->precision == SCMOE_PREC_BF16 ? ws.hmoe_bf16.get<__nv_bfloat16>(T * d) : nullptr;
    if (c->router_variant == 0 && !c->overlapped && front_small_ok(T, d, E, K, c->num_sms)) {
        // small batches: rmsnorm + router + softmax / top-K in one launch
        ProfScope _p(c, "front_small");
        launch_front_small(c, a1, gain, T, d, 1e-6f, r->w, E, K, r->n_ffn, r->b, hmoe, hb, idx,
                           gates, ffn_count);
    } else {
        {
            ProfScope _p(c, "rmsnorm");
            launch_rmsnorm(c, a1, gain, T, d, 1e-6f, hmoe, hb);
        }
        float* logits = ws.logits.get<float>(T * E);
        route_logits(c, r, hmoe, T, logits);
        {
            ProfScope _p(c, "softmax_topk");
            launch_softmax_topk(c, logits, T, E, K, r->n_ffn, r->b, idx, gates, ffn_count,
                                nullptr);
        }
    }
    moe_front(c, b, hmoe, hb, T, idx, K, r->n_zero);
}

void check_layer_args(scmoe_router* r, scmoe_bank* b) {
    if (r->d != b->d) SCMOE_THROW(SCMOE_ERR_DIMENSION, "layer: router/bank width mismatch");
    if (r->n_ffn != b->n)
        SCMOE_THROW(SCMOE_ERR_DIMENSION, "moe_block: decision/bank FFN count mismatch");
    validate_router(r->n_ffn, r->n_zero, r->top_k, r->k_expected, r->mu);
}

}  // namespace

extern "C" {

const char* scmoe_version(void) { return "scmoe-b200 0.1 (sm_100a)"; }

int scmoe_ctx_create(int device, scmoe_ctx** out) {
    return guarded(nullptr, [&] {
        if (!out) SCMOE_THROW(SCMOE_ERR_PARAMETER, "null out");
        int n = 0;
        SCMOE_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) SCMOE_THROW(SCMOE_ERR_CUDA, "no such CUDA device");
        SCMOE_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        SCMOE_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            SCMOE_THROW(SCMOE_ERR_CUDA, "libscmoe is built for sm_100a (B200); device is sm_" +
                                            std::to_string(prop.major * 10 + prop.minor));
        auto* c = new scmoe_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        if (const char* g = getenv("SCMOE_GEMM1_GATHER")) c->gemm1_gather = atoi(g) != 0;
        if (const char* g = getenv("SCMOE_ROUTER_SMS")) c->router_sms = atoi(g);
        if (const char* g = getenv("SCMOE_GEMM_SMS")) c->gemm_sms = atoi(g);
        if (const char* v = getenv("SCMOE_ROUTER")) {
            const std::string sv(v);
            c->router_variant =
                sv == "slab"    ? 1
                : sv == "lean"  ? 2
                : sv == "tiled" ? 3
                : sv == "tma"   ? 4
                : sv == "corun" ? 5
                : sv == "small" ? 6
                                : 0;
        }
        SCMOE_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        SCMOE_CUDA(cudaMalloc(&c->dev_status, sizeof(int)));
        stream_zero(c, c->dev_status, sizeof(int));
        *out = c;
    });
}

int scmoe_ctx_destroy(scmoe_ctx* c) {
    if (!c) return SCMOE_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->ws.release_all();
    c->ws_alt.release_all();
    if (c->s_front) {
        cudaStreamDestroy(c->s_front);
        cudaStreamDestroy(c->s_back);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(c->ev_front[i]);
            cudaEventDestroy(c->ev_back[i]);
        }
        cudaEventDestroy(c->ev_join);
    }
    if (c->s_moe) {
        cudaStreamSynchronize(c->s_moe);
        cudaStreamDestroy(c->s_moe);
        for (auto& e : c->ev_full) cudaEventDestroy(e);
    }
    if (c->s_h2d) {
        cudaStreamSynchronize(c->s_d2h);
        cudaStreamDestroy(c->s_h2d);
        cudaStreamDestroy(c->s_d2h);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(c->ev_in[i]);
            cudaEventDestroy(c->ev_in_a1[i]);
            cudaEventDestroy(c->ev_done[i]);
            cudaEventDestroy(c->ev_out[i]);
        }
    }
    for (auto& slot : c->io)
        for (auto& b : slot) b.release();
    for (auto& rec : c->prof.recs) {
        cudaEventDestroy(rec.a);
        cudaEventDestroy(rec.b);
    }
    Stage& st = stage_of(c);
    for (auto& b : st.bufs) b.release();
    if (c->dev_status) cudaFree(c->dev_status);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return SCMOE_OK;
}

const char* scmoe_last_error(const scmoe_ctx* c) { return c ? c->last_error.c_str() : "null context"; }

int scmoe_set_stream(scmoe_ctx* c, void* s) {
    return guarded(c, [&] {
        require_ctx(c);
        c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    });
}
void* scmoe_get_stream(const scmoe_ctx* c) { return c ? (void*)c->stream : nullptr; }

int scmoe_ctx_set_overlapped(scmoe_ctx* c, int on) {
    return guarded(c, [&] {
        require_ctx(c);
        c->overlapped = on != 0;
    });
}

int scmoe_ctx_set_sm_budget(scmoe_ctx* c, int router_sms, int gemm_sms) {
    return guarded(c, [&] {
        require_ctx(c);
        if (router_sms < 0 || gemm_sms < 0)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "sm budget must be >= 0");
        c->router_sms = router_sms;
        c->gemm_sms = gemm_sms;
    });
}

int scmoe_synchronize(scmoe_ctx* c) {
    return guarded(c, [&] {
        require_ctx(c);
        sync_and_check(c);
    });
}
uint64_t scmoe_kernel_launches(const scmoe_ctx* c) { return c ? c->launches : 0; }

int scmoe_device_alloc(scmoe_ctx* c, size_t bytes, void** out) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaMalloc(out, bytes ? bytes : 16));
    });
}
int scmoe_device_free(scmoe_ctx* c, void* p) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaFree(p));
    });
}
int scmoe_copy_h2d(scmoe_ctx* c, void* dst, const void* src, size_t bytes) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    });
}
int scmoe_copy_d2h(scmoe_ctx* c, void* dst, const void* src, size_t bytes) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// ---- router ---------------------------------------------------------------

int scmoe_router_create(scmoe_ctx* c, size_t d, size_t n_ffn, size_t n_zero, size_t top_k,
                        size_t k_expected, double mu, double mu_decay, scmoe_router** out) {
    return guarded(c, [&] {
        require_ctx(c);
        validate_router(n_ffn, n_zero, top_k, k_expected, mu);
        auto* r = new scmoe_router();
        r->d = d;
        r->n_ffn = n_ffn;
        r->n_zero = n_zero;
        r->top_k = top_k;
        r->k_expected = k_expected;
        r->mu = mu;
        r->mu_decay = mu_decay;
        const size_t E = r->E();
        SCMOE_CUDA(cudaMalloc(&r->w, std::max<size_t>(d * E, 1) * sizeof(float)));
        SCMOE_CUDA(cudaMalloc(&r->b, std::max<size_t>(E, 1) * sizeof(double)));
        SCMOE_CUDA(cudaMalloc(&r->routed, std::max<size_t>(E, 1) * sizeof(uint64_t)));
        stream_zero(c, r->w, std::max<size_t>(d * E, 1) * sizeof(float));
        stream_zero(c, r->b, std::max<size_t>(E, 1) * sizeof(double));
        stream_zero(c, r->routed, std::max<size_t>(E, 1) * sizeof(uint64_t));
        *out = r;
    });
}

int scmoe_router_destroy(scmoe_ctx* c, scmoe_router* r) {
    if (!r) return SCMOE_OK;
    if (c) cudaSetDevice(c->device);
    cudaFree(r->w);
    cudaFree(r->b);
    cudaFree(r->routed);
    delete r;
    return SCMOE_OK;
}

int scmoe_router_set_weights_host(scmoe_ctx* c, scmoe_router* r, const float* w) {
    return guarded(c, [&] {
        require_ctx(c);
        stream_copy(c, r->w, w, r->d * r->E() * sizeof(float));
    });
}
int scmoe_router_set_weights(scmoe_ctx* c, scmoe_router* r, const float* w) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaMemcpyAsync(r->w, w, r->d * r->E() * sizeof(float), cudaMemcpyDeviceToDevice,
                                   c->stream));
    });
}
int scmoe_router_set_bias_host(scmoe_ctx* c, scmoe_router* r, const double* b) {
    return guarded(c, [&] {
        require_ctx(c);
        for (size_t i = r->n_ffn; i < r->E(); ++i)
            if (b[i] != 0.0) SCMOE_THROW(SCMOE_ERR_CONFIG, "router: zero-expert bias must stay 0");
        stream_copy(c, r->b, b, r->E() * sizeof(double));
    });
}
int scmoe_router_get_bias_host(scmoe_ctx* c, scmoe_router* r, double* b) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        SCMOE_CUDA(cudaMemcpy(b, r->b, r->E() * sizeof(double), cudaMemcpyDeviceToHost));
    });
}
int scmoe_router_set_mu(scmoe_ctx* c, scmoe_router* r, double mu, double mu_decay) {
    return guarded(c, [&] {
        if (mu < 0.0) SCMOE_THROW(SCMOE_ERR_CONFIG, "router: mu must be >= 0");
        r->mu = mu;
        r->mu_decay = mu_decay;
    });
}
int scmoe_router_get_mu(scmoe_ctx* c, scmoe_router* r, double* mu, double* mu_decay) {
    return guarded(c, [&] {
        if (mu) *mu = r->mu;
        if (mu_decay) *mu_decay = r->mu_decay;
    });
}
int scmoe_router_get_counters_host(scmoe_ctx* c, scmoe_router* r, uint64_t* routed,
                                   uint64_t* seen) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        if (routed)
            SCMOE_CUDA(cudaMemcpy(routed, r->routed, r->E() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        if (seen) *seen = r->tokens_seen;
    });
}
int scmoe_router_set_counters_host(scmoe_ctx* c, scmoe_router* r, const uint64_t* routed,
                                   uint64_t seen) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        stream_copy(c, r->routed, routed, r->E() * sizeof(uint64_t));
        r->tokens_seen = seen;
    });
}
uint64_t* scmoe_router_counters_dev(scmoe_router* r) { return r ? r->routed : nullptr; }
const double* scmoe_router_bias_dev(scmoe_router* r) { return r ? r->b : nullptr; }

int scmoe_route_topk(scmoe_ctx* c, scmoe_router* r, const float* x, size_t T, uint32_t* idx,
                     double* gates, uint32_t* ffn_count, float* probs) {
    return guarded(c, [&] {
        require_ctx(c);
        validate_router(r->n_ffn, r->n_zero, r->top_k, r->k_expected, r->mu);
        if (T == 0) return;
        const size_t E = r->E();
        float* logits = c->ws.logits.get<float>(T * E);
        // router.hpp:136 -- one group, row tiles of 64 tokens
        route_logits(c, r, x, T, logits);
        { ProfScope _p(c, "softmax_topk"); launch_softmax_topk(c, logits, T, E, r->top_k, r->n_ffn, r->b, idx, gates, ffn_count, probs); }
    });
}

int scmoe_route_topk_host(scmoe_ctx* c, scmoe_router* r, const float* x, size_t T, uint32_t* idx,
                          double* gates, uint32_t* ffn_count, float* probs) {
    return guarded(c, [&] {
        require_ctx(c);
        Stage& s = stage_of(c);
        const size_t K = r->top_k, E = r->E();
        const float* xd = upload(c, s.bufs[0], x, T * r->d);
        uint32_t* di = s.bufs[1].get<uint32_t>(T * K);
        double* dg = s.bufs[2].get<double>(T * K);
        uint32_t* dc = s.bufs[3].get<uint32_t>(T);
        float* dp = probs ? s.bufs[4].get<float>(T * E) : nullptr;
        int rc = scmoe_route_topk(c, r, xd, T, di, dg, dc, dp);
        if (rc) throw ScmoeError{rc, c->last_error};
        download(c, idx, di, T * K);
        download(c, gates, dg, T * K);
        download(c, ffn_count, dc, T);
        if (probs) download(c, probs, dp, T * E);
        sync_and_check(c);
    });
}

#define ROUTE_FROM_PROBS(S, SUF)                                                                   \
    int scmoe_route_from_probs_##SUF(scmoe_ctx* c, scmoe_router* r, const S* probs, size_t T,      \
                                     uint32_t* idx, double* gates, uint32_t* ffn_count) {          \
        return guarded(c, [&] {                                                                    \
            require_ctx(c);                                                                        \
            validate_router(r->n_ffn, r->n_zero, r->top_k, r->k_expected, r->mu);                  \
            launch_topk_from_probs_##SUF(c, probs, T, r->E(), r->top_k, r->n_ffn, r->b, idx,       \
                                         gates, ffn_count);                                        \
        });                                                                                        \
    }                                                                                              \
    int scmoe_route_from_probs_##SUF##_host(scmoe_ctx* c, scmoe_router* r, const S* probs,         \
                                            size_t T, uint32_t* idx, double* gates,                \
                                            uint32_t* ffn_count) {                                 \
        return guarded(c, [&] {                                                                    \
            require_ctx(c);                                                                        \
            Stage& s = stage_of(c);                                                                \
            const size_t K = r->top_k;                                                             \
            const S* pd = upload(c, s.bufs[0], probs, T * r->E());                                 \
            uint32_t* di = s.bufs[1].get<uint32_t>(T * K);                                         \
            double* dg = s.bufs[2].get<double>(T * K);                                             \
            uint32_t* dc = s.bufs[3].get<uint32_t>(T);                                             \
            int rc = scmoe_route_from_probs_##SUF(c, r, pd, T, di, dg, dc);                        \
            if (rc) throw ScmoeError{rc, c->last_error};                                           \
            download(c, idx, di, T * K);                                                           \
            download(c, gates, dg, T * K);                                                         \
            download(c, ffn_count, dc, T);                                                         \
            sync_and_check(c);                                                                     \
        });                                                                                        \
    }
ROUTE_FROM_PROBS(float, f32)
ROUTE_FROM_PROBS(double, f64)

int scmoe_routing_stats(scmoe_ctx* c, const uint32_t* idx, const uint32_t* cnt, size_t T,
                        size_t K, size_t n_ffn, size_t n_zero, size_t k_expected,
                        size_t lb_groups, double* mean_ffn, double* std_ffn, double* load,
                        double* lb) {
    return guarded(c, [&] {
        require_ctx(c);
        if (lb && (lb_groups == 0 || n_ffn % lb_groups != 0))
            SCMOE_THROW(SCMOE_ERR_CONFIG, "lb_loss: group count must divide FFN expert count");
        const size_t E = n_ffn + n_zero;
        uint64_t* hist = c->ws.misc.get<uint64_t>(E + 2);
        double* mom = reinterpret_cast<double*>(hist + E);
        SCMOE_CUDA(cudaMemsetAsync(hist, 0, E * sizeof(uint64_t), c->stream));
        launch_accumulate(c, idx, T * K, E, hist);
        launch_ffn_moments(c, cnt, T, mom);
        std::vector<uint64_t> h(E + 2);
        SCMOE_CUDA(cudaMemcpyAsync(h.data(), hist, (E + 2) * sizeof(uint64_t),
                                   cudaMemcpyDeviceToHost, c->stream));
        sync_and_check(c);  // StateError on an index >= E
        memcpy(mean_ffn, &h[E], sizeof(double));
        memcpy(std_ffn, &h[E + 1], sizeof(double));
        // the reference accumulates 1.0 per slot (exact integers) then divides
        const double slots = (double)(T * K), tc = (double)T;
        if (load)
            for (size_t e = 0; e < E; ++e) load[e] = (double)h[e] / slots;
        if (lb) {
            const size_t gsz = n_ffn / lb_groups;
            for (size_t j = 0; j < lb_groups; ++j) {
                uint64_t f = 0;
                for (size_t e = j * gsz; e < (j + 1) * gsz; ++e) f += h[e];
                lb[j] = (double)f * ((double)lb_groups / ((double)k_expected * tc));
            }
            if (n_zero > 0) {
                uint64_t f = 0;
                for (size_t e = n_ffn; e < E; ++e) f += h[e];
                lb[lb_groups] = (double)f / ((double)(K - k_expected) * tc);
            }
        }
    });
}
int scmoe_routing_stats_host(scmoe_ctx* c, const uint32_t* idx, const uint32_t* cnt, size_t T,
                             size_t K, size_t n_ffn, size_t n_zero, size_t k_expected,
                             size_t lb_groups, double* mean_ffn, double* std_ffn, double* load,
                             double* lb) {
    return guarded(c, [&] {
        require_ctx(c);
        Stage& s = stage_of(c);
        const uint32_t* di = upload(c, s.bufs[1], idx, T * K);
        const uint32_t* dc = upload(c, s.bufs[3], cnt, T);
        int rc = scmoe_routing_stats(c, di, dc, T, K, n_ffn, n_zero, k_expected, lb_groups,
                                     mean_ffn, std_ffn, load, lb);
        if (rc) throw ScmoeError{rc, c->last_error};
    });
}

int scmoe_route_topk_f64(scmoe_ctx* c, scmoe_router* r, const double* x, size_t T,
                         const double* w, uint32_t* idx, double* gates, uint32_t* ffn_count,
                         double* probs) {
    return guarded(c, [&] {
        require_ctx(c);
        validate_router(r->n_ffn, r->n_zero, r->top_k, r->k_expected, r->mu);
        if (T == 0) return;
        const size_t E = r->E();
        double* logits = c->ws.logits.get<double>(T * E);
        {
            ProfScope _p(c, "router_gemm_f64");
            launch_router_f64(c, x, w, logits, T, r->d, E);
        }
        ProfScope _p(c, "softmax_topk_f64");
        launch_softmax_topk_f64(c, logits, T, E, r->top_k, r->n_ffn, r->b, idx, gates, ffn_count,
                                probs);
    });
}

int scmoe_route_topk_f64_host(scmoe_ctx* c, scmoe_router* r, const double* x, size_t T,
                              const double* w, uint32_t* idx, double* gates, uint32_t* ffn_count,
                              double* probs) {
    return guarded(c, [&] {
        require_ctx(c);
        Stage& s = stage_of(c);
        const size_t K = r->top_k, E = r->E();
        const double* xd = upload(c, s.bufs[0], x, T * r->d);
        const double* wd = upload(c, s.bufs[7], w, r->d * E);
        uint32_t* di = s.bufs[1].get<uint32_t>(T * K);
        double* dg = s.bufs[2].get<double>(T * K);
        uint32_t* dc = s.bufs[3].get<uint32_t>(T);
        double* dp = probs ? s.bufs[4].get<double>(T * E) : nullptr;
        int rc = scmoe_route_topk_f64(c, r, xd, T, wd, di, dg, dc, dp);
        if (rc) throw ScmoeError{rc, c->last_error};
        download(c, idx, di, T * K);
        download(c, gates, dg, T * K);
        download(c, ffn_count, dc, T);
        if (probs) download(c, probs, dp, T * E);
        sync_and_check(c);
    });
}

int scmoe_debug_exp(scmoe_ctx* c, const double* in, double* out, size_t n) {
    return guarded(c, [&] {
        require_ctx(c);
        launch_debug_exp(c, in, out, n);
    });
}

int scmoe_accumulate_counters(scmoe_ctx* c, scmoe_router* r, const uint32_t* idx, size_t T) {
    return guarded(c, [&] {
        require_ctx(c);
        launch_accumulate(c, idx, T * r->top_k, r->E(), r->routed);
        r->tokens_seen += T;
    });
}
int scmoe_accumulate_counters_host(scmoe_ctx* c, scmoe_router* r, const uint32_t* idx, size_t T) {
    return guarded(c, [&] {
        require_ctx(c);
        Stage& s = stage_of(c);
        const uint32_t* di = upload(c, s.bufs[1], idx, T * r->top_k);
        int rc = scmoe_accumulate_counters(c, r, di, T);
        if (rc) throw ScmoeError{rc, c->last_error};
        sync_and_check(c);
    });
}

int scmoe_bias_update(scmoe_ctx* c, scmoe_router* r, double* delta) {
    return guarded(c, [&] {
        require_ctx(c);
        if (r->tokens_seen == 0) SCMOE_THROW(SCMOE_ERR_STATE, "bias_update: empty batch");
        double* dd = c->ws.misc.get<double>(r->E());
        launch_bias_update(c, r, dd);
        sync_and_check(c);  // StateError on counter mismatch (router.hpp:161-162)
        if (delta) SCMOE_CUDA(cudaMemcpy(delta, dd, r->E() * sizeof(double), cudaMemcpyDeviceToHost));
        r->mu *= r->mu_decay;  // router.hpp:172
        r->tokens_seen = 0;
    });
}

// ---- bank -----------------------------------------------------------------

int scmoe_bank_create(scmoe_ctx* c, size_t n, size_t d, size_t inter, int precision, size_t m,
                      int gamma_mode, scmoe_bank** out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (m < 1) SCMOE_THROW(SCMOE_ERR_PARAMETER, "variance_gamma: m must be >= 1");
        if (precision != SCMOE_PREC_F32_EXACT && precision != SCMOE_PREC_BF16 &&
            precision != SCMOE_PREC_F64_EXACT)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "bank: unknown precision");
        if (gamma_mode < 0 || gamma_mode > 2) SCMOE_THROW(SCMOE_ERR_PARAMETER, "unknown gamma mode");
        if (precision == SCMOE_PREC_BF16) {
            // both GEMMs tile the weight rows by 256 (two 128-row MMA slabs)
            if (d % 256 != 0 || inter % 256 != 0)
                SCMOE_THROW(SCMOE_ERR_DIMENSION,
                            "bank: bf16 tensor-core path needs d % 256 == 0 and inter % 256 == 0");
        }
        auto* b = new scmoe_bank();
        b->n = n;
        b->d = d;
        b->inter = inter;
        b->m = m;
        b->precision = precision;
        b->gamma_mode = gamma_mode;
        const size_t per = d * inter;
        if (precision == SCMOE_PREC_F32_EXACT) {
            SCMOE_CUDA(cudaMalloc(&b->w_in32, std::max<size_t>(n * per, 1) * sizeof(float)));
            SCMOE_CUDA(cudaMalloc(&b->w_out32, std::max<size_t>(n * per, 1) * sizeof(float)));
            stream_zero(c, b->w_in32, std::max<size_t>(n * per, 1) * sizeof(float));
            stream_zero(c, b->w_out32, std::max<size_t>(n * per, 1) * sizeof(float));
        } else if (precision == SCMOE_PREC_F64_EXACT) {
            SCMOE_CUDA(cudaMalloc(&b->w_in64, std::max<size_t>(n * per, 1) * sizeof(double)));
            SCMOE_CUDA(cudaMalloc(&b->w_out64, std::max<size_t>(n * per, 1) * sizeof(double)));
            stream_zero(c, b->w_in64, std::max<size_t>(n * per, 1) * sizeof(double));
            stream_zero(c, b->w_out64, std::max<size_t>(n * per, 1) * sizeof(double));
        } else {
            SCMOE_CUDA(cudaMalloc(&b->w1t, std::max<size_t>(n * per, 1) * sizeof(__nv_bfloat16)));
            SCMOE_CUDA(cudaMalloc(&b->w2t, std::max<size_t>(n * per, 1) * sizeof(__nv_bfloat16)));
            stream_zero(c, b->w1t, std::max<size_t>(n * per, 1) * sizeof(__nv_bfloat16));
            stream_zero(c, b->w2t, std::max<size_t>(n * per, 1) * sizeof(__nv_bfloat16));
        }
        *out = b;
    });
}

int scmoe_bank_destroy(scmoe_ctx* c, scmoe_bank* b) {
    if (!b) return SCMOE_OK;
    if (c) cudaSetDevice(c->device);
    cudaFree(b->w_in32);
    cudaFree(b->w_out32);
    cudaFree(b->w1t);
    cudaFree(b->w2t);
    cudaFree(b->w_in64);
    cudaFree(b->w_out64);
    delete b;
    return SCMOE_OK;
}

int scmoe_bank_set_expert(scmoe_ctx* c, scmoe_bank* b, size_t e, const float* w_in,
                          const float* w_out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (e >= b->n) SCMOE_THROW(SCMOE_ERR_DIMENSION, "bank: expert index out of range");
        if (b->precision == SCMOE_PREC_F64_EXACT)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "bank: an fp64 bank takes scmoe_bank_set_expert_f64");
        const size_t per = b->d * b->inter;
        if (b->precision == SCMOE_PREC_F32_EXACT) {
            SCMOE_CUDA(cudaMemcpyAsync(b->w_in32 + e * per, w_in, per * sizeof(float),
                                       cudaMemcpyDeviceToDevice, c->stream));
            SCMOE_CUDA(cudaMemcpyAsync(b->w_out32 + e * per, w_out, per * sizeof(float),
                                       cudaMemcpyDeviceToDevice, c->stream));
        } else {
            // w_in [d, I] -> w1t [I, d];  w_out [I, d] -> w2t [d, I]
            launch_f32_to_bf16_t(c, w_in, b->d, b->inter, b->w1t + e * per);
            launch_f32_to_bf16_t(c, w_out, b->inter, b->d, b->w2t + e * per);
        }
    });
}

int scmoe_bank_set_expert_host(scmoe_ctx* c, scmoe_bank* b, size_t e, const float* w_in,
                               const float* w_out) {
    return guarded(c, [&] {
        require_ctx(c);
        Stage& s = stage_of(c);
        const size_t per = b->d * b->inter;
        const float* di = upload(c, s.bufs[8], w_in, per);
        const float* dout = upload(c, s.bufs[9], w_out, per);
        int rc = scmoe_bank_set_expert(c, b, e, di, dout);
        if (rc) throw ScmoeError{rc, c->last_error};
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int scmoe_bank_init_uniform(scmoe_ctx* c, scmoe_bank* b, uint64_t seed, uint64_t stream0,
                            double variance) {
    return guarded(c, [&] {
        require_ctx(c);
        if (variance < 0.0) SCMOE_THROW(SCMOE_ERR_PARAMETER, "seeded_init: variance must be >= 0");
        const double hw = std::sqrt(3.0 * variance);
        const size_t per = b->d * b->inter;
        for (size_t e = 0; e < b->n; ++e) {
            const uint64_t s_in = scmoe_rng_stream_seed(seed, stream0 + 2 * e);
            const uint64_t s_out = scmoe_rng_stream_seed(seed, stream0 + 2 * e + 1);
            if (b->precision == SCMOE_PREC_F32_EXACT) {
                launch_uniform_init(c, s_in, 0, per, hw, b->w_in32 + e * per);
                launch_uniform_init(c, s_out, 0, per, hw, b->w_out32 + e * per);
            } else {
                launch_uniform_init_bf16_t(c, s_in, b->d, b->inter, hw, b->w1t + e * per);
                launch_uniform_init_bf16_t(c, s_out, b->inter, b->d, hw, b->w2t + e * per);
            }
        }
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    });
}

double scmoe_bank_gamma_ffn(const scmoe_bank* b) { return b ? b->gamma_ffn() : 0.0; }
double scmoe_bank_gamma_zero(const scmoe_bank* b) { return b ? b->gamma_zero() : 0.0; }
size_t scmoe_bank_device_bytes(const scmoe_bank* b) {
    if (!b) return 0;
    const size_t per = b->d * b->inter * b->n * 2;
    return b->precision == SCMOE_PREC_F64_EXACT ? per * 8
           : b->precision == SCMOE_PREC_F32_EXACT ? per * 4
                                                   : per * 2;
}

// ---- MoE forward / layer ---------------------------------------------------

int scmoe_moe_forward(scmoe_ctx* c, scmoe_bank* b, const float* x, size_t T, const uint32_t* idx,
                      const double* gates, size_t K, size_t n_zero, int renorm,
                      const float* residual, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (T == 0) return;
        launch_check_indices(c, idx, T * K, b->n + n_zero);
        moe_forward_dev(c, b, x, nullptr, T, idx, gates, K, n_zero, renorm, residual, out);
    });
}

int scmoe_moe_forward_host(scmoe_ctx* c, scmoe_bank* b, const float* x, size_t T,
                           const uint32_t* idx, const double* gates, size_t K, size_t n_zero,
                           int renorm, const float* residual, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        // blocks.hpp:375-377 -- index range check before any work
        for (size_t i = 0; i < T * K; ++i)
            if (idx[i] >= b->n + n_zero) SCMOE_THROW(SCMOE_ERR_STATE, "moe_forward: expert index out of range");
        if (T == 0) return;
        Stage& s = stage_of(c);
        const float* xd = upload(c, s.bufs[0], x, T * b->d);
        const uint32_t* di = upload(c, s.bufs[1], idx, T * K);
        const double* dg = upload(c, s.bufs[2], gates, T * K);
        const float* dr = residual ? upload(c, s.bufs[3], residual, T * b->d) : nullptr;
        float* dout = s.bufs[4].get<float>(T * b->d);
        int rc = scmoe_moe_forward(c, b, xd, T, di, dg, K, n_zero, renorm, dr, dout);
        if (rc) throw ScmoeError{rc, c->last_error};
        download(c, out, dout, T * b->d);
        sync_and_check(c);
    });
}

int scmoe_bank_set_expert_f64(scmoe_ctx* c, scmoe_bank* b, size_t e, const double* w_in,
                              const double* w_out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (b->precision != SCMOE_PREC_F64_EXACT)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "bank: scmoe_bank_set_expert_f64 needs an fp64 bank");
        if (e >= b->n) SCMOE_THROW(SCMOE_ERR_DIMENSION, "bank: expert index out of range");
        const size_t per = b->d * b->inter;
        SCMOE_CUDA(cudaMemcpyAsync(b->w_in64 + e * per, w_in, per * sizeof(double),
                                   cudaMemcpyDefault, c->stream));
        SCMOE_CUDA(cudaMemcpyAsync(b->w_out64 + e * per, w_out, per * sizeof(double),
                                   cudaMemcpyDefault, c->stream));
    });
}
int scmoe_bank_set_expert_f64_host(scmoe_ctx* c, scmoe_bank* b, size_t e, const double* w_in,
                                   const double* w_out) {
    return guarded(c, [&] {
        require_ctx(c);
        int rc = scmoe_bank_set_expert_f64(c, b, e, w_in, w_out);
        if (rc) throw ScmoeError{rc, c->last_error};
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int scmoe_moe_forward_f64(scmoe_ctx* c, scmoe_bank* b, const double* x, size_t T,
                          const uint32_t* idx, const double* gates, size_t K, size_t n_zero,
                          int renorm, const double* residual, double* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (b->precision != SCMOE_PREC_F64_EXACT)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "moe_forward_f64: needs an fp64 bank");
        SCMOE_CHECK_ARG(K >= 1 && K <= 64, SCMOE_ERR_CONFIG, "moe_forward: top_k must be in [1, 64]");
        if (T == 0) return;
        const size_t n_ffn = b->n, d = b->d, I = b->inter, E = n_ffn + n_zero;
        launch_check_indices(c, idx, T * K, E);
        PermResult pr;
        {
            ProfScope _p(c, "permute");
            pr = launch_permute(c, idx, T, K, n_ffn, E, 64);
        }
        Workspace& ws = c->ws;
        double* h = ws.h.get<double>(T * K * I + 1);
        double* y = ws.y.get<double>(T * K * d + 1);
        {
            ProfScope _p(c, "expert_gemm1_f64");
            launch_seq_gemm_f64(c, x, d, pr.row_token, b->w_in64, I, d * I, h, I, d, I, 1,
                                pr.tiles, pr.n_tiles, pr.max_tiles);
        }
        {
            ProfScope _p(c, "expert_gemm2_f64");
            launch_seq_gemm_f64(c, h, I, nullptr, b->w_out64, d, I * d, y, d, I, d, 0, pr.tiles,
                                pr.n_tiles, pr.max_tiles);
        }
        ProfScope _p(c, "combine_f64");
        launch_combine_f64(c, x, y, idx, gates, pr.slot_pos, T, d, K, n_ffn, b->gamma_ffn(),
                           b->gamma_zero(), renorm, residual, out);
    });
}
int scmoe_moe_forward_f64_host(scmoe_ctx* c, scmoe_bank* b, const double* x, size_t T,
                               const uint32_t* idx, const double* gates, size_t K, size_t n_zero,
                               int renorm, const double* residual, double* out) {
    return guarded(c, [&] {
        require_ctx(c);
        // blocks.hpp:375-377 -- index range check before any work
        for (size_t i = 0; i < T * K; ++i)
            if (idx[i] >= b->n + n_zero) SCMOE_THROW(SCMOE_ERR_STATE, "moe_forward: expert index out of range");
        if (T == 0) return;
        Stage& s = stage_of(c);
        const double* xd = upload(c, s.bufs[0], x, T * b->d);
        const uint32_t* di = upload(c, s.bufs[1], idx, T * K);
        const double* dg = upload(c, s.bufs[2], gates, T * K);
        const double* dr = residual ? upload(c, s.bufs[3], residual, T * b->d) : nullptr;
        double* dout = s.bufs[4].get<double>(T * b->d);
        int rc = scmoe_moe_forward_f64(c, b, xd, T, di, dg, K, n_zero, renorm, dr, dout);
        if (rc) throw ScmoeError{rc, c->last_error};
        download(c, out, dout, T * b->d);
        sync_and_check(c);
    });
}

int scmoe_rmsnorm(scmoe_ctx* c, const float* x, const float* gain, size_t rows, size_t d, float eps,
                  float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        launch_rmsnorm(c, x, gain, rows, d, eps, out, nullptr);
    });
}

int scmoe_layer_forward(scmoe_ctx* c, scmoe_router* r, scmoe_bank* b, const float* a1,
                        const float* a3, const float* gain, size_t T, int renorm, uint32_t* idx,
                        double* gates, uint32_t* ffn_count, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        check_layer_args(r, b);
        if (T == 0) return;
        layer_front(c, r, b, a1, gain, T, idx, gates, ffn_count);
        moe_back(c, b, c->ws.hmoe.get<float>(T * r->d), T, idx, gates, r->top_k, renorm, a3, out);
    });
}

}  // extern "C"

namespace {

struct BatchIO {
    const float* a1;
    const float* a3;
    uint32_t* idx;
    double* gates;
    uint32_t* cnt;
    float* out;
};

void ensure_batch_streams(scmoe_ctx* c) {
    if (c->s_front) return;
    SCMOE_CUDA(cudaStreamCreateWithFlags(&c->s_front, cudaStreamNonBlocking));
    SCMOE_CUDA(cudaStreamCreateWithFlags(&c->s_back, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_front[i], cudaEventDisableTiming));
        SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_back[i], cudaEventDisableTiming));
    }
    SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
}

// Two-stream batch pipeline shared by scmoe_layer_forward_batches and
// scmoe_layer_forward_host_batches: the front half of batch i+1 (rmsnorm,
// exact router -- the small-footprint kernel that co-resides with the grouped
// GEMM --, top-K, permutation, gather) runs on s_front while the back half of
// batch i (expert GEMMs, combine) runs on s_back.  Two workspaces alternate
// between batches.  io(i) returns batch i's device pointers (and may make
// s_front wait for its inputs); pre_back(i) lets s_back wait for the output
// buffers; post_back(i) is called once back(i) is enqueued.
template <class IO, class PreBack, class PostBack>
void run_batches(scmoe_ctx* c, scmoe_router* r, scmoe_bank* b, size_t n, const float* gain,
                 size_t T, int renorm, IO&& io, PreBack&& pre_back, PostBack&& post_back) {
    ensure_batch_streams(c);
    cudaStream_t user = c->stream;
    SCMOE_CUDA(cudaEventRecord(c->ev_join, user));
    SCMOE_CUDA(cudaStreamWaitEvent(c->s_front, c->ev_join, 0));
    SCMOE_CUDA(cudaStreamWaitEvent(c->s_back, c->ev_join, 0));
    c->overlapped = true;
    int slot = 0;  // c->ws holds slot `slot`'s buffers, c->ws_alt the other's
    struct Restore {
        scmoe_ctx* c;
        cudaStream_t user;
        int* slot;
        ~Restore() {
            if (*slot) std::swap(c->ws, c->ws_alt);
            c->stream = user;
            c->overlapped = false;
        }
    } restore{c, user, &slot};
    for (size_t i = 0; i < n; ++i) {
        const int want = (int)(i & 1);
        if (want != slot) {
            std::swap(c->ws, c->ws_alt);
            slot = want;
        }
        // front(i) reuses the workspace of batch i-2: wait for its back half
        c->stream = c->s_front;
        if (i >= 2) SCMOE_CUDA(cudaStreamWaitEvent(c->s_front, c->ev_back[slot], 0));
        const BatchIO x = io(i);
        layer_front(c, r, b, x.a1, gain, T, x.idx, x.gates, x.cnt);
        SCMOE_CUDA(cudaEventRecord(c->ev_front[slot], c->s_front));
        c->stream = c->s_back;
        SCMOE_CUDA(cudaStreamWaitEvent(c->s_back, c->ev_front[slot], 0));
        pre_back(i);
        moe_back(c, b, c->ws.hmoe.get<float>(T * r->d), T, x.idx, x.gates, r->top_k, renorm, x.a3,
                 x.out);
        SCMOE_CUDA(cudaEventRecord(c->ev_back[slot], c->s_back));
        post_back(i);
    }
    // the caller's stream resumes after the last back half (s_back is in order)
    SCMOE_CUDA(cudaStreamWaitEvent(user, c->ev_back[(n - 1) & 1], 0));
}

}  // namespace

extern "C" {

int scmoe_layer_forward_batches(scmoe_ctx* c, scmoe_router* r, scmoe_bank* b, size_t n_batches,
                                const float* const* a1, const float* const* a3, const float* gain,
                                size_t T, int renorm, uint32_t* const* idx, double* const* gates,
                                uint32_t* const* ffn_count, float* const* out) {
    return guarded(c, [&] {
        require_ctx(c);
        check_layer_args(r, b);
        if (T == 0 || n_batches == 0) return;
        run_batches(
            c, r, b, n_batches, gain, T, renorm,
            [&](size_t i) {
                return BatchIO{a1[i], a3 ? a3[i] : nullptr, idx[i], gates[i], ffn_count[i], out[i]};
            },
            [](size_t) {}, [](size_t) {});
    });
}

int scmoe_layer_forward_host_batches(scmoe_ctx* c, scmoe_router* r, scmoe_bank* b,
                                     size_t n_batches, const float* const* a1,
                                     const float* const* a3, const float* gain, size_t T,
                                     int renorm, uint32_t* const* idx, double* const* gates,
                                     uint32_t* const* ffn_count, float* const* out) {
    return guarded(c, [&] {
        require_ctx(c);
        check_layer_args(r, b);
        if (T == 0 || n_batches == 0) return;
        if (!c->s_h2d) {
            SCMOE_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
            SCMOE_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming));
                SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_in_a1[i], cudaEventDisableTiming));
                SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
                SCMOE_CUDA(cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming));
            }
        }
        // Compute stays serial on the caller's stream: this path is bound by the
        // host->device copy of the fp32 inputs (8 B per token-feature), and the
        // pipelined device schedule's small-footprint router would only add
        // latency here (measured: 9.2 vs 10.5 ms per LongCat batch).
        const size_t d = r->d, K = r->top_k;
        cudaStream_t comp = c->stream;
        const float* dg = gain ? upload(c, stage_of(c).bufs[6], gain, d) : nullptr;
        // copies of batch i may not start before work already queued on the
        // compute stream (earlier calls) has finished with the slot buffers
        SCMOE_CUDA(cudaEventRecord(c->ev_done[0], comp));
        SCMOE_CUDA(cudaEventRecord(c->ev_done[1], comp));
        SCMOE_CUDA(cudaEventRecord(c->ev_out[0], comp));
        SCMOE_CUDA(cudaEventRecord(c->ev_out[1], comp));
        for (size_t i = 0; i < n_batches; ++i) {
            const int s = (int)(i & 1);
            DevBuf* io = c->io[s];
            float* da1 = io[0].get<float>(T * d);
            float* da3 = a3 && a3[i] ? io[1].get<float>(T * d) : nullptr;
            float* dout = io[2].get<float>(T * d);
            uint32_t* di = io[3].get<uint32_t>(T * K);
            double* dgt = io[4].get<double>(T * K);
            uint32_t* dc = io[5].get<uint32_t>(T);
            // H2D(i): the slot's inputs were last read by compute(i-2)
            SCMOE_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_done[s], 0));
            SCMOE_CUDA(cudaMemcpyAsync(da1, a1[i], T * d * sizeof(float), cudaMemcpyHostToDevice,
                                       c->s_h2d));
            SCMOE_CUDA(cudaEventRecord(c->ev_in_a1[s], c->s_h2d));
            if (da3)
                SCMOE_CUDA(cudaMemcpyAsync(da3, a3[i], T * d * sizeof(float),
                                           cudaMemcpyHostToDevice, c->s_h2d));
            SCMOE_CUDA(cudaEventRecord(c->ev_in[s], c->s_h2d));
            // compute(i): needs its inputs, and the slot's outputs drained by D2H(i-2)
            // the front half needs a1 only: a3 (the residual) is still in flight
            SCMOE_CUDA(cudaStreamWaitEvent(comp, c->ev_in_a1[s], 0));
            SCMOE_CUDA(cudaStreamWaitEvent(comp, c->ev_out[s], 0));
            layer_front(c, r, b, da1, dg, T, di, dgt, dc);
            moe_back(c, b, c->ws.hmoe.get<float>(T * d), T, di, dgt, K, renorm, nullptr, nullptr,
                     /*phase=*/1);  // expert FFN
            SCMOE_CUDA(cudaStreamWaitEvent(comp, c->ev_in[s], 0));  // a3 for the combine
            moe_back(c, b, c->ws.hmoe.get<float>(T * d), T, di, dgt, K, renorm, da3, dout,
                     /*phase=*/2);
            SCMOE_CUDA(cudaEventRecord(c->ev_done[s], comp));
            // D2H(i)
            SCMOE_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_done[s], 0));
            SCMOE_CUDA(cudaMemcpyAsync(out[i], dout, T * d * sizeof(float), cudaMemcpyDeviceToHost,
                                       c->s_d2h));
            if (idx && idx[i])
                SCMOE_CUDA(cudaMemcpyAsync(idx[i], di, T * K * sizeof(uint32_t),
                                           cudaMemcpyDeviceToHost, c->s_d2h));
            if (gates && gates[i])
                SCMOE_CUDA(cudaMemcpyAsync(gates[i], dgt, T * K * sizeof(double),
                                           cudaMemcpyDeviceToHost, c->s_d2h));
            if (ffn_count && ffn_count[i])
                SCMOE_CUDA(cudaMemcpyAsync(ffn_count[i], dc, T * sizeof(uint32_t),
                                           cudaMemcpyDeviceToHost, c->s_d2h));
            SCMOE_CUDA(cudaEventRecord(c->ev_out[s], c->s_d2h));
        }
        SCMOE_CUDA(cudaStreamSynchronize(c->s_d2h));
        sync_and_check(c);
    });
}

int scmoe_dense_ffn(scmoe_ctx* c, scmoe_bank* b, const float* a1, const float* gain, size_t T,
                    float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!b || b->n != 1 || b->precision != SCMOE_PREC_BF16)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "dense_ffn: needs a one-expert bf16 bank");
        if (T == 0) return;
        const size_t d = b->d, I = b->inter;
        Workspace& ws = c->ws;
        const int tr = grouped_gemm_tile_rows_large();
        const size_t ntile = ceil_div(T, tr);
        __nv_bfloat16* xb = ws.dn_x.get<__nv_bfloat16>(T * d);
        __nv_bfloat16* h = ws.dn_h.get<__nv_bfloat16>(T * I);
        __nv_bfloat16* y = ws.dn_y.get<__nv_bfloat16>(T * d);
        TokenTile* tiles = ws.dn_tiles.get<TokenTile>(ntile + 1);
        int* ntd = reinterpret_cast<int*>(tiles + ntile);
        {
            ProfScope _p(c, "dense_rmsnorm");
            launch_rmsnorm(c, a1, gain, T, d, 1e-6f, nullptr, xb);
        }
        launch_row_tiles(c, T, tr, tiles, ntd);
        {
            ProfScope _p(c, "dense_gemm1_tcgen05");
            launch_grouped_gemm_bf16(c, b->w1t, 1, I, d, xb, T, nullptr, h, /*silu=*/1, tiles, ntd,
                                     ntile, tr);
        }
        {
            ProfScope _p(c, "dense_gemm2_tcgen05");
            launch_grouped_gemm_bf16(c, b->w2t, 1, d, I, h, T, nullptr, y, /*silu=*/0, tiles, ntd,
                                     ntile, tr);
        }
        ProfScope _p(c, "dense_residual");
        launch_add_bf16_residual(c, a1, y, T * d, out);
    });
}

int scmoe_layer_forward_host(scmoe_ctx* c, scmoe_router* r, scmoe_bank* b, const float* a1,
                             const float* a3, const float* gain, size_t T, int renorm,
                             uint32_t* idx, double* gates, uint32_t* ffn_count, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (T == 0) return;
        Stage& s = stage_of(c);
        const size_t d = r->d, K = r->top_k;
        const float* da1 = upload(c, s.bufs[0], a1, T * d);
        const float* da3 = a3 ? upload(c, s.bufs[5], a3, T * d) : nullptr;
        const float* dg = gain ? upload(c, s.bufs[6], gain, d) : nullptr;
        uint32_t* di = s.bufs[1].get<uint32_t>(T * K);
        double* dgt = s.bufs[2].get<double>(T * K);
        uint32_t* dc = s.bufs[3].get<uint32_t>(T);
        float* dout = s.bufs[4].get<float>(T * d);
        int rc = scmoe_layer_forward(c, r, b, da1, da3, dg, T, renorm, di, dgt, dc, dout);
        if (rc) throw ScmoeError{rc, c->last_error};
        if (idx) download(c, idx, di, T * K);
        if (gates) download(c, gates, dgt, T * K);
        if (ffn_count) download(c, ffn_count, dc, T);
        download(c, out, dout, T * d);
        sync_and_check(c);
    });
}

int scmoe_rng_fill_uniform(scmoe_ctx* c, uint64_t seed, uint64_t first, size_t n, double variance,
                           float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (variance < 0.0) SCMOE_THROW(SCMOE_ERR_PARAMETER, "seeded_init: variance must be >= 0");
        if (variance == 0.0) {
            SCMOE_CUDA(cudaMemsetAsync(out, 0, n * sizeof(float), c->stream));
            return;
        }
        launch_uniform_init(c, seed, first, n, std::sqrt(3.0 * variance), out);
    });
}

int scmoe_debug_expf(scmoe_ctx* c, const float* in, float* out, size_t n) {
    return guarded(c, [&] {
        require_ctx(c);
        launch_debug_expf(c, in, out, n);
    });
}

int scmoe_profile_enable(scmoe_ctx* c, int on) {
    return guarded(c, [&] {
        require_ctx(c);
        c->prof.on = on != 0;
    });
}

int scmoe_profile_flush(scmoe_ctx* c, int* n_entries) {
    return guarded(c, [&] {
        require_ctx(c);
        // device-wide: stages recorded on a second stream (overlapped layer)
        SCMOE_CUDA(cudaDeviceSynchronize());
        Profiler& p = c->prof;
        p.agg.clear();
        p.spans.clear();
        for (size_t i = 0; i < p.used; ++i) {
            float ms = 0.f, t0 = 0.f;
            SCMOE_CUDA(cudaEventElapsedTime(&ms, p.recs[i].a, p.recs[i].b));
            SCMOE_CUDA(cudaEventElapsedTime(&t0, p.recs[0].a, p.recs[i].a));
            p.spans.push_back(Profiler::Span{p.recs[i].name, (double)t0, (double)t0 + ms});
            ProfAgg* a = nullptr;
            for (auto& x : p.agg)
                if (x.name == p.recs[i].name) a = &x;
            if (!a) {
                p.agg.push_back(ProfAgg{p.recs[i].name, 0.0, 0});
                a = &p.agg.back();
            }
            a->ms += ms;
            a->count++;
        }
        p.used = 0;
        if (n_entries) *n_entries = (int)p.agg.size();
    });
}

int scmoe_profile_entry(scmoe_ctx* c, int i, const char** name, double* total_ms,
                        uint64_t* launches) {
    return guarded(c, [&] {
        if (i < 0 || (size_t)i >= c->prof.agg.size()) SCMOE_THROW(SCMOE_ERR_PARAMETER, "no such entry");
        if (name) *name = c->prof.agg[i].name.c_str();
        if (total_ms) *total_ms = c->prof.agg[i].ms;
        if (launches) *launches = c->prof.agg[i].count;
    });
}

int scmoe_profile_span(scmoe_ctx* c, int i, const char** name, double* start_ms, double* end_ms) {
    return guarded(c, [&] {
        if (i < 0 || (size_t)i >= c->prof.spans.size()) SCMOE_THROW(SCMOE_ERR_PARAMETER, "no such span");
        if (name) *name = c->prof.spans[i].name.c_str();
        if (start_ms) *start_ms = c->prof.spans[i].start_ms;
        if (end_ms) *end_ms = c->prof.spans[i].end_ms;
    });
}

int scmoe_debug_expf_range(scmoe_ctx* c, uint32_t first, float* out, size_t n) {
    return guarded(c, [&] {
        require_ctx(c);
        launch_debug_expf_range(c, first, out, n);
    });
}

// ---- expert parallelism -------------------------------------------------------

int scmoe_bank_init_uniform_shard(scmoe_ctx* c, scmoe_bank* b, uint64_t seed, uint64_t stream0,
                                  double variance, size_t first) {
    return scmoe_bank_init_uniform(c, b, seed, stream0 + 2 * first, variance);
}

int scmoe_rmsnorm_route(scmoe_ctx* c, scmoe_router* r, const float* a1, const float* gain,
                        size_t T, float* hmoe, void* hmoe_bf16, uint32_t* idx, double* gates,
                        uint32_t* ffn_count) {
    return guarded(c, [&] {
        require_ctx(c);
        validate_router(r->n_ffn, r->n_zero, r->top_k, r->k_expected, r->mu);
        if (T == 0) return;
        const size_t d = r->d, E = r->E();
        {
            ProfScope _p(c, "rmsnorm");
            launch_rmsnorm(c, a1, gain, T, d, 1e-6f, hmoe,
                           static_cast<__nv_bfloat16*>(hmoe_bf16));
        }
        float* logits = c->ws.logits.get<float>(T * E);
        route_logits(c, r, hmoe, T, logits);
        ProfScope _p(c, "softmax_topk");
        launch_softmax_topk(c, logits, T, E, r->top_k, r->n_ffn, r->b, idx, gates, ffn_count,
                            nullptr);
    });
}

int scmoe_ep_plan(scmoe_ctx* c, const uint32_t* idx, size_t T, size_t K, size_t n_ffn,
                  size_t n_zero, int world, int* send_counts, int* slot_send_pos, int* send_token,
                  int* send_expert) {
    return guarded(c, [&] {
        require_ctx(c);
        if (world < 1 || n_ffn % (size_t)world != 0)
            SCMOE_THROW(SCMOE_ERR_CONFIG, "ep: world size must divide the FFN expert count");
        if (T == 0) {
            SCMOE_CUDA(cudaMemsetAsync(send_counts, 0, world * sizeof(int), c->stream));
            return;
        }
        launch_check_indices(c, idx, T * K, n_ffn + n_zero);
        uint32_t* bins = c->ws.ep_bins.get<uint32_t>(T * K);
        launch_ep_bins(c, idx, T * K, n_ffn, n_ffn / world, world, bins);
        // one permutation over the G rank bins (+1 zero bin): offsets per rank,
        // position of each slot in the send buffer, token of each send row
        PermResult pr;
        {
            ProfScope _p(c, "ep_plan");
            pr = launch_permute(c, bins, T, K, world, world + 1, 256, /*multi=*/true);
        }
        SCMOE_CUDA(cudaMemcpyAsync(send_counts, pr.expert_count, world * sizeof(int),
                                   cudaMemcpyDeviceToDevice, c->stream));
        SCMOE_CUDA(cudaMemcpyAsync(slot_send_pos, pr.slot_pos, T * K * sizeof(int),
                                   cudaMemcpyDeviceToDevice, c->stream));
        SCMOE_CUDA(cudaMemcpyAsync(send_token, pr.row_token, T * K * sizeof(int),
                                   cudaMemcpyDeviceToDevice, c->stream));
        launch_ep_send_expert(c, idx, pr.slot_pos, T * K, send_expert);
    });
}

int scmoe_permutation(scmoe_ctx* c, const uint32_t* idx, size_t T, size_t K, size_t n_ffn,
                      size_t n_zero, int* expert_count, int* slot_row) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CHECK_ARG(K >= 1 && K <= 64, SCMOE_ERR_CONFIG, "moe_forward: top_k must be in [1, 64]");
        const size_t E = n_ffn + n_zero;
        if (T == 0) {
            if (expert_count) SCMOE_CUDA(cudaMemsetAsync(expert_count, 0, E * sizeof(int), c->stream));
            return;
        }
        launch_check_indices(c, idx, T * K, E);
        PermResult pr;
        {
            ProfScope _p(c, "permute");
            pr = launch_permute(c, idx, T, K, n_ffn, E, 192);
        }
        if (expert_count)
            SCMOE_CUDA(cudaMemcpyAsync(expert_count, pr.expert_count, E * sizeof(int),
                                       cudaMemcpyDeviceToDevice, c->stream));
        if (slot_row) launch_slot_rows(c, idx, pr.slot_pos, pr.expert_base, T * K, (int)n_ffn, slot_row);
    });
}

int scmoe_gather_rows_bf16(scmoe_ctx* c, const void* src, size_t d, const int* rows,
                           size_t n_rows, void* dst) {
    return guarded(c, [&] {
        require_ctx(c);
        ProfScope _p(c, "gather_rows");
        launch_gather_rows_bf16(c, static_cast<const __nv_bfloat16*>(src), d, rows, n_rows,
                                static_cast<__nv_bfloat16*>(dst));
    });
}

}  // extern "C"

namespace {
// Expert rows of the received slots; GEMM2's rows go to y (received order,
// through an unpermute copy) or, with row_dst, straight to row_dst[r] for
// received row r (e.g. the source rank's buffer over NVLink).
// token-tile width of the expert-parallel GEMMs: 256 (default) or 192
// (SCMOE_EP_TILE_ROWS=192: the smaller-footprint GEMM that the co-resident
// router fits next to)
int ep_tile_rows(const scmoe_ctx* c) {
    (void)c;
    static const int v = [] {
        const char* e = getenv("SCMOE_EP_TILE_ROWS");
        const int x = e ? atoi(e) : 256;
        return x == 128 || x == 192 ? x : 256;
    }();
    return v;
}

}  // namespace

namespace scmoe {
// R_dev: the row count lives on the device (R is then the capacity); the
// output must go to row_dst (expert-parallel receive side, ep.cu).
void moe_rows_impl(scmoe_ctx* c, scmoe_bank* b, const void* x_bf16, const int* row_expert,
                   int expert_offset, size_t R, void* y_bf16, const uint64_t* row_dst,
                   const int* R_dev) {
    if (b->precision != SCMOE_PREC_BF16)
        SCMOE_THROW(SCMOE_ERR_CONFIG, "moe_rows: needs a bf16 (tensor-core) bank");
    if (R == 0) return;
    SCMOE_CHECK_ARG(!R_dev || row_dst, SCMOE_ERR_INTERNAL, "moe_rows: device count needs row_dst");
    const size_t d = b->d, I = b->inter, n = b->n;
    Workspace& ws = c->ws;
    uint32_t* loc = ws.ep_local.get<uint32_t>(R);
    launch_ep_localize(c, row_expert, R, expert_offset, (int)n, loc, R_dev);
    // each row is a "token" routed to exactly one local expert (K = 1)
    PermResult pr;
    {
        ProfScope _p(c, "permute");
        pr = launch_permute(c, loc, R, 1, n, n, ep_tile_rows(c), false, R_dev);
    }
    const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x_bf16);
    __nv_bfloat16* xp = ws.xp.get<__nv_bfloat16>(R * d);
    __nv_bfloat16* h = ws.h.get<__nv_bfloat16>(R * I);
    {
        ProfScope _p(c, "gather");
        launch_gather_bf16(c, xb, d, pr.row_token, pr.expert_base, n, R, xp);
    }
    {
        ProfScope _p(c, "gemm1_tcgen05");
        launch_grouped_gemm_bf16(c, b->w1t, n, I, d, xp, R, nullptr, h, 1, pr.tiles, pr.n_tiles,
                                 pr.max_tiles, ep_tile_rows(c));
    }
    if (row_dst) {
        // permuted row p holds received row row_token[p]
        ProfScope _p(c, "gemm2_tcgen05");
        launch_grouped_gemm_bf16(c, b->w2t, n, d, I, h, R, nullptr, nullptr, 0, pr.tiles,
                                 pr.n_tiles, pr.max_tiles, ep_tile_rows(c), row_dst,
                                 pr.row_token);
        return;
    }
    __nv_bfloat16* y = ws.ep_y.get<__nv_bfloat16>(R * d);
    {
        ProfScope _p(c, "gemm2_tcgen05");
        launch_grouped_gemm_bf16(c, b->w2t, n, d, I, h, R, nullptr, y, 0, pr.tiles, pr.n_tiles,
                                 pr.max_tiles, ep_tile_rows(c));
    }
    // back to the received order: y_out[r] = y[slot_pos[r]]
    ProfScope _p(c, "unpermute");
    launch_gather_rows_bf16(c, y, d, pr.slot_pos, R, static_cast<__nv_bfloat16*>(y_bf16));
}
}  // namespace scmoe

extern "C" {

int scmoe_moe_rows(scmoe_ctx* c, scmoe_bank* b, const void* x_bf16, const int* row_expert,
                   int expert_offset, size_t R, void* y_bf16) {
    return guarded(c, [&] {
        require_ctx(c);
        moe_rows_impl(c, b, x_bf16, row_expert, expert_offset, R, y_bf16, nullptr, nullptr);
    });
}

int scmoe_moe_rows_to(scmoe_ctx* c, scmoe_bank* b, const void* x_bf16, const int* row_expert,
                      int expert_offset, size_t R, const uint64_t* row_dst) {
    return guarded(c, [&] {
        require_ctx(c);
        SCMOE_CHECK_ARG(row_dst != nullptr || R == 0, SCMOE_ERR_PARAMETER,
                        "moe_rows_to: row_dst is required");
        moe_rows_impl(c, b, x_bf16, row_expert, expert_offset, R, nullptr, row_dst, nullptr);
    });
}

int scmoe_ep_put_rows(scmoe_ctx* c, const void* src_bf16, size_t d, const int* send_token,
                      const int* send_expert, size_t n_send, const int* send_start,
                      const int64_t* dst_offset, const uint64_t* peer_rows,
                      const uint64_t* peer_expert, int world) {
    return guarded(c, [&] {
        require_ctx(c);
        ProfScope _p(c, "ep_put_rows");
        launch_ep_put_rows(c, static_cast<const __nv_bfloat16*>(src_bf16), d, send_token,
                           send_expert, n_send, send_start, dst_offset, peer_rows, peer_expert,
                           world);
    });
}

int scmoe_combine_rows(scmoe_ctx* c, scmoe_bank* b, const float* x, const void* y_rows,
                       const int* slot_row, const uint32_t* idx, const double* gates, size_t T,
                       size_t K, size_t n_ffn_total, int renorm, const float* residual,
                       float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (T == 0) return;
        ProfScope _p(c, "combine");
        launch_combine_bf16(c, x, static_cast<const __nv_bfloat16*>(y_rows), idx, gates, slot_row,
                            T, b->d, K, n_ffn_total, (float)b->gamma_ffn(), (float)b->gamma_zero(),
                            renorm, residual, out);
    });
}

}  // extern "C"

// ===========================================================================
// MLA, forward value (f2 row): blocks.hpp:38-181.
// ===========================================================================
namespace {

void mla_check_tc_dims(const scmoe_mla* m) {
    if (m->d % 64 || m->dq % 64 || m->dkv % 64 || (m->H * m->dhc) % 64 || m->dhc > 256)
        SCMOE_THROW(SCMOE_ERR_CONFIG,
                    "mla: the tensor-core path needs d, d_q, d_kv, H*d_head_c multiples of 64 "
                    "and d_head_c <= 256");
}

void mla_check_dims(size_t d, size_t dq, size_t dkv, size_t H, size_t dhr) {
    if (d == 0 || dq == 0 || dkv == 0)
        SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla_scale_factors: dims must be positive");
    if (H == 0) SCMOE_THROW(SCMOE_ERR_DIMENSION, "rope: heads must divide width");
    if (dhr % 2 != 0) SCMOE_THROW(SCMOE_ERR_DIMENSION, "rope: rotary width per head must be even");
}

// (cos, sin) table of rope_apply (tensor.hpp:207-215) for positions
// [0, npos): theta = pos * pow(base, -2p/hd) in double, then cast to float --
// the reference's own expression, evaluated by the same libm.
void mla_ensure_rope(scmoe_ctx* c, scmoe_mla* m, size_t npos) {
    const size_t half = m->dhr / 2;
    if (half == 0 || npos <= m->rope_rows) return;
    const size_t rows = std::max(npos, 2 * m->rope_rows);
    std::vector<float2> t(rows * half);
    for (size_t pos = 0; pos < rows; ++pos)
        for (size_t p = 0; p < half; ++p) {
            const double theta = static_cast<double>(pos) *
                                 std::pow(m->rope_base, -2.0 * static_cast<double>(p) /
                                                            static_cast<double>(m->dhr));
            t[pos * half + p] = make_float2(static_cast<float>(std::cos(theta)),
                                            static_cast<float>(std::sin(theta)));
        }
    SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(m->rope);
    m->rope = nullptr;
    SCMOE_CUDA(cudaMalloc(&m->rope, t.size() * sizeof(float2)));
    stream_copy(c, m->rope, t.data(), t.size() * sizeof(float2));
    m->rope_rows = rows;
}

// C[rows, N] (ldc) = A[rows, K] (lda) . B[K, N]: sequential-k chains.
void mla_gemm(scmoe_ctx* c, DevBuf& tiles_buf, const float* A, size_t lda, size_t rows,
              const float* B, size_t K, size_t N, float* C, size_t ldc) {
    if (rows == 0 || N == 0) return;
    if (rows <= 4 && launch_seq_gemv(c, A, lda, rows, B, N, C, ldc, K, N)) return;  // decode
    // 128 x 128 tiles (8 x 8 chains per thread) once they fill two waves
    static const bool big_ok = [] {
        const char* e = getenv("SCMOE_MLA_TILE");
        return !(e && atoi(e) == 64);
    }();
    const int tr = big_ok && ceil_div(rows, 128) * ceil_div(N, 128) >= (size_t)c->num_sms * 2
                       ? 128
                       : seq_gemm_tile_rows(rows, N, c->num_sms);
    const size_t ntile = ceil_div(rows, tr);
    TokenTile* tiles = tiles_buf.get<TokenTile>(ntile + 1);
    int* ntd = reinterpret_cast<int*>(tiles + ntile);
    launch_row_tiles(c, rows, tr, tiles, ntd);
    launch_seq_gemm(c, A, lda, nullptr, B, N, 0, C, ldc, K, N, /*silu=*/0, tiles, ntd, ntile, tr);
}

void mla_cache_reserve(scmoe_ctx* c, scmoe_mla* m, scmoe_mla_cache* k, size_t need) {
    if (need <= k->cap) return;
    const size_t cap = std::max<size_t>({need, 2 * k->cap, 16});
    float *ckv = nullptr, *kr = nullptr, *kv = nullptr;
    SCMOE_CUDA(cudaMalloc(&ckv, cap * m->dkv * sizeof(float)));
    SCMOE_CUDA(cudaMalloc(&kr, std::max<size_t>(cap * m->dhr, 1) * sizeof(float)));
    SCMOE_CUDA(cudaMalloc(&kv, cap * m->n3() * sizeof(float)));
    if (k->len) {
        SCMOE_CUDA(cudaMemcpyAsync(ckv, k->c_kv, k->len * m->dkv * sizeof(float),
                                   cudaMemcpyDeviceToDevice, c->stream));
        if (m->dhr)
            SCMOE_CUDA(cudaMemcpyAsync(kr, k->k_r, k->len * m->dhr * sizeof(float),
                                       cudaMemcpyDeviceToDevice, c->stream));
        SCMOE_CUDA(cudaMemcpyAsync(kv, k->kv, k->len * m->n3() * sizeof(float),
                                   cudaMemcpyDeviceToDevice, c->stream));
    }
    SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(k->c_kv);
    cudaFree(k->k_r);
    cudaFree(k->kv);
    k->c_kv = ckv;
    k->k_r = kr;
    k->kv = kv;
    k->cap = cap;
}

}  // namespace

int scmoe_mla_create(scmoe_ctx* c, size_t d, size_t dq, size_t dkv, size_t H, size_t dhc,
                     size_t dhr, double rope_base, int va, scmoe_mla** out) {
    return guarded(c, [&] {
        require_ctx(c);
        mla_check_dims(d, dq, dkv, H, dhr);
        auto* m = new scmoe_mla();
        m->d = d; m->dq = dq; m->dkv = dkv; m->H = H; m->dhc = dhc; m->dhr = dhr;
        m->rope_base = rope_base;
        m->variance_alignment = va;
        // MlaParams::alpha_q/alpha_kv (blocks.hpp:51-56), cast as g.scale does
        m->alpha_q = va ? static_cast<float>(std::sqrt(static_cast<double>(d) / dq)) : 1.0f;
        m->alpha_kv = va ? static_cast<float>(std::sqrt(static_cast<double>(d) / dkv)) : 1.0f;
        m->att_scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(dhc + dhr)));
        const size_t sizes[4] = {d * m->n1(), dq * m->n2(), dkv * m->n3(), H * dhc * d};
        float** ptrs[4] = {&m->w_h, &m->w_q, &m->w_kv, &m->w_o};
        for (int i = 0; i < 4; ++i) {
            SCMOE_CUDA(cudaMalloc(ptrs[i], std::max<size_t>(sizes[i], 1) * sizeof(float)));
            stream_zero(c, *ptrs[i], std::max<size_t>(sizes[i], 1) * sizeof(float));
        }
        *out = m;
    });
}

int scmoe_mla_destroy(scmoe_ctx* c, scmoe_mla* m) {
    if (!m) return SCMOE_OK;
    if (c) cudaSetDevice(c->device);
    cudaFree(m->w_h);
    cudaFree(m->w_q);
    cudaFree(m->w_kv);
    cudaFree(m->w_o);
    cudaFree(m->rope);
    for (auto* w : m->tc_w) cudaFree(w);
    delete m;
    return SCMOE_OK;
}

int scmoe_mla_set_precision(scmoe_ctx* c, scmoe_mla* m, int precision) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null handle");
        if (precision != SCMOE_PREC_F32_EXACT && precision != SCMOE_PREC_BF16)
            SCMOE_THROW(SCMOE_ERR_CONFIG, "mla: precision must be F32_EXACT or BF16");
        if (precision == SCMOE_PREC_BF16) mla_check_tc_dims(m);
        m->precision = precision;
    });
}

static int mla_set_weight(scmoe_ctx* c, scmoe_mla* m, int which, const float* w) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null handle");
        const size_t H = m->H, dhc = m->dhc, dhr = m->dhr;
        // destination matrix, its row count / leading dimension, column offset, width
        float* dst = nullptr;
        size_t rows = 0, ld = 0, col = 0, width = 0;
        switch (which) {
            case SCMOE_MLA_W_DQ: dst = m->w_h; rows = m->d; ld = m->n1(); col = 0; width = m->dq; break;
            case SCMOE_MLA_W_DKV: dst = m->w_h; rows = m->d; ld = m->n1(); col = m->dq; width = m->dkv; break;
            case SCMOE_MLA_W_KR: dst = m->w_h; rows = m->d; ld = m->n1(); col = m->dq + m->dkv; width = dhr; break;
            case SCMOE_MLA_W_UQ: dst = m->w_q; rows = m->dq; ld = m->n2(); col = 0; width = H * dhc; break;
            case SCMOE_MLA_W_QR: dst = m->w_q; rows = m->dq; ld = m->n2(); col = H * dhc; width = H * dhr; break;
            case SCMOE_MLA_W_UK: dst = m->w_kv; rows = m->dkv; ld = m->n3(); col = 0; width = H * dhc; break;
            case SCMOE_MLA_W_UV: dst = m->w_kv; rows = m->dkv; ld = m->n3(); col = H * dhc; width = H * dhc; break;
            case SCMOE_MLA_W_O: dst = m->w_o; rows = H * dhc; ld = m->d; col = 0; width = m->d; break;
            default: SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: unknown weight id");
        }
        if (width == 0 || rows == 0) return;
        m->tc_dirty = true;  // the tensor-core copy is rebuilt on the next bf16 forward
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        SCMOE_CUDA(cudaMemcpy2DAsync(dst + col, ld * sizeof(float), w, width * sizeof(float),
                                     width * sizeof(float), rows, cudaMemcpyDefault, c->stream));
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
    });
}
int scmoe_mla_set_weight_host(scmoe_ctx* c, scmoe_mla* m, int which, const float* w) {
    return mla_set_weight(c, m, which, w);
}
int scmoe_mla_set_weight(scmoe_ctx* c, scmoe_mla* m, int which, const float* w) {
    return mla_set_weight(c, m, which, w);
}

int scmoe_mla_forward(scmoe_ctx* c, scmoe_mla* m, const float* h, size_t rows, size_t seq_len,
                      float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null handle");
        if (seq_len == 0 || rows % seq_len != 0)
            SCMOE_THROW(SCMOE_ERR_DIMENSION, "attention: rows must pack whole sequences");
        if (rows == 0) return;
        Workspace& ws = c->ws;
        const size_t d = m->d, dq = m->dq, dkv = m->dkv, H = m->H, dhc = m->dhc, dhr = m->dhr;
        const size_t n1 = m->n1(), n2 = m->n2(), n3 = m->n3();
        const size_t B = rows / seq_len;
        mla_ensure_rope(c, m, seq_len);
        if (m->precision == SCMOE_PREC_BF16) {  // tensor cores (mla_tc.cu)
            mla_forward_tc(c, m, h, rows, seq_len, m->rope, out);
            return;
        }
        float* p1 = ws.mla_p1.get<float>(rows * n1);  // [cq | ckv | kr]
        float* qb = ws.mla_q.get<float>(rows * n2);   // [qc | qr]
        float* kv = ws.mla_kv.get<float>(rows * n3);  // [kc | vv]
        const size_t nkt = ceil_div(seq_len, 64);
        float* att = ws.mla_att.get<float>(B * H * seq_len * (seq_len + nkt));
        float* mg = ws.mla_m.get<float>(rows * H * dhc);
        {
            ProfScope _p(c, "mla_proj_h");
            mla_gemm(c, ws.mla_tiles, h, d, rows, m->w_h, d, n1, p1, n1);
            launch_mla_scale_rope(c, p1, n1, rows, (int)dq, m->alpha_q, (int)dkv, m->alpha_kv,
                                  (int)(dq + dkv), 1, (int)dhr, m->rope, 0, seq_len);
        }
        {
            ProfScope _p(c, "mla_proj_q");
            mla_gemm(c, ws.mla_tiles, p1, n1, rows, m->w_q, dq, n2, qb, n2);
            launch_mla_scale_rope(c, qb, n2, rows, 0, 1.f, 0, 1.f, (int)(H * dhc), (int)H,
                                  (int)dhr, m->rope, 0, seq_len);
        }
        {
            ProfScope _p(c, "mla_proj_kv");
            mla_gemm(c, ws.mla_tiles, p1 + dq, n1, rows, m->w_kv, dkv, n3, kv, n3);
        }
        MlaAttnArgs a{};
        a.qc = qb; a.qr = qb + H * dhc; a.ldq = n2;
        a.kc = kv; a.v = kv + H * dhc; a.ldkv = n3;
        a.kr = p1 + dq + dkv; a.ldkr = n1;
        a.att = att; a.part_max = att + B * H * seq_len * seq_len;
        a.merged = mg; a.ldm = H * dhc;
        a.H = (int)H; a.dhc = (int)dhc; a.dhr = (int)dhr;
        a.nq = (int)seq_len; a.nk = (int)seq_len; a.q0 = 0;
        a.scale = m->att_scale;
        launch_mla_attention(c, a, (int)B);
        ProfScope _p(c, "mla_proj_o");
        mla_gemm(c, ws.mla_tiles, mg, H * dhc, rows, m->w_o, H * dhc, d, out, d);
    });
}

int scmoe_mla_forward_host(scmoe_ctx* c, scmoe_mla* m, const float* h, size_t rows,
                           size_t seq_len, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null handle");
        Stage& s = stage_of(c);
        const float* dh = upload(c, s.bufs[0], h, rows * m->d);
        float* dout = s.bufs[4].get<float>(rows * m->d);
        int rc = scmoe_mla_forward(c, m, dh, rows, seq_len, dout);
        if (rc) throw ScmoeError{rc, c->last_error};
        download(c, out, dout, rows * m->d);
        sync_and_check(c);
    });
}

int scmoe_mla_cache_create(scmoe_ctx* c, scmoe_mla* m, size_t capacity_hint,
                           scmoe_mla_cache** out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null handle");
        auto* k = new scmoe_mla_cache();
        try {
            mla_cache_reserve(c, m, k, std::max<size_t>(capacity_hint, 1));
        } catch (...) {
            delete k;
            throw;
        }
        *out = k;
    });
}

int scmoe_mla_cache_destroy(scmoe_ctx* c, scmoe_mla_cache* k) {
    if (!k) return SCMOE_OK;
    if (c) cudaSetDevice(c->device);
    cudaFree(k->c_kv);
    cudaFree(k->k_r);
    cudaFree(k->kv);
    delete k;
    return SCMOE_OK;
}

int scmoe_mla_cache_length(scmoe_ctx* c, scmoe_mla_cache* k, size_t* length) {
    return guarded(c, [&] {
        if (!k || !length) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla cache: null argument");
        *length = k->len;
    });
}

int scmoe_mla_cache_read_host(scmoe_ctx* c, scmoe_mla* m, scmoe_mla_cache* k, float* c_kv,
                              float* k_r) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m || !k) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla cache: null argument");
        if (c_kv) download(c, c_kv, k->c_kv, k->len * m->dkv);
        if (k_r) download(c, k_r, k->k_r, k->len * m->dhr);
        sync_and_check(c);
    });
}

int scmoe_mla_infer_step(scmoe_ctx* c, scmoe_mla* m, scmoe_mla_cache* k, const float* h_t,
                         size_t position, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m || !k) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null argument");
        if (k->len != position)
            SCMOE_THROW(SCMOE_ERR_STATE, "mla_infer_step: cache holds " + std::to_string(k->len) +
                                             " rows but position is " + std::to_string(position));
        Workspace& ws = c->ws;
        const size_t d = m->d, dq = m->dq, dkv = m->dkv, H = m->H, dhc = m->dhc, dhr = m->dhr;
        const size_t n1 = m->n1(), n2 = m->n2(), n3 = m->n3();
        mla_ensure_rope(c, m, position + 1);
        mla_cache_reserve(c, m, k, position + 1);
        float* p1 = ws.mla_p1.get<float>(n1);
        float* qb = ws.mla_q.get<float>(n2);
        float* att = ws.mla_att.get<float>(H * (position + 1 + ceil_div(position + 1, 64)));
        float* mg = ws.mla_m.get<float>(H * dhc);
        ProfScope _p(c, "mla_infer_step");
        mla_gemm(c, ws.mla_tiles, h_t, d, 1, m->w_h, d, n1, p1, n1);
        launch_mla_scale_rope(c, p1, n1, 1, (int)dq, m->alpha_q, (int)dkv, m->alpha_kv,
                              (int)(dq + dkv), 1, (int)dhr, m->rope, position, 1);
        // append to the compressed cache (blocks.hpp:145-146)
        SCMOE_CUDA(cudaMemcpyAsync(k->c_kv + position * dkv, p1 + dq, dkv * sizeof(float),
                                   cudaMemcpyDeviceToDevice, c->stream));
        if (dhr)
            SCMOE_CUDA(cudaMemcpyAsync(k->k_r + position * dhr, p1 + dq + dkv, dhr * sizeof(float),
                                       cudaMemcpyDeviceToDevice, c->stream));
        mla_gemm(c, ws.mla_tiles, p1, n1, 1, m->w_q, dq, n2, qb, n2);
        launch_mla_scale_rope(c, qb, n2, 1, 0, 1.f, 0, 1.f, (int)(H * dhc), (int)H, (int)dhr,
                              m->rope, position, 1);
        // this row's expanded kc | vv, kept beside the compressed cache
        mla_gemm(c, ws.mla_tiles, k->c_kv + position * dkv, dkv, 1, m->w_kv, dkv, n3,
                 k->kv + position * n3, n3);
        k->len = position + 1;
        MlaAttnArgs a{};
        a.qc = qb; a.qr = qb + H * dhc; a.ldq = n2;
        a.kc = k->kv; a.v = k->kv + H * dhc; a.ldkv = n3;
        a.kr = k->k_r; a.ldkr = dhr;
        a.att = att; a.part_max = att + H * (position + 1);
        a.merged = mg; a.ldm = H * dhc;
        a.H = (int)H; a.dhc = (int)dhc; a.dhr = (int)dhr;
        a.nq = 1; a.nk = (int)(position + 1); a.q0 = (int)position;
        a.scale = m->att_scale;
        launch_mla_attention(c, a, 1);
        mla_gemm(c, ws.mla_tiles, mg, H * dhc, 1, m->w_o, H * dhc, d, out, d);
    });
}

int scmoe_mla_infer_step_host(scmoe_ctx* c, scmoe_mla* m, scmoe_mla_cache* k, const float* h_t,
                              size_t position, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        if (!m) SCMOE_THROW(SCMOE_ERR_PARAMETER, "mla: null handle");
        Stage& s = stage_of(c);
        const float* dh = upload(c, s.bufs[0], h_t, m->d);
        float* dout = s.bufs[4].get<float>(m->d);
        int rc = scmoe_mla_infer_step(c, m, k, dh, position, dout);
        if (rc) throw ScmoeError{rc, c->last_error};
        download(c, out, dout, m->d);
        sync_and_check(c);
    });
}

// ===========================================================================
// The full ScMoE layer (Model::build_layer, model.hpp:355-409, one chunk):
//   a1  = x  + MLA1(rmsnorm(x, norm1))
//   dd  = a1 + FFN(rmsnorm(a1, norm_ffn))            (dense shortcut branch)
//   a3  = dd + MLA2(rmsnorm(dd, norm2))
//   out = a3 + moe(rmsnorm(a1, norm_moe))             (scmoe: MoE input is a1)
// overlap = 1 runs the MoE branch (routing, permutation, expert FFN) on a
// second stream as soon as a1 exists, beside the dense FFN and MLA2 -- the
// shortcut connection's point (PAPER.md SBO); only the final combine waits
// for a3.  Same results either way (every kernel is order-independent of the
// schedule).
// ===========================================================================
int scmoe_layer_full_forward(scmoe_ctx* c, scmoe_mla* mla1, scmoe_mla* mla2, scmoe_bank* dense,
                             scmoe_router* r, scmoe_bank* b, const float* norm1,
                             const float* norm_ffn, const float* norm2, const float* norm_moe,
                             const float* x, size_t T, size_t seq_len, int renorm, int overlap,
                             uint32_t* idx, double* gates, uint32_t* ffn_count, float* a1_out,
                             float* a3_out, float* out) {
    return guarded(c, [&] {
        require_ctx(c);
        check_layer_args(r, b);
        if (!mla1 || !mla2 || !dense)
            SCMOE_THROW(SCMOE_ERR_PARAMETER, "layer_full: null MLA / dense handle");
        const size_t d = r->d;
        if (mla1->d != d || mla2->d != d || dense->d != d)
            SCMOE_THROW(SCMOE_ERR_DIMENSION, "layer_full: d_model mismatch");
        if (seq_len == 0 || T % seq_len != 0)
            SCMOE_THROW(SCMOE_ERR_DIMENSION, "attention: rows must pack whole sequences");
        if (T == 0) return;
        Workspace& ws = c->ws;
        float* xn = ws.full_n.get<float>(T * d);
        float* m = ws.full_m.get<float>(T * d);
        float* a1 = a1_out ? a1_out : ws.full_a1.get<float>(T * d);
        float* dd = ws.full_dd.get<float>(T * d);
        float* a3 = a3_out ? a3_out : ws.full_a3.get<float>(T * d);
        const cudaStream_t sa = c->stream;
        auto run = [&](int rc) {
            if (rc) throw ScmoeError{rc, c->last_error};
        };
        if (overlap && !c->s_moe) {
            // highest priority: as MLA CTAs retire, the CTA scheduler hands the
            // freed SM space to the MoE branch's kernels first, so a grouped-GEMM
            // CTA (HBM / tensor bound) shares SMs with an MLA CTA (FP32 pipe)
            int lo = 0, hi = 0;
            SCMOE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            const char* pe = getenv("SCMOE_MOE_PRIO");
            const int prio = (pe && pe[0] == 'h') ? hi : lo;
            SCMOE_CUDA(cudaStreamCreateWithPriority(&c->s_moe, cudaStreamNonBlocking, prio));
            for (auto& e : c->ev_full) SCMOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const cudaStream_t sb = overlap ? c->s_moe : sa;
        // a1 = x + MLA1(rmsnorm(x))
        launch_rmsnorm(c, x, norm1, T, d, 1e-6f, xn, nullptr);
        run(scmoe_mla_forward(c, mla1, xn, T, seq_len, m));
        launch_add_f32(c, x, m, T * d, a1);
        // MoE branch up to the expert outputs (stream b)
        if (overlap) {
            SCMOE_CUDA(cudaEventRecord(c->ev_full[0], sa));
            SCMOE_CUDA(cudaStreamWaitEvent(sb, c->ev_full[0], 0));
        }
        c->stream = sb;
        // overlapped: the MoE branch's exact router is FP32-pipe work; its
        // small co-resident kernel shares the SMs with the dense / MLA2 GEMMs of
        // stream a, which take the smaller-footprint ring to leave it room
        const bool ov_prev = c->overlapped;
        c->overlapped = overlap != 0;
        try {
            layer_front(c, r, b, a1, norm_moe, T, idx, gates, ffn_count);
            c->overlapped = ov_prev;
            moe_back(c, b, ws.hmoe.get<float>(T * d), T, idx, gates, r->top_k, renorm, nullptr,
                     nullptr, /*phase=*/1);
        } catch (...) {
            c->stream = sa;
            c->overlapped = ov_prev;
            throw;
        }
        c->stream = sa;
        // dd = a1 + FFN(rmsnorm(a1)); a3 = dd + MLA2(rmsnorm(dd)) (stream a)
        struct CorunGuard {
            scmoe_ctx* c;
            bool prev;
            ~CorunGuard() { c->corun_gemm = prev; }
        } corun_guard{c, c->corun_gemm};
        c->corun_gemm = overlap != 0;
        run(scmoe_dense_ffn(c, dense, a1, norm_ffn, T, dd));
        launch_rmsnorm(c, dd, norm2, T, d, 1e-6f, xn, nullptr);
        run(scmoe_mla_forward(c, mla2, xn, T, seq_len, m));
        launch_add_f32(c, dd, m, T * d, a3);
        c->corun_gemm = corun_guard.prev;
        // out = a3 + combine (stream b, after a3)
        if (overlap) {
            SCMOE_CUDA(cudaEventRecord(c->ev_full[1], sa));
            SCMOE_CUDA(cudaStreamWaitEvent(sb, c->ev_full[1], 0));
        }
        c->stream = sb;
        try {
            moe_back(c, b, ws.hmoe.get<float>(T * d), T, idx, gates, r->top_k, renorm, a3, out,
                     /*phase=*/2);
        } catch (...) {
            c->stream = sa;
            throw;
        }
        c->stream = sa;
        if (overlap) {
            SCMOE_CUDA(cudaEventRecord(c->ev_full[2], sb));
            SCMOE_CUDA(cudaStreamWaitEvent(sa, c->ev_full[2], 0));
        }
    });
}
