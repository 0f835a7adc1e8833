// ep.cu -- expert-parallel ScMoE layer behind the C ABI.
//
// One process (or thread) per GPU.  Router and bias replicated, tokens
// sharded, FFN experts block-partitioned (rank g owns [g*N/G, (g+1)*N/G)),
// zero experts stay local.  Per layer, all stream-ordered on
// the device with no host synchronisation:
//
//   route      rmsnorm + exact router + top-K          (model.hpp:394-397)
//   plan       FFN slots grouped by owning rank, (token, slot) order
//   exchange   every rank stores its row of the [G][G] slot-count matrix into
//              every peer's buffer, then an epoch flag; the same kernel waits
//              for all rows and derives the offsets (send / receive / return)
//   dispatch   one warp per slot stores its bf16 row (+ expert id) straight
//              into the owner's receive buffer over NVLink; epoch barrier
//   experts    grouped GEMM1(+SiLU) / GEMM2 on the received rows (tcgen05),
//              the row count read on the device; GEMM2's epilogue writes every
//              output row into the SOURCE rank's return buffer (the return
//              all-to-all fused into the GEMM, tile by tile); epoch barrier
//   combine    rank-order combine + zero-expert identity + residual at the
//              source (blocks.hpp:251-274)
//
// Expert rows come back per slot and the GEMM's accumulation per element does
// not depend on the tile composition, so the G-rank output is bitwise equal to
// the single-GPU layer.  NCCL provides the communicator (ncclCommInitRank), the
// one-time exchange of the buffers' CUDA IPC handles, and the controller's
// counter all-reduce (router.hpp:158-169 needs the global batch); the data path
// is our own kernels over peer memory.
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace scmoe;

// NCCL is bound at run time, not link time: a process that also loads
// another NCCL (e.g. PyTorch's newer build) must see exactly one libnccl.so.2,
// whichever was loaded first.  Resolution order: an already-loaded
// libnccl.so.2, $SCMOE_NCCL_LIB, then the system libnccl.so.2.
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGetErrorString) getErrorString = nullptr;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            if (const char* p = getenv("SCMOE_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.getErrorString =
            reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.getUniqueId || !api.commInitRank || !api.allGather || !api.allReduce ||
        !api.commDestroy || !api.getErrorString)
        SCMOE_THROW(SCMOE_ERR_CUDA, "ep: libnccl.so.2 not found (set SCMOE_NCCL_LIB)");
    return api;
}

#define SCMOE_NCCL(expr)                                                                       \
    do {                                                                                       \
        ncclResult_t _r = (expr);                                                              \
        if (_r != ncclSuccess)                                                                 \
            SCMOE_THROW(SCMOE_ERR_CUDA,                                                        \
                        std::string(#expr " failed: ") + nccl().getErrorString(_r));           \
    } while (0)

namespace {

constexpr int kMaxWorld = 32;
constexpr int kChannels = 3;  // per buffer set: 0 count exchange, 1 dispatch done, 2 return done
constexpr int kSets = 2;      // alternate between consecutive batches (pipelined schedule)

// Per-call routing plan, derived on the device from the exchanged count matrix.
struct EpPlan {
    int send_start[kMaxWorld + 1];    // my send rows for rank g: [send_start[g], send_start[g+1])
    int64_t dst_offset[kMaxWorld];    // where my rows start in rank g's receive buffer
    int recv_start[kMaxWorld + 1];    // rows from source s in my receive buffer
    int back_start[kMaxWorld];        // where in source s's send order its rows for me start
    int n_recv;
    int pad;
};

// Symmetric slab (same layout on every rank, mapped by every peer).
struct SlabLayout {
    size_t counts, flags, recv, recv_exp, back, bytes;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ld_acquire_sys_s32(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Cross-rank epoch barrier on channel `ch` of one buffer set.  With my_counts,
// this rank's row of the slot-count matrix travels with the barrier (stored in
// every peer's matrix before the flag) and, once every row has arrived, the
// plan is derived from the matrix.  Thread g talks to rank g.  The release
// store of the flag is ordered after this kernel's row stores and, by the
// stream order plus the system-scope fence, after the previous kernels' peer
// stores (the dispatch, GEMM2's return rows).
__global__ void ep_signal_wait_kernel(const unsigned long long* __restrict__ peer_base,
                                      SlabLayout lay, int ch, unsigned long long epoch, int me,
                                      int G, const int* __restrict__ my_counts,
                                      EpPlan* __restrict__ plan, int* __restrict__ dev_status) {
    const int g = threadIdx.x;
    if (g < G) {
        if (my_counts) {
            int* row = reinterpret_cast<int*>(peer_base[g] + lay.counts) + me * kMaxWorld;
            for (int j = 0; j < G; ++j) row[j] = my_counts[j];
        }
        __threadfence_system();
        st_release_sys(reinterpret_cast<unsigned long long*>(peer_base[g] + lay.flags) +
                           ch * kMaxWorld + me,
                       epoch);
        const unsigned long long* mine =
            reinterpret_cast<const unsigned long long*>(peer_base[me] + lay.flags) +
            ch * kMaxWorld + g;
        // a peer that never arrives (crashed rank) must not hang the GPU
        const uint64_t t0 = global_ns();
        while (ld_acquire_sys(mine) < epoch) {
            __nanosleep(100);
            if (global_ns() - t0 > 60ull * 1000000000ull) {
                atomicExch(dev_status, DEV_ERR_TIMEOUT);
                break;
            }
        }
    }
    __syncthreads();
    if (plan && g == 0) {
        const int* M = reinterpret_cast<const int*>(peer_base[me] + lay.counts);
        auto m = [&](int s, int d) { return ld_acquire_sys_s32(M + s * kMaxWorld + d); };
        int acc = 0;
        for (int d = 0; d < G; ++d) {
            plan->send_start[d] = acc;
            acc += m(me, d);
        }
        plan->send_start[G] = acc;
        for (int d = 0; d < G; ++d) {
            int64_t o = 0;
            for (int s = 0; s < me; ++s) o += m(s, d);
            plan->dst_offset[d] = o;
        }
        acc = 0;
        for (int s = 0; s < G; ++s) {
            plan->recv_start[s] = acc;
            acc += m(s, me);
            int b = 0;
            for (int d = 0; d < me; ++d) b += m(s, d);
            plan->back_start[s] = b;
        }
        plan->recv_start[G] = acc;
        plan->n_recv = acc;
    }
}

// Received row r (source s's j-th row for me) returns to source s's return
// buffer at row back_start[s] + j.  comm off (timing reference): the rows stay
// in this rank's own return buffer at the same positions.
__global__ void ep_row_dst_kernel(const EpPlan* __restrict__ plan,
                                  const unsigned long long* __restrict__ peer_base, size_t off_back,
                                  int G, int me, int comm, size_t row_bytes, int cap,
                                  uint64_t* __restrict__ row_dst) {
    const int n = min(plan->n_recv, cap);
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        int s = 0;
        while (s + 1 < G && plan->recv_start[s + 1] <= r) ++s;
        const int j = r - plan->recv_start[s];
        const unsigned long long base = peer_base[comm ? s : me] + off_back;
        row_dst[r] = base + (uint64_t)(plan->back_start[s] + j) * row_bytes;
    }
}

// comm off (timing reference): no dispatch; the received rows' expert ids are
// spread over the local experts like a balanced router's would be.
__global__ void ep_fake_recv_kernel(const EpPlan* __restrict__ plan, int first, int n_local, int cap,
                                    int* __restrict__ recv_exp) {
    const int n = min(plan->n_recv, cap);
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        recv_exp[r] = first + r % n_local;
}

// The receive count, clamped to the buffer (overflow is latched by the dispatch).
__global__ void ep_recv_count_kernel(const EpPlan* __restrict__ plan, int cap,
                                     int* __restrict__ n_out, int* __restrict__ dev_status) {
    const int n = plan->n_recv;
    if (n > cap) atomicExch(dev_status, DEV_ERR_CAPACITY);
    *n_out = min(n, cap);
}

// Controller: move this rank's counters (and its tokens_seen) into the
// all-reduce buffer and reset them.
__global__ void ep_pack_counters_kernel(unsigned long long* __restrict__ routed, int E,
                                        unsigned long long seen, unsigned long long* __restrict__ buf) {
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
        buf[i] = routed[i];
        routed[i] = 0;
    }
    if (threadIdx.x == 0) buf[E] = seen;
}

struct EpSet {
    void* slab = nullptr;                       // cudaMalloc'd, IPC-exported
    unsigned long long* peer_base_dev = nullptr;  // [G] slab base of every rank (mine included)
    uint64_t* peer_recv_dev = nullptr;          // [G] receive-row buffer of every rank
    uint64_t* peer_exp_dev = nullptr;           // [G] receive expert-id buffer of every rank
    std::vector<void*> peer_base;               // host copies
    std::vector<int> opened;                    // 1 = cudaIpcOpenMemHandle'd (closed on destroy)
    unsigned long long epoch[kChannels] = {0, 0, 0};
    // per-call state that lives until the back half of the call
    EpPlan* plan = nullptr;
    int* counts = nullptr;       // [G] my slot count per destination
    int* n_recv = nullptr;       // clamped receive count
    uint64_t* row_dst = nullptr; // [cap_recv]
    float* hmoe = nullptr;       // [cap_tok, d]
    __nv_bfloat16* hb = nullptr; // [cap_tok, d]
    int* slot_pos = nullptr;     // [cap_tok * K] position in my send order (-1 zero expert)
    int* send_token = nullptr;   // [cap_tok * K]
    int* send_expert = nullptr;  // [cap_tok * K]
    float* dd = nullptr;         // [cap_tok, d] dense-branch output (the combine's residual)
};

}  // namespace

struct scmoe_ep {
    scmoe_ctx* ctx = nullptr;    // the caller's context (front half, serial calls)
    scmoe_ctx* ctx_b = nullptr;  // back half of the pipelined schedule (own workspace)
    scmoe_ctx* ctx_d = nullptr;  // dense shortcut branch (own workspace and stream)
    int* saved_status[2] = {nullptr, nullptr};
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
    size_t d = 0, n_ffn = 0, n_zero = 0, K = 0, n_local = 0, first = 0;
    size_t cap_tok = 0, cap_recv = 0, cap_send = 0;
    SlabLayout lay{};
    EpSet sets[kSets];
    bool comm_on = true;
    int reserve_sms = 16;
    unsigned long long* ctrl = nullptr;  // [E + 1] controller all-reduce buffer
    double* delta = nullptr;             // [E]
    cudaStream_t s_front = nullptr, s_back = nullptr;
    cudaEvent_t ev_front[kSets] = {}, ev_back[kSets] = {}, ev_join = nullptr, ev_in = nullptr,
                ev_dense = nullptr;
    int last_set = 0;  // buffer set of the most recent call (its count matrix: stats)
};

namespace {

template <typename F>
int ep_guarded(scmoe_ep* ep, F&& f) {
    scmoe_ctx* c = ep ? ep->ctx : nullptr;
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

// Call a C-ABI entry point from inside the implementation; rethrow its status.
void chk(scmoe_ctx* c, int rc) {
    if (rc != SCMOE_OK) throw ScmoeError{rc, c->last_error};
}

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    SCMOE_CUDA(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
    return static_cast<T*>(p);
}

SlabLayout make_layout(size_t d, size_t cap_recv, size_t cap_send) {
    SlabLayout l{};
    size_t o = 0;
    l.counts = o;
    o = align_up(o + kMaxWorld * kMaxWorld * sizeof(int), 256);
    l.flags = o;
    o = align_up(o + kChannels * kMaxWorld * sizeof(unsigned long long), 1024);
    l.recv = o;
    o = align_up(o + cap_recv * d * 2, 1024);
    l.recv_exp = o;
    o = align_up(o + cap_recv * sizeof(int), 1024);
    l.back = o;
    o = align_up(o + cap_send * d * 2, 1024);
    l.bytes = o;
    return l;
}

void signal_wait(scmoe_ep* ep, scmoe_ctx* c, EpSet& st, int ch, const int* my_counts,
                 EpPlan* plan) {
    const unsigned long long epoch = ++st.epoch[ch];
    ep_signal_wait_kernel<<<1, 32, 0, c->stream>>>(st.peer_base_dev, ep->lay, ch, epoch, ep->rank,
                                                   ep->world, my_counts, plan, c->dev_status);
    SCMOE_LAUNCH_CHECK(c);
}

// Front half: route, plan, count exchange, dispatch, barrier.  On c's stream.
void ep_front(scmoe_ep* ep, scmoe_ctx* c, EpSet& st, scmoe_router* r, const float* a1,
              const float* gain, size_t T, uint32_t* idx, double* gates, uint32_t* cnt) {
    const int G = ep->world;
    chk(c, scmoe_rmsnorm_route(c, r, a1, gain, T, st.hmoe, st.hb, idx, gates, cnt));
    chk(c, scmoe_ep_plan(c, idx, T, ep->K, ep->n_ffn, ep->n_zero, G, st.counts, st.slot_pos,
                         st.send_token, st.send_expert));
    {
        ProfScope _p(c, "ep_exchange");
        signal_wait(ep, c, st, 0, st.counts, st.plan);
    }
    if (ep->comm_on) {
        ProfScope _p(c, "ep_put_rows");
        launch_ep_put_rows(c, st.hb, ep->d, st.send_token, st.send_expert, T * ep->K,
                           st.plan->send_start, st.plan->dst_offset, st.peer_recv_dev,
                           st.peer_exp_dev, G, (int64_t)ep->cap_recv);
    } else {
        ep_fake_recv_kernel<<<c->num_sms, 256, 0, c->stream>>>(
            st.plan, (int)ep->first, (int)ep->n_local, (int)ep->cap_recv,
            reinterpret_cast<int*>(static_cast<char*>(st.slab) + ep->lay.recv_exp));
        SCMOE_LAUNCH_CHECK(c);
    }
    ProfScope _p(c, "ep_dispatch_barrier");
    signal_wait(ep, c, st, 1, nullptr, nullptr);
}

// Back half: expert GEMMs on the received rows (GEMM2 rows to the sources),
// barrier, combine.  On c's stream.
void ep_back(scmoe_ep* ep, scmoe_ctx* c, EpSet& st, scmoe_bank* bank, size_t T, const uint32_t* idx,
             const double* gates, int renorm, const float* residual, float* out) {
    char* slab = static_cast<char*>(st.slab);
    {
        ProfScope _p(c, "ep_row_dst");
        ep_recv_count_kernel<<<1, 1, 0, c->stream>>>(st.plan, (int)ep->cap_recv, st.n_recv,
                                                     c->dev_status);
        SCMOE_LAUNCH_CHECK(c);
        ep_row_dst_kernel<<<c->num_sms, 256, 0, c->stream>>>(
            st.plan, st.peer_base_dev, ep->lay.back, ep->world, ep->rank, ep->comm_on ? 1 : 0,
            ep->d * 2, (int)ep->cap_recv, st.row_dst);
        SCMOE_LAUNCH_CHECK(c);
    }
    moe_rows_impl(c, bank, slab + ep->lay.recv,
                  reinterpret_cast<const int*>(slab + ep->lay.recv_exp), (int)ep->first,
                  ep->cap_recv, nullptr, st.row_dst, st.n_recv);
    {
        ProfScope _p(c, "ep_return_barrier");
        signal_wait(ep, c, st, 2, nullptr, nullptr);
    }
    if (T == 0) return;
    ProfScope _p(c, "combine");
    launch_combine_bf16(c, st.hmoe, reinterpret_cast<const __nv_bfloat16*>(slab + ep->lay.back),
                        idx, gates, st.slot_pos, T, ep->d, ep->K, ep->n_ffn,
                        (float)bank->gamma_ffn(), (float)bank->gamma_zero(), renorm, residual, out);
}

void check_ep_args(scmoe_ep* ep, scmoe_router* r, scmoe_bank* bank, size_t T) {
    SCMOE_CHECK_ARG(ep && r && bank, SCMOE_ERR_PARAMETER, "ep: null handle");
    if (r->d != ep->d || bank->d != ep->d)
        SCMOE_THROW(SCMOE_ERR_DIMENSION, "ep: router/bank width mismatch");
    if (r->n_ffn != ep->n_ffn || r->n_zero != ep->n_zero || r->top_k != ep->K)
        SCMOE_THROW(SCMOE_ERR_CONFIG, "ep: router does not match the layer");
    if (bank->n != ep->n_local || bank->precision != SCMOE_PREC_BF16)
        SCMOE_THROW(SCMOE_ERR_CONFIG, "ep: bank must hold this rank's n_ffn/world bf16 experts");
    if (T > ep->cap_tok) SCMOE_THROW(SCMOE_ERR_DIMENSION, "ep: more tokens than max_tokens");
}

scmoe_ctx* make_internal_ctx(scmoe_ep* ep, int slot) {
    scmoe_ctx* c = nullptr;
    chk(ep->ctx, scmoe_ctx_create(ep->device, &c));
    // device-side errors of the internal contexts latch into the caller's status
    ep->saved_status[slot] = c->dev_status;
    c->dev_status = ep->ctx->dev_status;
    c->gemm1_gather = ep->ctx->gemm1_gather;
    return c;
}

void destroy_internal_ctx(scmoe_ep* ep, scmoe_ctx*& c, int slot) {
    if (!c) return;
    c->dev_status = ep->saved_status[slot];
    scmoe_ctx_destroy(c);
    c = nullptr;
}

}  // namespace

extern "C" {

int scmoe_ep_unique_id(void* out) {
    try {
        if (!out) return SCMOE_ERR_PARAMETER;
        ncclUniqueId id;
        if (nccl().getUniqueId(&id) != ncclSuccess) return SCMOE_ERR_CUDA;
        std::memcpy(out, &id, sizeof(id));
        return SCMOE_OK;
    } catch (...) {
        return SCMOE_ERR_INTERNAL;
    }
}

size_t scmoe_ep_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

int scmoe_ep_create(scmoe_ctx* c, int world, int rank, const void* nccl_id, size_t d_model,
                    size_t n_ffn, size_t n_zero, size_t top_k, size_t max_tokens,
                    size_t max_recv_rows, scmoe_ep** out) {
    auto* ep = new scmoe_ep();
    ep->ctx = c;
    const int rc = ep_guarded(ep, [&] {
        SCMOE_CHECK_ARG(c && out && nccl_id, SCMOE_ERR_PARAMETER, "ep_create: null argument");
        SCMOE_CUDA(cudaSetDevice(c->device));
        if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
            SCMOE_THROW(SCMOE_ERR_CONFIG, "ep: need 1 <= world <= 32 and 0 <= rank < world");
        if (n_ffn % (size_t)world != 0)
            SCMOE_THROW(SCMOE_ERR_CONFIG, "ep: world size must divide the FFN expert count");
        if (d_model % 64 != 0) SCMOE_THROW(SCMOE_ERR_DIMENSION, "ep: d_model must be a multiple of 64");
        if (top_k < 1 || top_k > 64) SCMOE_THROW(SCMOE_ERR_CONFIG, "ep: top_k must be in [1, 64]");
        ep->world = world;
        ep->rank = rank;
        ep->device = c->device;
        ep->d = d_model;
        ep->n_ffn = n_ffn;
        ep->n_zero = n_zero;
        ep->K = top_k;
        ep->n_local = n_ffn / world;
        ep->first = (size_t)rank * ep->n_local;
        ep->cap_tok = std::max<size_t>(max_tokens, 1);
        ep->cap_send = ep->cap_tok * top_k;
        // worst case: every source's tokens each hit min(K, n_local) of my experts
        const size_t worst = (size_t)world * ep->cap_tok * std::min(top_k, ep->n_local);
        ep->cap_recv = max_recv_rows ? std::min(max_recv_rows, worst) : worst;
        ep->lay = make_layout(d_model, ep->cap_recv, ep->cap_send);
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        SCMOE_NCCL(nccl().commInitRank(&ep->comm, world, id, rank));
        // symmetric slabs: allocate, zero (flags start at epoch 0), export
        struct Exported {
            cudaIpcMemHandle_t h[kSets];
            unsigned long long ptr[kSets];
            long long pid;
            int device;
            int pad;
        };
        Exported mine{};
        for (int k = 0; k < kSets; ++k) {
            EpSet& st = ep->sets[k];
            SCMOE_CUDA(cudaMalloc(&st.slab, ep->lay.bytes));
            SCMOE_CUDA(cudaMemsetAsync(st.slab, 0, ep->lay.recv, c->stream));
            SCMOE_CUDA(cudaIpcGetMemHandle(&mine.h[k], st.slab));
            mine.ptr[k] = reinterpret_cast<unsigned long long>(st.slab);
        }
        mine.pid = (long long)getpid();
        mine.device = c->device;
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        Exported* xdev = dalloc<Exported>((size_t)world);
        SCMOE_CUDA(cudaMemcpyAsync(xdev + rank, &mine, sizeof(mine), cudaMemcpyHostToDevice,
                                   c->stream));
        SCMOE_NCCL(nccl().allGather(xdev + rank, xdev, sizeof(Exported), ncclChar, ep->comm,
                                 c->stream));
        std::vector<Exported> all(world);
        SCMOE_CUDA(cudaMemcpyAsync(all.data(), xdev, world * sizeof(Exported),
                                   cudaMemcpyDeviceToHost, c->stream));
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(xdev);
        for (int k = 0; k < kSets; ++k) {
            EpSet& st = ep->sets[k];
            st.peer_base.assign(world, nullptr);
            st.opened.assign(world, 0);
            for (int g = 0; g < world; ++g) {
                if (g == rank) {
                    st.peer_base[g] = st.slab;
                } else if (all[g].pid == mine.pid) {
                    // same process (one thread per GPU): plain peer access
                    const cudaError_t e = cudaDeviceEnablePeerAccess(all[g].device, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                        SCMOE_CUDA(e);
                    cudaGetLastError();
                    st.peer_base[g] = reinterpret_cast<void*>(all[g].ptr[k]);
                } else {
                    SCMOE_CUDA(cudaIpcOpenMemHandle(&st.peer_base[g], all[g].h[k],
                                                    cudaIpcMemLazyEnablePeerAccess));
                    st.opened[g] = 1;
                }
            }
            std::vector<unsigned long long> pb(world);
            std::vector<uint64_t> pr(world), pe(world);
            for (int g = 0; g < world; ++g) {
                pb[g] = reinterpret_cast<unsigned long long>(st.peer_base[g]);
                pr[g] = pb[g] + ep->lay.recv;
                pe[g] = pb[g] + ep->lay.recv_exp;
            }
            st.peer_base_dev = dalloc<unsigned long long>(world);
            st.peer_recv_dev = dalloc<uint64_t>(world);
            st.peer_exp_dev = dalloc<uint64_t>(world);
            SCMOE_CUDA(cudaMemcpy(st.peer_base_dev, pb.data(), world * 8, cudaMemcpyHostToDevice));
            SCMOE_CUDA(cudaMemcpy(st.peer_recv_dev, pr.data(), world * 8, cudaMemcpyHostToDevice));
            SCMOE_CUDA(cudaMemcpy(st.peer_exp_dev, pe.data(), world * 8, cudaMemcpyHostToDevice));
            st.plan = dalloc<EpPlan>(1);
            st.counts = dalloc<int>(world);
            st.n_recv = dalloc<int>(1);
            st.row_dst = dalloc<uint64_t>(ep->cap_recv);
            st.hmoe = dalloc<float>(ep->cap_tok * d_model);
            st.hb = dalloc<__nv_bfloat16>(ep->cap_tok * d_model);
            st.slot_pos = dalloc<int>(ep->cap_send);
            st.send_token = dalloc<int>(ep->cap_send);
            st.send_expert = dalloc<int>(ep->cap_send);
        }
        ep->ctrl = dalloc<unsigned long long>(n_ffn + n_zero + 1);
        ep->delta = dalloc<double>(n_ffn + n_zero);
        SCMOE_CUDA(cudaEventCreateWithFlags(&ep->ev_join, cudaEventDisableTiming));
        SCMOE_CUDA(cudaEventCreateWithFlags(&ep->ev_in, cudaEventDisableTiming));
        SCMOE_CUDA(cudaEventCreateWithFlags(&ep->ev_dense, cudaEventDisableTiming));
        for (int k = 0; k < kSets; ++k) {
            SCMOE_CUDA(cudaEventCreateWithFlags(&ep->ev_front[k], cudaEventDisableTiming));
            SCMOE_CUDA(cudaEventCreateWithFlags(&ep->ev_back[k], cudaEventDisableTiming));
        }
        SCMOE_CUDA(cudaStreamCreateWithFlags(&ep->s_front, cudaStreamNonBlocking));
        // every rank has mapped every slab before anyone stores into one
        SCMOE_NCCL(nccl().allReduce(ep->ctrl, ep->ctrl, 1, ncclUint64, ncclSum, ep->comm, c->stream));
        SCMOE_CUDA(cudaStreamSynchronize(c->stream));
        *out = ep;
    });
    if (rc != SCMOE_OK) {
        scmoe_ep_destroy(ep);
        if (out) *out = nullptr;
    }
    return rc;
}

int scmoe_ep_destroy(scmoe_ep* ep) {
    if (!ep) return SCMOE_OK;
    if (ep->ctx) {
        cudaSetDevice(ep->device);
        cudaStreamSynchronize(ep->ctx->stream);
    }
    cudaDeviceSynchronize();
    // no rank may unmap while a peer still stores into its slab
    if (ep->comm && ep->ctrl && ep->ctx) {
        nccl().allReduce(ep->ctrl, ep->ctrl, 1, ncclUint64, ncclSum, ep->comm, ep->ctx->stream);
        cudaStreamSynchronize(ep->ctx->stream);
    }
    for (auto& st : ep->sets) {
        for (size_t g = 0; g < st.opened.size(); ++g)
            if (st.opened[g]) cudaIpcCloseMemHandle(st.peer_base[g]);
        for (void* p : {(void*)st.peer_base_dev, (void*)st.peer_recv_dev, (void*)st.peer_exp_dev,
                        (void*)st.plan, (void*)st.counts, (void*)st.n_recv, (void*)st.row_dst,
                        (void*)st.hmoe, (void*)st.hb, (void*)st.slot_pos, (void*)st.send_token,
                        (void*)st.send_expert, (void*)st.dd, st.slab})
            if (p) cudaFree(p);
    }
    if (ep->ctrl) cudaFree(ep->ctrl);
    if (ep->delta) cudaFree(ep->delta);
    for (int k = 0; k < kSets; ++k) {
        if (ep->ev_front[k]) cudaEventDestroy(ep->ev_front[k]);
        if (ep->ev_back[k]) cudaEventDestroy(ep->ev_back[k]);
    }
    for (cudaEvent_t e : {ep->ev_join, ep->ev_in, ep->ev_dense})
        if (e) cudaEventDestroy(e);
    if (ep->s_front) cudaStreamDestroy(ep->s_front);
    destroy_internal_ctx(ep, ep->ctx_b, 0);
    destroy_internal_ctx(ep, ep->ctx_d, 1);
    if (ep->comm) nccl().commDestroy(ep->comm);
    delete ep;
    return SCMOE_OK;
}

int scmoe_ep_set_comm(scmoe_ep* ep, int on) {
    return ep_guarded(ep, [&] {
        SCMOE_CHECK_ARG(ep, SCMOE_ERR_PARAMETER, "null ep");
        ep->comm_on = on != 0;
    });
}

int scmoe_ep_set_dense_reserve(scmoe_ep* ep, int reserve_sms) {
    return ep_guarded(ep, [&] {
        SCMOE_CHECK_ARG(ep && reserve_sms >= 0, SCMOE_ERR_PARAMETER, "ep: bad reserve");
        ep->reserve_sms = reserve_sms;
        if (ep->ctx_d)
            ep->ctx_d->gemm_sms = std::max(1, ep->ctx_d->num_sms - reserve_sms);
    });
}

size_t scmoe_ep_capacity_rows(const scmoe_ep* ep) { return ep ? ep->cap_recv : 0; }

uint64_t scmoe_ep_kernel_launches(const scmoe_ep* ep) {
    if (!ep) return 0;
    return (ep->ctx ? ep->ctx->launches : 0) + (ep->ctx_b ? ep->ctx_b->launches : 0) +
           (ep->ctx_d ? ep->ctx_d->launches : 0);
}

int scmoe_ep_layer_forward(scmoe_ep* ep, scmoe_router* r, scmoe_bank* bank, scmoe_bank* dense,
                           const float* a1, const float* a3, const float* gain, size_t T,
                           int renorm, uint32_t* idx, double* gates, uint32_t* cnt, float* out) {
    return ep_guarded(ep, [&] {
        check_ep_args(ep, r, bank, T);
        scmoe_ctx* c = ep->ctx;
        SCMOE_CUDA(cudaSetDevice(c->device));
        EpSet& st = ep->sets[0];
        ep->last_set = 0;
        const float* residual = a3;
        if (dense) {
            // the ScMoE overlap window: dd = a1 + ffn(rmsnorm(a1)) on its own
            // stream and SMs, beside routing, dispatch, expert GEMMs and return
            if (!ep->ctx_d) {
                ep->ctx_d = make_internal_ctx(ep, 1);
                ep->ctx_d->gemm_sms = std::max(1, ep->ctx_d->num_sms - ep->reserve_sms);
            }
            if (!st.dd) st.dd = dalloc<float>(ep->cap_tok * ep->d);
            SCMOE_CUDA(cudaEventRecord(ep->ev_in, c->stream));
            SCMOE_CUDA(cudaStreamWaitEvent(ep->ctx_d->stream, ep->ev_in, 0));
            chk(ep->ctx_d, scmoe_dense_ffn(ep->ctx_d, dense, a1, gain, T, st.dd));
            SCMOE_CUDA(cudaEventRecord(ep->ev_dense, ep->ctx_d->stream));
            residual = st.dd;
        }
        ep_front(ep, c, st, r, a1, gain, T, idx, gates, cnt);
        if (dense) SCMOE_CUDA(cudaStreamWaitEvent(c->stream, ep->ev_dense, 0));
        ep_back(ep, c, st, bank, T, idx, gates, renorm, residual, out);
    });
}

int scmoe_ep_layer_forward_batches(scmoe_ep* ep, scmoe_router* r, scmoe_bank* bank,
                                   size_t n_batches, const float* const* a1,
                                   const float* const* a3, const float* gain, size_t T,
                                   int renorm, int corun_router, uint32_t* const* idx,
                                   double* const* gates, uint32_t* const* cnt,
                                   float* const* out) {
    return ep_guarded(ep, [&] {
        check_ep_args(ep, r, bank, T);
        scmoe_ctx* c = ep->ctx;
        SCMOE_CUDA(cudaSetDevice(c->device));
        if (n_batches == 0) return;
        if (!ep->ctx_b) ep->ctx_b = make_internal_ctx(ep, 0);
        scmoe_ctx* cb = ep->ctx_b;
        cudaStream_t user = c->stream;
        SCMOE_CUDA(cudaEventRecord(ep->ev_join, user));
        SCMOE_CUDA(cudaStreamWaitEvent(ep->s_front, ep->ev_join, 0));
        SCMOE_CUDA(cudaStreamWaitEvent(cb->stream, ep->ev_join, 0));
        struct Restore {
            scmoe_ctx* c;
            cudaStream_t s;
            bool ov;
            ~Restore() {
                c->stream = s;
                c->overlapped = ov;
            }
        } restore{c, user, c->overlapped};
        c->stream = ep->s_front;
        c->overlapped = corun_router != 0;
        // co-residency needs both sides small: the router kernel (front) and the
        // grouped GEMM's ring (back)
        struct RestoreB {
            scmoe_ctx* c;
            ~RestoreB() { c->corun_gemm = false; }
        } restore_b{cb};
        cb->corun_gemm = corun_router != 0;
        for (size_t i = 0; i < n_batches; ++i) {
            const int k = (int)(i & 1);
            EpSet& st = ep->sets[k];
            // front(i) reuses set k of batch i-2: its back half must be done
            if (i >= 2) SCMOE_CUDA(cudaStreamWaitEvent(ep->s_front, ep->ev_back[k], 0));
            ep_front(ep, c, st, r, a1[i], gain, T, idx[i], gates[i], cnt[i]);
            SCMOE_CUDA(cudaEventRecord(ep->ev_front[k], ep->s_front));
            SCMOE_CUDA(cudaStreamWaitEvent(cb->stream, ep->ev_front[k], 0));
            ep_back(ep, cb, st, bank, T, idx[i], gates[i], renorm, a3 ? a3[i] : nullptr, out[i]);
            SCMOE_CUDA(cudaEventRecord(ep->ev_back[k], cb->stream));
            ep->last_set = k;
        }
        SCMOE_CUDA(cudaStreamWaitEvent(user, ep->ev_back[(n_batches - 1) & 1], 0));
        SCMOE_CUDA(cudaStreamWaitEvent(user, ep->ev_front[(n_batches - 1) & 1], 0));
    });
}

int scmoe_ep_controller_step(scmoe_ep* ep, scmoe_router* r, const uint32_t* idx, size_t T,
                             int update, double* delta) {
    return ep_guarded(ep, [&] {
        SCMOE_CHECK_ARG(ep && r, SCMOE_ERR_PARAMETER, "ep: null handle");
        scmoe_ctx* c = ep->ctx;
        SCMOE_CUDA(cudaSetDevice(c->device));
        chk(c, scmoe_accumulate_counters(c, r, idx, T));  // accumulate_counters, local slots
        if (!update) return;
        const size_t E = r->E();
        ProfScope _p(c, "ep_controller");
        ep_pack_counters_kernel<<<1, 256, 0, c->stream>>>(
            reinterpret_cast<unsigned long long*>(r->routed), (int)E,
            (unsigned long long)r->tokens_seen, ep->ctrl);
        SCMOE_LAUNCH_CHECK(c);
        // the global batch (router.hpp:158-169): exact integer sums, order-free
        SCMOE_NCCL(nccl().allReduce(ep->ctrl, ep->ctrl, E + 1, ncclUint64, ncclSum, ep->comm,
                                 c->stream));
        launch_bias_update(c, r, ep->delta, reinterpret_cast<const uint64_t*>(ep->ctrl),
                           reinterpret_cast<const uint64_t*>(ep->ctrl + E));
        r->mu *= r->mu_decay;  // router.hpp:172
        r->tokens_seen = 0;
        if (delta) {
            SCMOE_CUDA(cudaMemcpyAsync(delta, ep->delta, E * sizeof(double), cudaMemcpyDeviceToHost,
                                       c->stream));
            chk(c, scmoe_synchronize(c));
        }
    });
}

int scmoe_ep_count_matrix_host(scmoe_ep* ep, int* matrix) {
    return ep_guarded(ep, [&] {
        SCMOE_CHECK_ARG(ep && matrix, SCMOE_ERR_PARAMETER, "ep: null argument");
        scmoe_ctx* c = ep->ctx;
        SCMOE_CUDA(cudaSetDevice(c->device));
        SCMOE_CUDA(cudaDeviceSynchronize());
        std::vector<int> m(kMaxWorld * kMaxWorld);
        SCMOE_CUDA(cudaMemcpy(m.data(), static_cast<char*>(ep->sets[ep->last_set].slab) + ep->lay.counts,
                              m.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int s = 0; s < ep->world; ++s)
            for (int d = 0; d < ep->world; ++d) matrix[s * ep->world + d] = m[s * kMaxWorld + d];
    });
}

}  // extern "C"
