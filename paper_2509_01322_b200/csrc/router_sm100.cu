// router_sm100.cu -- the router projection logits = x W_r (router.hpp:136) for
// large batches, fed by TMA.  Compiled on its own with --fmad=false and
// ptxas -O1: at -O2/-O3 ptxas software-pipelines the weight loads of the k
// loop and pays ~13 register moves per 84 packed FP32 instructions at the
// loop back-edge (the loop is FP32-pipe bound, so those moves cost ~8%);
// -O1 emits the same loop without them and without spills.
#include <cuda.h>

#include "f32x2.cuh"
#include "internal.cuh"
#include "sm100_util.cuh"

namespace scmoe {

// ---------------------------------------------------------------------------
// Router projection, TMA-fed slab (the default for large batches).  CTA tile
// = 56 tokens x all E <= 768 experts, 512 threads = 8 token groups x 64
// expert groups, 7 x 12 independent f32x2 chains per thread (84 accumulator
// registers: with 4 warps per SM sub-partition each thread may hold 128
// registers, so nothing spills -- the 768-thread slab kernel is capped at 80
// and spills in its inner loop).  Thread eg owns expert quads 4eg, 256+4eg,
// 512+4eg: each warp's weight loads are three conflict-free 512-byte rows.
// The operands arrive by TMA into a 4-stage ring guarded by mbarriers:
//   stage = W chunk [3 boxes][16 k][256 experts] (48 KB) + X chunk
//           [56 tokens][16 k] (3.5 KB, rows past T zero-filled by TMA).
// Thread 0 refills the stage of chunk c-2 at the top of chunk c (two chunks
// of slack for laggard warps); each warp arrives on a stage's empty barrier
// when done with it, so compute warps never meet at a CTA-wide barrier.
// Tokens are read as warp-broadcast scalars straight from the X rows (no
// transpose).  Arithmetic identical to seq_gemm_kernel: c = 0; c = c + x*w in
// k order, every product and sum rounded (f32x2 scheme as router_slab_kernel).
// ---------------------------------------------------------------------------
constexpr int kRtTok = 7, kRtExp = 12, kRtTG = 8, kRtEG = 64;
constexpr int kRtRows = kRtTok * kRtTG;                      // 56
constexpr int kRtThreads = kRtTG * kRtEG;                    // 512
constexpr int kRtKC = 16;
constexpr int kRtStages = 4;
constexpr int kRtBox = 256;                                  // experts per W box
constexpr int kRtW = 768;                                    // padded expert width
constexpr int kRtWFloats = kRtKC * kRtW;                     // 12288
constexpr int kRtXFloats = kRtRows * kRtKC;                  // 896
constexpr int kRtStageFloats = kRtWFloats + kRtXFloats;
constexpr int kRtStageBytes = kRtStageFloats * 4;            // 52736 (128-byte multiple)
static_assert(kRtStageBytes % 128 == 0, "TMA destinations must stay 128-byte aligned");
constexpr int kRtWarps = kRtThreads / 32;                    // 16
constexpr size_t kRtSmem = (size_t)kRtStages * kRtStageBytes + 2 * kRtStages * 8 + 128;
static_assert(kRtEG * 4 == kRtBox && kRtExp / 4 == kRtW / kRtBox, "quad layout");

__global__ void __launch_bounds__(kRtThreads, 1) router_tma_kernel(
    const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
    float* __restrict__ logits, int T, int K, int E) {
    extern __shared__ __align__(128) float rt_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(rt_smem + kRtStages * kRtStageFloats);
    uint64_t* empty = full + kRtStages;
    const int tid = threadIdx.x;
    const int tg = tid / kRtEG, eg = tid % kRtEG;
    const int row0 = blockIdx.x * kRtRows;
    const int nchunks = K / kRtKC;
    if (tid == 0) {
        for (int s = 0; s < kRtStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kRtWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int s = c % kRtStages;
        float* st = rt_smem + s * kRtStageFloats;
        mbar_expect_tx(&full[s], kRtStageBytes);
#pragma unroll
        for (int b = 0; b < kRtW / kRtBox; ++b)
            tma_load_2d(&map_w, &full[s], st + b * kRtKC * kRtBox, b * kRtBox, c * kRtKC,
                        policy_evict_last());
        tma_load_2d(&map_x, &full[s], st + kRtWFloats, c * kRtKC, row0, policy_evict_first());
    };
    if (tid == 0)
        for (int c = 0; c < kRtStages && c < nchunks; ++c) issue(c);

    const int wq = 4 * eg;                                    // quad offset inside each box
    const int xoff = kRtWFloats + kRtTok * tg * kRtKC;

    // acc[i][q] = (c[i][e+1], c[i][e]) for token i, expert pair e = column of pair q
    uint64_t acc[kRtTok][kRtExp / 2];
#pragma unroll
    for (int i = 0; i < kRtTok; ++i)
#pragma unroll
        for (int q = 0; q < kRtExp / 2; ++q) acc[i][q] = 0;

    for (int c = 0; c < nchunks; ++c) {
        const int s = c % kRtStages;
        if (tid == 0 && c >= 2 && c - 2 + kRtStages < nchunks) {
            mbar_wait(&empty[(c - 2) % kRtStages], ((c - 2) / kRtStages) & 1);
            issue(c - 2 + kRtStages);
        }
        mbar_wait(&full[s], (c / kRtStages) & 1);
        const float* st = rt_smem + s * kRtStageFloats;
#pragma unroll 2
        for (int k = 0; k < kRtKC; ++k) {
            uint64_t bv[kRtExp / 2];
#pragma unroll
            for (int b = 0; b < kRtExp / 4; ++b) {
                const ulonglong2 v =
                    *reinterpret_cast<const ulonglong2*>(st + b * kRtKC * kRtBox + k * kRtBox + wq);
                bv[2 * b] = v.x;
                bv[2 * b + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < kRtTok; ++i) {
                const float a = st[xoff + i * kRtKC + k];
#pragma unroll
                for (int q = 0; q < kRtExp / 2; ++q)
                    acc[i][q] = f2_add_swapped(acc[i][q], f2_mul_bcast(a, bv[q]));
            }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
    const int nrows = min(kRtRows, T - row0);
#pragma unroll
    for (int i = 0; i < kRtTok; ++i) {
        const int r = kRtTok * tg + i;
        if (r >= nrows) continue;
#pragma unroll
        for (int b = 0; b < kRtExp / 4; ++b) {
            const int col = b * kRtBox + wq;
            if (col >= E) continue;
            const uint64_t p0 = acc[i][2 * b], p1 = acc[i][2 * b + 1];
            *reinterpret_cast<float4*>(logits + (size_t)(row0 + r) * E + col) =
                make_float4(f2_hi(p0), f2_lo(p0), f2_hi(p1), f2_lo(p1));
        }
    }
}

// Persistent form, templated on the CTA shape, for a reduced SM budget or
// for running beside the grouped GEMM (scmoe_layer_forward_batches): this CTA
// takes slabs blockIdx.x, +gridDim.x, ... and the ring runs on one global
// chunk counter g = (local slab) * nchunks + c, so the next slab's first
// chunks stream in while the current one finishes.  TG token groups of 7
// (TG*64 threads), KC k-rows per stage, S stages; thread 0 refills the stage
// of chunk g-LAG at the top of chunk g.
//   <8, 16, 4, 2>: the full-SM tile of router_tma_kernel (206 KB smem);
//   <4, 4, 2, 1>:  256 threads x 128 registers, 25.5 KB smem -- fits next to
//                  one grouped-GEMM CTA (352 x 64 registers, 189 KB) per SM
//                  (and per SM sub-partition: 2 x 4096 + 3 x 2048 registers).
template <int TG, int KC, int S, int LAG>
__global__ void __launch_bounds__(TG * kRtEG, 512 / (TG * kRtEG)) router_tma_persistent_kernel(
    const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
    float* __restrict__ logits, int T, int K, int E) {
    constexpr int Rows = kRtTok * TG, Threads = TG * kRtEG, Warps = Threads / 32;
    // stages start 128-byte aligned (TMA destination requirement)
    constexpr int WFloats = KC * kRtW, StageFloats = (WFloats + Rows * KC + 31) / 32 * 32;
    constexpr uint32_t StageBytes = (WFloats + Rows * KC) * 4;  // bytes the TMAs deliver
    extern __shared__ __align__(128) float rt_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(rt_smem + S * StageFloats);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    const int tg = tid / kRtEG, eg = tid % kRtEG;
    const int nchunks = K / KC;
    const int nslabs = (T + Rows - 1) / Rows;
    const int my_slabs = blockIdx.x < nslabs ? (nslabs - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int G = my_slabs * nchunks;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], Warps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    }
    __syncthreads();
    auto issue = [&](int g) {
        const int s = g % S;
        const int c = g % nchunks;
        const int row0 = (blockIdx.x + (g / nchunks) * gridDim.x) * Rows;
        float* st = rt_smem + s * StageFloats;
        mbar_expect_tx(&full[s], StageBytes);
#pragma unroll
        for (int b = 0; b < kRtW / kRtBox; ++b)
            tma_load_2d(&map_w, &full[s], st + b * KC * kRtBox, b * kRtBox, c * KC,
                        policy_evict_last());
        tma_load_2d(&map_x, &full[s], st + WFloats, c * KC, row0, policy_evict_first());
    };
    if (tid == 0)
        for (int g = 0; g < S && g < G; ++g) issue(g);

    const int wq = 4 * eg;                                    // quad offset inside each box
    const int xoff = WFloats + kRtTok * tg * KC;

    for (int j = 0; j < my_slabs; ++j) {
        // acc[i][q] = (c[i][e+1], c[i][e]) for token i, expert pair e = column of pair q
        uint64_t acc[kRtTok][kRtExp / 2];
#pragma unroll
        for (int i = 0; i < kRtTok; ++i)
#pragma unroll
            for (int q = 0; q < kRtExp / 2; ++q) acc[i][q] = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int g = j * nchunks + c;
            const int s = g % S;
            if (tid == 0 && g >= LAG && g - LAG + S < G) {
                mbar_wait(&empty[(g - LAG) % S], ((g - LAG) / S) & 1);
                issue(g - LAG + S);
            }
            mbar_wait(&full[s], (g / S) & 1);
            const float* st = rt_smem + s * StageFloats;
#pragma unroll 2
            for (int k = 0; k < KC; ++k) {
                uint64_t bv[kRtExp / 2];
#pragma unroll
                for (int b = 0; b < kRtExp / 4; ++b) {
                    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(
                        st + b * KC * kRtBox + k * kRtBox + wq);
                    bv[2 * b] = v.x;
                    bv[2 * b + 1] = v.y;
                }
#pragma unroll
                for (int i = 0; i < kRtTok; ++i) {
                    const float a = st[xoff + i * KC + k];
#pragma unroll
                    for (int q = 0; q < kRtExp / 2; ++q)
                        acc[i][q] = f2_add_swapped(acc[i][q], f2_mul_bcast(a, bv[q]));
                }
            }
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[s]);
        }
        const int row0 = (blockIdx.x + j * gridDim.x) * Rows;
        const int nrows = min(Rows, T - row0);
#pragma unroll
        for (int i = 0; i < kRtTok; ++i) {
            const int r = kRtTok * tg + i;
            if (r >= nrows) continue;
#pragma unroll
            for (int b = 0; b < kRtExp / 4; ++b) {
                const int col = b * kRtBox + wq;
                if (col >= E) continue;
                const uint64_t p0 = acc[i][2 * b], p1 = acc[i][2 * b + 1];
                *reinterpret_cast<float4*>(logits + (size_t)(row0 + r) * E + col) =
                    make_float4(f2_hi(p0), f2_lo(p0), f2_hi(p1), f2_lo(p1));
            }
        }
    }
}

template <int TG, int KC, int S, int LAG>
static void launch_persistent(scmoe_ctx* c, const float* X, const float* W, float* logits,
                              size_t T, size_t K, size_t E, int ctas) {
    constexpr int Rows = kRtTok * TG;
    constexpr size_t Smem = (size_t)S * ((KC * kRtW + Rows * KC + 31) / 32 * 32) * 4 + 2 * S * 8 + 128;
    auto kern = router_tma_persistent_kernel<TG, KC, S, LAG>;
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(kern), (int)Smem, c->device);
    const CUtensorMap mw = make_tma_map_2d(W, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, sizeof(float), K, E,
                                           KC, kRtBox, CU_TENSOR_MAP_SWIZZLE_NONE);
    const CUtensorMap mx = make_tma_map_2d(X, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, sizeof(float), T, K,
                                           Rows, KC, CU_TENSOR_MAP_SWIZZLE_NONE);
    const size_t slabs = ceil_div(T, Rows);
    kern<<<(unsigned)std::min<size_t>(slabs, (size_t)ctas), TG * kRtEG, Smem, c->stream>>>(
        mw, mx, logits, (int)T, (int)K, (int)E);
    SCMOE_LAUNCH_CHECK(c);
}

bool router_tma_ok(size_t T, size_t K, size_t E, int num_sms) {
    // TMA rows need 16-byte strides (E, K multiples of 4); K in 16-row chunks;
    // enough 56-token slabs to fill most SMs
    return E <= (size_t)kRtW && E % 4 == 0 && K % kRtKC == 0 &&
           ceil_div(T, kRtRows) >= (size_t)num_sms * 3 / 4;
}

void launch_router_tma(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                       size_t K, size_t E) {
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(router_tma_kernel), (int)kRtSmem,
                            c->device);
    const CUtensorMap mw = make_tma_map_2d(W, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, sizeof(float), K, E,
                                           kRtKC, kRtBox, CU_TENSOR_MAP_SWIZZLE_NONE);
    const CUtensorMap mx = make_tma_map_2d(X, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, sizeof(float), T, K,
                                           kRtRows, kRtKC, CU_TENSOR_MAP_SWIZZLE_NONE);
    const size_t slabs = ceil_div(T, kRtRows);
    if (c->router_sms > 0 && (size_t)c->router_sms < slabs) {
        launch_persistent<8, 16, 4, 2>(c, X, W, logits, T, K, E, c->router_sms);
        return;
    }
    router_tma_kernel<<<slabs, kRtThreads, kRtSmem, c->stream>>>(mw, mx, logits, (int)T, (int)K,
                                                                 (int)E);
    SCMOE_LAUNCH_CHECK(c);
}

bool router_corun_ok(size_t T, size_t K, size_t E) {
    return E <= (size_t)kRtW && E % 4 == 0 && K % 4 == 0 && T > 0;
}

// The small-footprint tile (256 threads, 38 KB) on at most one CTA per SM, so
// it co-resides with the persistent grouped GEMM of the previous batch.
void launch_router_corun(scmoe_ctx* c, const float* X, const float* W, float* logits, size_t T,
                         size_t K, size_t E) {
    static const int stages = getenv("SCMOE_CORUN_STAGES") ? atoi(getenv("SCMOE_CORUN_STAGES")) : 2;
    const int ctas = c->router_sms > 0 ? c->router_sms : c->num_sms;
    // SCMOE_CORUN_STAGES: 2 (default) <4,4,2,1> 25 KB; 3 <4,4,3,1> 37 KB;
    // 4 <4,4,4,2> 50 KB; 8 <4,8,2,1> 50 KB; 9 <4,8,3,1> 74 KB
    switch (stages) {
        case 3: launch_persistent<4, 4, 3, 1>(c, X, W, logits, T, K, E, ctas); break;
        case 4: launch_persistent<4, 4, 4, 2>(c, X, W, logits, T, K, E, ctas); break;
        case 8: launch_persistent<4, 8, 2, 1>(c, X, W, logits, T, K, E, ctas); break;
        case 9: launch_persistent<4, 8, 3, 1>(c, X, W, logits, T, K, E, ctas); break;
        default: launch_persistent<4, 4, 2, 1>(c, X, W, logits, T, K, E, ctas); break;
    }
}

}  // namespace scmoe
