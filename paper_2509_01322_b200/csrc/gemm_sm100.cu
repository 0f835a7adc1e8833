// gemm_sm100.cu -- persistent, warp-specialised grouped GEMM on the 5th-gen
// tensor cores (tcgen05 + TMEM accumulators + TMA, sm_100a) for the expert
// FFN of the ScMoE layer (blocks.hpp:361-365: y = silu(x W_in) W_out).
//
// Orientation ("SwapAB", SURVEY.md 7 hard part 2): the expert weights are
// the MMA's M side and the tokens routed to the expert its N side,
//     D[m, j] = sum_k W[e][m][k] * X[pos0 + j][k]       (M = weight rows)
// so an expert with ~128 tokens fills one N=128 tile instead of padding a
// 128-row token tile.  W is stored K-major ([e][M][K] bf16: w_in^T for GEMM1,
// w_out^T for GEMM2) and X/H are token-major rows ([rows][K] bf16), so both
// operands are K-major 128-byte-swizzled TMA tiles.
//
// Work unit = (token tile of one expert, block of 256 weight rows).  Each
// CTA (one per SM, persistent) runs three roles:
//   warp 0      TMA producer: A (2 x 128-row weight slabs) + B (128 token
//               rows) per 64-wide K block into a 4-stage smem ring;
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma
//               (M=128, N=128, K=16) into two TMEM accumulators of 128
//               columns, double-buffered across units (4 x 128 = 512 cols);
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers, optional SiLU,
//               bf16 store of out[pos0 + j][m] (token-major rows again).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace scmoe {

namespace {

constexpr int BK = 64;          // K elements per stage (128 B rows, SWIZZLE_128B)
constexpr int SLABS = 2;        // 128-row weight slabs per unit (BM = 256)
constexpr int BM = 128 * SLABS;
constexpr int NT = 128;         // token columns per tile
constexpr int STAGES = 4;
constexpr int ACC_BUFS = 2;
constexpr int A_SLAB_BYTES = 128 * BK * 2;        // 16 KB
constexpr int B_BYTES = NT * BK * 2;              // 16 KB
constexpr int STAGE_BYTES = SLABS * A_SLAB_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;
constexpr int NUM_THREADS = 192;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

static_assert(ACC_BUFS * SLABS * NT <= TMEM_COLS, "TMEM overflow");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// K-major, 128B-swizzled UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major, 1), SBO>>4 [32,46)
// = 1024 B between 8-row groups, version [46,48) = 1, layout [61,64) = 2 (SW128).
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor, kind::f16: D f32 [4,6)=1, A bf16 [7,10)=1, B bf16
// [10,13)=1, both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float silu_fast(float v) { return __fdividef(v, 1.0f + __expf(-v)); }

struct GemmArgs {
    const TokenTile* tiles;
    const int* n_tiles;
    __nv_bfloat16* out;  // [rows][M]
    int M, K;            // weight rows per expert, reduction length
    int silu;
};

__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_w,
                        const __grid_constant__ CUtensorMap map_x, const GemmArgs args) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + ACC_BUFS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC_BUFS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int mblocks = args.M / BM;
    const int kblocks = args.K / BK;
    const int n_units = (*args.n_tiles) * mblocks;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < ACC_BUFS; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const TokenTile tile = args.tiles[u / mblocks];
                const int mb = u % mblocks;
                const int wrow = tile.e * args.M + mb * BM;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* sbase = smem + stage * STAGE_BYTES;
                    mbar_expect_tx(&full[stage], STAGE_BYTES);
#pragma unroll
                    for (int s = 0; s < SLABS; ++s)
                        tma_load_2d(&map_w, &full[stage], sbase + s * A_SLAB_BYTES, kb * BK,
                                    wrow + s * 128);
                    tma_load_2d(&map_x, &full[stage], sbase + SLABS * A_SLAB_BYTES, kb * BK,
                                tile.pos);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        constexpr uint32_t idesc = make_idesc(128, NT);
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++local) {
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d_base = tmem_base + acc * (SLABS * NT);
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint32_t sbase = smem_u32(smem + stage * STAGE_BYTES);
                    const uint32_t bbase = sbase + SLABS * A_SLAB_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t bdesc = make_desc_sw128(bbase + k * 32);
#pragma unroll
                        for (int s = 0; s < SLABS; ++s) {
                            const uint64_t adesc = make_desc_sw128(sbase + s * A_SLAB_BYTES + k * 32);
                            mma_bf16(d_base + s * NT, adesc, bdesc, idesc, (kb | k) != 0);
                        }
                    }
                    mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) mma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else {
        // ===== epilogue (warps 2..5) =====
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        int local = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++local) {
            const TokenTile tile = args.tiles[u / mblocks];
            const int mb = u % mblocks;
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tfull[acc], acc_phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int s = 0; s < SLABS; ++s) {
                const int m = mb * BM + s * 128 + quad * 32 + lane;
                const uint32_t taddr =
                    tmem_base + ((uint32_t)(quad * 32) << 16) + acc * (SLABS * NT) + s * NT;
                for (int j0 = 0; j0 < NT; j0 += 16) {
                    if (j0 >= tile.count) break;
                    uint32_t v[16];
                    tmem_ld16(taddr + j0, v);
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int j = j0 + jj;
                        if (j < tile.count) {
                            float f = __uint_as_float(v[jj]);
                            if (args.silu) f = silu_fast(f);
                            args.out[(size_t)(tile.pos + j) * args.M + m] = __float2bfloat16_rn(f);
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        SCMOE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            SCMOE_THROW(SCMOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

CUtensorMap make_map_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                        uint32_t box_cols) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * sizeof(__nv_bfloat16)};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) SCMOE_THROW(SCMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

}  // namespace

void launch_grouped_gemm_bf16(scmoe_ctx* c, const __nv_bfloat16* W, size_t n_experts, size_t M,
                              size_t K, const __nv_bfloat16* X, size_t x_rows,
                              __nv_bfloat16* out, int silu, const TokenTile* tiles,
                              const int* n_tiles_dev, size_t max_tiles, int tile_rows) {
    if (max_tiles == 0 || n_experts == 0) return;
    SCMOE_CHECK_ARG(tile_rows == NT, SCMOE_ERR_INTERNAL, "gemm: tile rows must equal NT");
    SCMOE_CHECK_ARG(M % BM == 0 && K % BK == 0, SCMOE_ERR_DIMENSION,
                    "gemm: M must be a multiple of 256 and K of 64");
    const CUtensorMap mw = make_map_2d(W, n_experts * M, K, 128, BK);
    const CUtensorMap mx = make_map_2d(X, std::max<size_t>(x_rows, 1), K, NT, BK);
    static bool attr_set = false;
    if (!attr_set) {
        SCMOE_CUDA(cudaFuncSetAttribute(grouped_gemm_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr_set = true;
    }
    GemmArgs a;
    a.tiles = tiles;
    a.n_tiles = n_tiles_dev;
    a.out = out;
    a.M = (int)M;
    a.K = (int)K;
    a.silu = silu;
    const size_t units_max = max_tiles * (M / BM);
    const int grid = (int)std::min<size_t>(units_max, (size_t)c->num_sms);
    grouped_gemm_kernel<<<grid, NUM_THREADS, SMEM_BYTES, c->stream>>>(mw, mx, a);
    SCMOE_LAUNCH_CHECK(c);
}

}  // namespace scmoe
