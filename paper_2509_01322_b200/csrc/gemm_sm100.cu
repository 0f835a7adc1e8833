// gemm_sm100.cu -- persistent, warp-specialised grouped GEMM on the 5th-gen
// tensor cores (tcgen05 + TMEM accumulators + TMA, sm_100a) for the expert
// FFN of the ScMoE layer (blocks.hpp:361-365: y = silu(x W_in) W_out).
//
// Orientation ("SwapAB", SURVEY.md 7 hard part 2): the expert weights are
// the MMA's M side and the tokens routed to the expert its N side,
//     D[m, j] = sum_k W[e][m][k] * X[pos0 + j][k]       (M = weight rows)
// W is stored K-major ([e][M][K] bf16: w_in^T for GEMM1, w_out^T for GEMM2)
// and X/H are token-major rows ([rows][K] bf16), so both operands are
// K-major 128-byte-swizzled TMA tiles.
//
// A token tile holds up to NT=192 tokens of one expert, so at the LongCat
// prefill shape (98..163 tokens per expert) every expert's weights are
// streamed from HBM exactly once per GEMM.  The MMA's N is chosen per tile at
// run time (tokens rounded up to 16), so short tiles (decode: ~4 tokens per
// expert) issue N=16 MMAs and load only the token rows they use.  Weights are
// stored in a blocked layout (internal.cuh wblk_index) so every weight TMA box
// is one contiguous 16 KB read.
//
// Work unit = (token tile, block of 256 weight rows).  Each CTA (one per SM,
// persistent, static round-robin over units) runs four roles:
//   warp 0      weight producer: per 64-wide K block two 128-row slabs into a
//               4-stage ring (HBM stream, the bytes that must be in flight);
//   warp 2      token producer: the tile's token rows into a 3-stage ring
//               (64-row TMA boxes; or cp.async row gathers, SCMOE_GEMM1_GATHER);
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma
//               (M=128, N=16..192, K=16) into two TMEM accumulators (one per
//               weight slab);
//   warps 3-10  epilogue, one per (TMEM lane quadrant, slab): tcgen05.ld ->
//               registers, optional SiLU, bf16, per-warp smem transpose, 64-byte
//               token-row stores of out[pos0 + j][m].
// The accumulators are single-buffered (2 x 192 columns); while the epilogue
// drains them the producers keep streaming the next unit into free stages.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.cuh"
#include "sm100_util.cuh"

namespace scmoe {

namespace {

constexpr int BK = 64;          // K elements per stage (128 B rows, SWIZZLE_128B)
constexpr int SLABS = 2;        // 128-row weight slabs per unit (BM = 256)
constexpr int BM = 128 * SLABS;
constexpr int NT = 192;         // max token columns per tile
// Separate rings: weights come from HBM (deep ring, most bytes in flight),
// token rows from L2 (shallow ring).
constexpr int A_STAGES = 3;
constexpr int B_STAGES = 3;
constexpr int A_SLAB_BYTES = 128 * BK * 2;        // 16 KB
constexpr int B_HALF_BYTES = 128 * BK * 2;        // 16 KB per 128 token rows (first box)
constexpr int A_STAGE_BYTES = SLABS * A_SLAB_BYTES;   // 32 KB
constexpr int B_STAGE_BYTES = NT * BK * 2;            // 24 KB (up to NT tokens)
constexpr int RING_BYTES = A_STAGES * A_STAGE_BYTES + B_STAGES * B_STAGE_BYTES;  // 192 KB
constexpr int TMEM_COLS = 512;
constexpr int EPI_WARPS = 4 * SLABS;             // one per (TMEM lane quadrant, slab)
constexpr int EPI_WARP0 = 3;                     // warps 0: W producer, 1: MMA, 2: X producer
constexpr int NUM_THREADS = 32 * (EPI_WARP0 + EPI_WARPS);
constexpr int EPI_PITCH = BM * 2;                     // epilogue staging row (dense: TMA store box)
constexpr int EPI_STAGE_BYTES = 32 * EPI_PITCH;          // [32 tokens][256 rows] bf16
constexpr int SMEM_BYTES = RING_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_STAGE_BYTES;

static_assert(SLABS * NT <= TMEM_COLS, "TMEM overflow");

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

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Same load, no wait: the caller overlaps it and issues tcgen05.wait::ld.
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

__device__ __forceinline__ float silu_fast(float v) { return __fdividef(v, 1.0f + __expf(-v)); }

struct GemmArgs {
    const TokenTile* tiles;
    const int* n_tiles;
    const int* x_rows;   // gather mode: permuted row -> source row of X (nullptr: X is permuted)
    const __nv_bfloat16* x;  // X base (gather mode reads rows directly)
    __nv_bfloat16* out;  // [rows][M]
    // optional scattered output: permuted row p goes to row_dst[row_ids[p]]
    // (a full M-wide row, possibly in a peer GPU's memory over NVLink)
    const uint64_t* row_dst;
    const int* row_ids;
    int M, K;            // weight rows per expert, reduction length
    int tma_store;       // contiguous out: full 32-token chunks leave by one TMA tensor store
    int silu;
    // causal attention (mla_tc.cu): causal_rows = queries per group -> skip the
    // units whose weight rows (keys) all lie above the tile's last query;
    // causal_k -> a unit of weight rows (queries) [mb*BM, (mb+1)*BM) reduces
    // only over K blocks up to (mb+1)*BM (its probabilities vanish beyond)
    int causal_rows;
    int causal_k;
    int debug;           // timing / energy experiments only (pair kernel: 16 no MMAs,
                         // 32 no token loads): bit 0 skip epilogue stores,
                         // bit 1 skip the epilogue (release TMEM at once),
                         // bit 2 tile-major unit order, bit 3 weights always evict-first
};

__device__ __forceinline__ bool unit_skipped(const GemmArgs& a, const TokenTile& t, int mb,
                                             int bm) {
    if (!a.causal_rows) return false;
    return mb * bm > t.pos - t.e * a.causal_rows + t.count - 1;
}
__device__ __forceinline__ int unit_kblocks(const GemmArgs& a, int mb, int kblocks, int bm) {
    return a.causal_k ? min(kblocks, (mb + 1) * bm / BK) : kblocks;
}

// Unit u -> (token tile, 256-row weight block).  Units are expert-major:
// the tiles of one expert (TokenTile.pad = index in the expert << 16 | the
// expert's tile count) take consecutive units for each weight block, so the
// CTAs streaming the same expert weights run side by side and share them
// through L2 (an expert with 512 tokens has 3 tiles of <= 192).  pad = 0
// (row tiles) keeps the plain tile-major order.
__device__ __forceinline__ void unit_map(int u, int mblocks, const TokenTile* tiles, int& t,
                                         int& mb, int debug) {
    const int t0 = u / mblocks;
    const int g = (debug & 4) ? 0 : tiles[t0].pad;
    const int n = g & 0xffff;
    if (n <= 1) {
        t = t0;
        mb = u % mblocks;
        return;
    }
    const int first = t0 - (g >> 16);
    const int local = u - first * mblocks;
    mb = local / n;
    t = first + local % n;
}

// epilogue staging buffers: two (chunk c+1 fills one while chunk c's bulk
// copies still read the other) where the shared memory allows -- the 256-token
// variant, which never shares the SM with the router
template <int kNT>
__host__ __device__ constexpr int gemm_epi_bufs() {
    return kNT == 256 ? 2 : 1;
}
template <int kNT, int kS = SLABS>
constexpr int gemm_smem_bytes() {
    return A_STAGES * kS * A_SLAB_BYTES + B_STAGES * kNT * BK * 2 + 1024 + 256 +
           gemm_epi_bufs<kNT>() * 32 * (128 * kS * 2);
}

// <= 64 registers: one GEMM CTA (352 threads) must leave room for the
// co-resident router CTA (256 x 128 registers) on every SM sub-partition.
// kNT = max tokens per tile: 192 (single-GPU prefill; 186 KB smem, fits next
// to the router) or 256 (expert-parallel shards with 256+ tokens per expert:
// one tile of 256 instead of two of 128, 210 KB smem, 2 x 256 TMEM columns).
// kS = 128-row weight slabs per unit: 2 (BM = 256; the accumulators of a
// 256-token tile fill TMEM, so they are single-buffered) or 1 (BM = 128: two
// 256-column accumulators, so the epilogue of unit i drains one while the
// MMAs of unit i+1 fill the other; 4 epilogue warps).
// Register cap: 64 so the 192-token variant co-resides with the router; the
// 256-token variant (expert-parallel shards, never next to the router) takes
// 128 and prefetches the next chunk's accumulators during the epilogue.
template <int kNT, int kS = SLABS>
__global__ void __maxnreg__(kNT == 256 ? 128 : 64)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_w,
                        const __grid_constant__ CUtensorMap map_x,
                        const __grid_constant__ CUtensorMap map_out, const GemmArgs args) {
    constexpr int NT = kNT;
    // unit geometry for this instantiation (shadows the namespace defaults)
    constexpr int SLABS = kS;
    constexpr int BM = 128 * kS;
    constexpr int A_STAGE_BYTES = kS * A_SLAB_BYTES;
    constexpr int EPI_WARPS = 4 * kS;
    constexpr int EPI_PITCH = BM * 2;
    constexpr int EPI_STAGE_BYTES = 32 * EPI_PITCH;
    constexpr int B_STAGE_BYTES = NT * BK * 2;
    constexpr int RING_BYTES = A_STAGES * A_STAGE_BYTES + B_STAGES * B_STAGE_BYTES;
    static_assert(SLABS * NT <= TMEM_COLS, "TMEM overflow");
    // accumulator buffers: two when both fit in TMEM (NT <= 128), so the
    // epilogue of unit i drains one while the MMAs of unit i+1 fill the other
    constexpr int ACC_COLS = SLABS * NT;
    constexpr int NBUF = 2 * ACC_COLS <= TMEM_COLS ? 2 : 1;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // smem: weight ring [A_STAGES][SLABS][16 KB] | token ring [B_STAGES][2][16 KB] |
    //       barriers | epilogue transpose buffers
    unsigned char* a_ring = smem;
    unsigned char* b_ring = smem + A_STAGES * A_STAGE_BYTES;
    uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + RING_BYTES);
    uint64_t* a_empty = a_full + A_STAGES;
    uint64_t* b_full = a_empty + A_STAGES;
    uint64_t* b_empty = b_full + B_STAGES;
    uint64_t* tfull = b_empty + B_STAGES;  // [NBUF]
    uint64_t* tempty = tfull + NBUF;        // [NBUF]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int mblocks = args.M / BM;
    const int kblocks = args.K / BK;
    const int n_units = (*args.n_tiles) * mblocks;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < A_STAGES; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < B_STAGES; ++s) {
            // gather mode: the 32 producer lanes each arrive once per stage
            mbar_init(&b_full[s], args.x_rows ? 32 : 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
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
        // ===== weight producer: streams W from HBM, A_STAGES deep =====
        if (lane == 0) {
            // weights are read once (evict-first) unless the expert has several
            // token tiles, whose units stream the same block side by side:
            // then keep it (evict-last) until the sibling CTAs have read it
            const uint64_t pol_once = policy_evict_first(), pol_shared = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                int ti, mb;
                unit_map(u, mblocks, args.tiles, ti, mb, args.debug);
                const TokenTile tile = args.tiles[ti];
                if (unit_skipped(args, tile, mb, BM)) continue;
                const int kb_end = unit_kblocks(args, mb, kblocks, BM);
                // blocked weight layout (wblk_index): each (128-row, 64-col) tile is
                // 128 contiguous 64-element rows of the 2-D view the map describes
                const int ebase = tile.e * (args.M / 128) * kblocks * 128;
                const uint64_t pol_w = (tile.pad & 0xffff) > 1 && !(args.debug & 8) ? pol_shared
                                                                                   : pol_once;
                for (int kb = 0; kb < kb_end; ++kb) {
                    mbar_wait(&a_empty[stage], phase ^ 1);
                    unsigned char* abase = a_ring + stage * A_STAGE_BYTES;
                    mbar_expect_tx(&a_full[stage], A_STAGE_BYTES);
#pragma unroll
                    for (int s = 0; s < SLABS; ++s)
                        tma_load_2d(&map_w, &a_full[stage], abase + s * A_SLAB_BYTES, 0,
                                    ebase + ((mb * SLABS + s) * kblocks + kb) * 128, pol_w);
                    if (++stage == A_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 2) {
        // ===== token producer: the tile's rows of X (L2-resident), B_STAGES
        // deep; lane 0 issues tiled boxes, or every lane issues row gathers =====
        const uint64_t pol_x = policy_evict_last();
        const bool gather = args.x_rows != nullptr;
        int stage = 0;
        uint32_t phase = 0;
        int pending = -1;  // gather mode: stage whose copies are in flight, not yet published
        constexpr int kRowsPerLane = (NT + 31) / 32;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int ti, mb_;
            unit_map(u, mblocks, args.tiles, ti, mb_, args.debug);
            const TokenTile tile = args.tiles[ti];
            if (unit_skipped(args, tile, mb_, BM)) continue;
            const int kb_end = unit_kblocks(args, mb_, kblocks, BM);
            const int n_eff = max(16, (tile.count + 15) & ~15);
            // gather mode: this lane's rows r = lane + 32 i (padding rows repeat
            // the tile's last token; their columns are never stored)
            const __nv_bfloat16* src[kRowsPerLane];
            if (gather) {
#pragma unroll
                for (int i = 0; i < kRowsPerLane; ++i) {
                    const int r = lane + 32 * i;
                    src[i] = r < n_eff ? args.x + (size_t)args.x_rows[tile.pos + min(r, tile.count - 1)] *
                                                      args.K
                                       : nullptr;
                }
            }
            // tiled mode: boxes of 64 rows, as many as the tile needs
            const int nbox = (n_eff + 63) / 64;
            for (int kb = 0; kb < kb_end; ++kb) {
                mbar_wait(&b_empty[stage], phase ^ 1);
                unsigned char* bbase = b_ring + stage * B_STAGE_BYTES;
                if (!gather) {
                    if (lane == 0) {
                        mbar_expect_tx(&b_full[stage], (uint32_t)nbox * 64 * BK * 2);
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_load_2d(&map_x, &b_full[stage], bbase + bx * 64 * BK * 2, kb * BK,
                                        tile.pos + 64 * bx, pol_x);
                    }
                } else {
                    // 16-byte cp.async per (row, chunk) into the 128B-swizzled
                    // K-major layout the UMMA descriptor expects: chunk c of row r
                    // lands at chunk position c ^ (r & 7)
#pragma unroll
                    for (int i = 0; i < kRowsPerLane; ++i) {
                        if (!src[i]) continue;
                        const int r = lane + 32 * i;
                        const unsigned char* g =
                            reinterpret_cast<const unsigned char*>(src[i] + kb * BK);
                        const uint32_t d = smem_u32(bbase + r * 128);
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc)
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                             d + ((cc ^ (r & 7)) << 4)),
                                         "l"(g + cc * 16)
                                         : "memory");
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    // publish the previous stage once its copies have landed
                    if (pending >= 0) {
                        asm volatile("cp.async.wait_group 1;" ::: "memory");
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        mbar_arrive(&b_full[pending]);
                    }
                    pending = stage;
                }
                if (++stage == B_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        if (gather && pending >= 0) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&b_full[pending]);
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        int as = 0, bs = 0;
        uint32_t aph = 0, bph = 0;
        int local = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++local) {
            int ti, mb_;
            unit_map(u, mblocks, args.tiles, ti, mb_, args.debug);
            const TokenTile tile = args.tiles[ti];
            if (unit_skipped(args, tile, mb_, BM)) {
                --local;  // skipped units take no accumulator buffer
                continue;
            }
            const int kb_end = unit_kblocks(args, mb_, kblocks, BM);
            const int n_eff = max(16, (tile.count + 15) & ~15);
            const uint32_t idesc = make_idesc(128, n_eff);
            const int buf = local % NBUF;
            mbar_wait(&tempty[buf], ((local / NBUF) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int kb = 0; kb < kb_end; ++kb) {
                mbar_wait(&a_full[as], aph);
                mbar_wait(&b_full[bs], bph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint32_t abase = smem_u32(a_ring + as * A_STAGE_BYTES);
                    const uint32_t bbase = smem_u32(b_ring + bs * B_STAGE_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t bdesc = make_desc_sw128(bbase + k * 32);
#pragma unroll
                        for (int s = 0; s < SLABS; ++s) {
                            const uint64_t adesc = make_desc_sw128(abase + s * A_SLAB_BYTES + k * 32);
                            mma_bf16(tmem_base + buf * ACC_COLS + s * NT, adesc, bdesc, idesc,
                                     (kb | k) != 0);
                        }
                    }
                    mma_commit(&a_empty[as]);
                    mma_commit(&b_empty[bs]);
                }
                __syncwarp();
                if (++as == A_STAGES) {
                    as = 0;
                    aph ^= 1;
                }
                if (++bs == B_STAGES) {
                    bs = 0;
                    bph ^= 1;
                }
            }
            if (lane == 0) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else {
        // ===== epilogue (warps 3..10: one warp per TMEM lane quadrant and slab) =====
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int ew = warp - EPI_WARP0;
        const int s = ew >> 2;  // weight slab this warp drains
        // Shared [32 tokens][256 rows] bf16 staging, row pitch EPI_PITCH: the
        // 8 warps each write their 32 rows of a 32-token chunk; then every
        // token row of the unit (256 rows = 512 contiguous bytes) leaves by a
        // bulk async copy (TMA engine, cp.async.bulk shared -> global) issued
        // by lane t < 4 of warp ew for token ew*4 + t.  The stores thus never
        // occupy the LSU, and a row past the tile end is simply not issued.
        // Named barrier 1 syncs the 8 epilogue warps.
        unsigned char* stage0 = smem + RING_BYTES + 256;
        constexpr int EPI_BUFS = gemm_epi_bufs<NT>();
        int chunk = 0;  // running chunk counter: staging buffer = chunk % EPI_BUFS
        const int mrow = s * 128 + quad * 32;  // this warp's rows within the unit
        constexpr int ROWS_PER_WARP = 32 / EPI_WARPS;
        int local = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++local) {
            int ti, mb;
            unit_map(u, mblocks, args.tiles, ti, mb, args.debug);
            const TokenTile tile = args.tiles[ti];
            if (unit_skipped(args, tile, mb, BM)) {
                --local;
                continue;
            }
            const int buf = local % NBUF;
            mbar_wait(&tfull[buf], (local / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (!(args.debug & 2)) {
                const uint32_t taddr =
                    tmem_base + ((uint32_t)(quad * 32) << 16) + buf * ACC_COLS + s * NT;
                constexpr bool kPrefetch = NT == 256;
                uint32_t vn[kPrefetch ? 32 : 1];
                if constexpr (kPrefetch) {
                    if (tile.count > 0) tmem_ld32_async(taddr, vn);
                }
                for (int j0 = 0; j0 < tile.count; j0 += 32, ++chunk) {
                    unsigned char* stage = stage0 + (chunk % EPI_BUFS) * EPI_STAGE_BYTES;
                    uint32_t v[32];
                    if constexpr (kPrefetch) {
                        // chunk j0 was issued one iteration ago; issue j0 + 32 now
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int q = 0; q < 32; ++q) v[q] = vn[q];
                        if (j0 + 32 < tile.count) tmem_ld32_async(taddr + j0 + 32, vn);
                    } else {
                        tmem_ld32(taddr + j0, v);  // v[jj] = D[mb*BM + mrow + lane][j0 + jj]
                    }
                    if (args.tma_store == 2) {
                        // contiguous output, direct stores: for token j0+jj the warp's
                        // 32 lanes hold 32 consecutive rows m, i.e. 64 contiguous bytes
                        // of out[token][.]: one coalesced st.global per token, fire and
                        // forget (no staging buffer, no wait on a bulk copy's reads)
                        __nv_bfloat16* dst =
                            args.out + (size_t)(tile.pos + j0) * args.M + mb * BM + mrow + lane;
                        const int nj = min(32, tile.count - j0);
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            if (jj < nj) {
                                float f = __uint_as_float(v[jj]);
                                if (args.silu) f = silu_fast(f);
                                dst[(size_t)jj * args.M] = __float2bfloat16_rn(f);
                            }
                        }
                        continue;
                    }
                    if (args.tma_store) {
                        // contiguous output: every warp stages its own 32 rows x 32
                        // tokens ([token][32 rows], 64 B per token) and stores them
                        // itself -- one [32 x 32] tensor store per full chunk, 64-byte
                        // row copies for the tile's last partial chunk; no barrier
                        // couples the epilogue warps
                        unsigned char* wst = stage + ew * (32 * 64);
                        if constexpr (EPI_BUFS == 2)
                            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        else
                            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        __syncwarp();
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            float f = __uint_as_float(v[jj]);
                            if (args.silu) f = silu_fast(f);
                            *reinterpret_cast<__nv_bfloat16*>(wst + jj * 64 + lane * 2) =
                                __float2bfloat16_rn(f);
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (!(args.debug & 1)) {
                            if (j0 + 32 <= tile.count) {
                                if (lane == 0) {
                                    asm volatile(
                                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                            reinterpret_cast<uint64_t>(&map_out)),
                                        "r"(mb * BM + mrow), "r"(tile.pos + j0), "r"(smem_u32(wst))
                                        : "memory");
                                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                                }
                            } else if (j0 + lane < tile.count) {
                                __nv_bfloat16* dst = args.out + (size_t)(tile.pos + j0 + lane) * args.M +
                                                     mb * BM + mrow;
                                asm volatile(
                                    "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(
                                        reinterpret_cast<uint64_t>(dst)),
                                    "r"(smem_u32(wst + lane * 64))
                                    : "memory");
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            }
                        }
                        continue;
                    }
                    // the bulk copies that last read this staging buffer are done
                    if (lane < ROWS_PER_WARP) {
                        if constexpr (EPI_BUFS == 2)
                            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        else
                            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        float f = __uint_as_float(v[jj]);
                        if (args.silu) f = silu_fast(f);
                        *reinterpret_cast<__nv_bfloat16*>(stage + jj * EPI_PITCH + (mrow + lane) * 2) =
                            __float2bfloat16_rn(f);
                    }
                    // generic-proxy writes -> visible to the async (bulk copy) proxy
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
                    const int jj = ew * ROWS_PER_WARP + lane;
                    if (lane < ROWS_PER_WARP && j0 + jj < tile.count && !(args.debug & 1)) {
                        const int p = tile.pos + j0 + jj;
                        __nv_bfloat16* dst =
                            (args.row_dst ? reinterpret_cast<__nv_bfloat16*>(
                                                args.row_dst[args.row_ids ? args.row_ids[p] : p])
                                          : args.out + (size_t)p * args.M) +
                            mb * BM;
                        asm volatile(
                            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                reinterpret_cast<uint64_t>(dst)),
                            "r"(smem_u32(stage + jj * EPI_PITCH)), "n"(BM * 2)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }

    if (warp >= EPI_WARP0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS));
    }
}

// ===========================================================================
// CTA-pair variant (tcgen05.mma.cta_group::2): one unit = (token tile, 256
// weight rows) is computed by the two CTAs of a cluster on two SMs.  CTA r
// holds weight slab r (128 rows) and half of the token tile (rows
// [r*N/2, (r+1)*N/2)); the leader (r = 0) issues M=256 MMAs that read A from
// each CTA's own slab and B from both halves, and each CTA's TMEM receives
// its own 128 rows x N accumulator.  Per SM this halves the token-tile bytes
// (TMA writes and tensor-core smem reads), the epilogue warps and the token
// ring, which buys (a) a deeper weight ring (more HBM bytes in flight per
// SM), (b) double-buffered accumulators at every tile width (the epilogue of
// unit i drains under the MMAs of unit i+1), and (c) a smaller footprint
// beside the co-resident exact router.
//
// Synchronisation: both CTAs' TMA loads complete_tx on the LEADER's full
// barriers (cta_group::2 bulk tensor copies), the leader's producer lanes
// post the pair's byte counts; the leader's MMA commits arrive on the empty
// barriers and the accumulator-full barriers of BOTH CTAs (multicast); each
// CTA's epilogue warps arrive on the leader's accumulator-empty barrier.
// ===========================================================================
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(saddr), "r"(rank));
    return o;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar,
                                                 void* dst, int c0, int c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in BOTH CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

constexpr int P_BOX = 32;                   // token rows per TMA box
constexpr int P_EPI_WARPS = 4;              // one per TMEM lane quadrant (own 128 rows)
constexpr int P_THREADS = 32 * (EPI_WARP0 + P_EPI_WARPS);
// a pipeline stage holds P_KS consecutive 64-wide K blocks, so each MMA
// commit (and barrier round trip between the two SMs) covers 4 * P_KS MMAs
constexpr int P_KS = 2;
template <int kNT>
__host__ __device__ constexpr int pair_a_stage_bytes() { return P_KS * A_SLAB_BYTES; }
template <int kNT>
__host__ __device__ constexpr int pair_b_stage_bytes() { return P_KS * (kNT / 2) * BK * 2; }
constexpr int P_EPI_BYTES = 32 * 128 * 2;   // [32 tokens][128 rows] bf16 per staging buffer
// kAS / kBS: weight / token ring stages (each P_KS K blocks)
template <int kNT, int kAS, int kBS>
constexpr int gemm_pair_smem_bytes() {
    return kAS * pair_a_stage_bytes<kNT>() + kBS * pair_b_stage_bytes<kNT>() + 1024 + 256 +
           2 * P_EPI_BYTES;
}

template <int kNT, int kAS, int kBS>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(128)
    grouped_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_w,
                             const __grid_constant__ CUtensorMap map_x,
                             const __grid_constant__ CUtensorMap map_out, const GemmArgs args) {
    constexpr int NT = kNT;
    constexpr int AS = kAS;
    constexpr int BS = kBS;
    constexpr int A_STAGE = pair_a_stage_bytes<kNT>();
    constexpr int B_STAGE = pair_b_stage_bytes<kNT>();
    constexpr int B_KB = (kNT / 2) * BK * 2;  // one K block of this CTA's token half
    constexpr int RING = AS * A_STAGE + BS * B_STAGE;
    static_assert(2 * NT <= TMEM_COLS, "double-buffered accumulators must fit TMEM");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* a_ring = smem;
    unsigned char* b_ring = smem + AS * A_STAGE;
    uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + RING);
    uint64_t* a_empty = a_full + AS;
    uint64_t* b_full = a_empty + AS;
    uint64_t* b_empty = b_full + BS;
    uint64_t* tfull = b_empty + BS;  // [2]
    uint64_t* tempty = tfull + 2;     // [2] (leader's are the live ones)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    unsigned char* epi = smem + RING + 256;

    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int mblocks = args.M / BM;
    const int kblocks = args.K / BK;
    const int ksteps = kblocks / P_KS;  // the launcher guarantees K % (P_KS * BK) == 0
    const int n_units = (*args.n_tiles) * mblocks;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < AS; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < BS; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * P_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    }
    if (warp == 1) {  // same warp in both CTAs (cta_group::2 allocation)
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== weight producer: this CTA's 128-row slab of each 256-row block =====
        if (lane == 0) {
            const uint64_t pol_once = policy_evict_first(), pol_shared = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < n_units; u += n_pairs) {
                int ti, mb;
                unit_map(u, mblocks, args.tiles, ti, mb, args.debug);
                const TokenTile tile = args.tiles[ti];
                if (unit_skipped(args, tile, mb, BM)) continue;
                const int ks_end = unit_kblocks(args, mb, kblocks, BM) / P_KS;
                const int ebase = tile.e * (args.M / 128) * kblocks * 128;
                const uint64_t pol_w = (tile.pad & 0xffff) > 1 ? pol_shared : pol_once;
                const int slab = mb * SLABS + (int)rank;
                for (int ks = 0; ks < ks_end; ++ks) {
                    mbar_wait(&a_empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&a_full[stage], 2 * A_STAGE);
                    const uint32_t bar = mapa_rank(smem_u32(&a_full[stage]), 0);
#pragma unroll
                    for (int q = 0; q < P_KS; ++q)
                        tma_load_2d_pair(&map_w, bar, a_ring + stage * A_STAGE + q * A_SLAB_BYTES, 0,
                                         ebase + (slab * kblocks + ks * P_KS + q) * 128, pol_w);
                    if (++stage == AS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 2) {
        // ===== token producer: this CTA's half of the tile's rows =====
        if (lane == 0) {
            const uint64_t pol_x = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < n_units; u += n_pairs) {
                int ti, mb_;
                unit_map(u, mblocks, args.tiles, ti, mb_, args.debug);
                const TokenTile tile = args.tiles[ti];
                if (unit_skipped(args, tile, mb_, BM)) continue;
                const int ks_end = unit_kblocks(args, mb_, kblocks, BM) / P_KS;
                const int n_eff = max(32, (tile.count + 31) & ~31);
                const int half = n_eff >> 1;
                const int nbox = (half + P_BOX - 1) / P_BOX;
                const int row0 = tile.pos + (int)rank * half;
                for (int ks = 0; ks < ks_end; ++ks) {
                    mbar_wait(&b_empty[stage], phase ^ 1);
                    if (args.debug & 32) {  // energy experiment: no token traffic
                        if (leader) mbar_arrive(&b_full[stage]);
                        if (++stage == BS) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    if (leader)
                        mbar_expect_tx(&b_full[stage], (uint32_t)(2 * P_KS * nbox * P_BOX * BK * 2));
                    const uint32_t bar = mapa_rank(smem_u32(&b_full[stage]), 0);
                    for (int q = 0; q < P_KS; ++q) {
                        unsigned char* bbase = b_ring + stage * B_STAGE + q * B_KB;
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_load_2d_pair(&map_x, bar, bbase + bx * P_BOX * BK * 2,
                                             (ks * P_KS + q) * BK, row0 + P_BOX * bx, pol_x);
                    }
                    if (++stage == BS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: the leader CTA only =====
        if (leader) {
            int as = 0, bs = 0;
            uint32_t aph = 0, bph = 0;
            int local = 0;
            for (int u = pair; u < n_units; u += n_pairs, ++local) {
                int ti, mb_;
                unit_map(u, mblocks, args.tiles, ti, mb_, args.debug);
                const TokenTile tile = args.tiles[ti];
                if (unit_skipped(args, tile, mb_, BM)) {
                    --local;  // skipped units take no accumulator buffer
                    continue;
                }
                const int ks_end = unit_kblocks(args, mb_, kblocks, BM) / P_KS;
                const int n_eff = max(32, (tile.count + 31) & ~31);
                const uint32_t idesc = make_idesc(256, n_eff);
                const int buf = local & 1;
                mbar_wait(&tempty[buf], ((local >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int ks = 0; ks < ks_end; ++ks) {
                    mbar_wait(&a_full[as], aph);
                    mbar_wait(&b_full[bs], bph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (lane == 0) {
                        if (!(args.debug & 16)) {  // 16: no MMAs (energy experiment)
#pragma unroll
                            for (int q = 0; q < P_KS; ++q) {
                                const uint32_t abase =
                                    smem_u32(a_ring + as * A_STAGE + q * A_SLAB_BYTES);
                                const uint32_t bbase = smem_u32(b_ring + bs * B_STAGE + q * B_KB);
#pragma unroll
                                for (int k = 0; k < BK / 16; ++k)
                                    mma_bf16_pair(tmem_base + buf * NT,
                                                  make_desc_sw128(abase + k * 32),
                                                  make_desc_sw128(bbase + k * 32), idesc,
                                                  (ks | q | k) != 0);
                            }
                        }
                        mma_commit_pair(&a_empty[as]);
                        mma_commit_pair(&b_empty[bs]);
                    }
                    __syncwarp();
                    if (++as == AS) {
                        as = 0;
                        aph ^= 1;
                    }
                    if (++bs == BS) {
                        bs = 0;
                        bph ^= 1;
                    }
                }
                if (lane == 0) mma_commit_pair(&tfull[buf]);
                __syncwarp();
            }
        }
    } else {
        // ===== epilogue: warps 3..6 drain this CTA's 128 accumulator rows =====
        const int quad = warp & 3;
        const int ew = warp - EPI_WARP0;
        const uint32_t tempty_leader[2] = {mapa_rank(smem_u32(&tempty[0]), 0),
                                           mapa_rank(smem_u32(&tempty[1]), 0)};
        int chunk = 0;
        int local = 0;
        for (int u = pair; u < n_units; u += n_pairs, ++local) {
            int ti, mb;
            unit_map(u, mblocks, args.tiles, ti, mb, args.debug);
            const TokenTile tile = args.tiles[ti];
            if (unit_skipped(args, tile, mb, BM)) {
                --local;
                continue;
            }
            const int buf = local & 1;
            mbar_wait(&tfull[buf], (local >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int row_base = mb * BM + (int)rank * 128;  // this CTA's 128 rows
            const int mrow = quad * 32;                       // this warp's 32 of them
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * NT;
            uint32_t vn[32];
            if (tile.count > 0) tmem_ld32_async(taddr, vn);
            for (int j0 = 0; j0 < tile.count; j0 += 32, ++chunk) {
                unsigned char* stage = epi + (chunk & 1) * P_EPI_BYTES;
                uint32_t v[32];
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 32; ++q) v[q] = vn[q];
                if (j0 + 32 < tile.count) tmem_ld32_async(taddr + j0 + 32, vn);
                if (args.tma_store) {
                    // [32 tokens][32 rows] per warp, one tensor store per full chunk
                    unsigned char* wst = stage + ew * (32 * 64);
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        float f = __uint_as_float(v[jj]);
                        if (args.silu) f = silu_fast(f);
                        *reinterpret_cast<__nv_bfloat16*>(wst + jj * 64 + lane * 2) =
                            __float2bfloat16_rn(f);
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (j0 + 32 <= tile.count) {
                        if (lane == 0) {
                            asm volatile(
                                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                    reinterpret_cast<uint64_t>(&map_out)),
                                "r"(row_base + mrow), "r"(tile.pos + j0), "r"(smem_u32(wst))
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                    } else if (j0 + lane < tile.count) {
                        __nv_bfloat16* dst =
                            args.out + (size_t)(tile.pos + j0 + lane) * args.M + row_base + mrow;
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(
                                         reinterpret_cast<uint64_t>(dst)),
                                     "r"(smem_u32(wst + lane * 64))
                                     : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    continue;
                }
                // scattered rows (e.g. the EP return over NVLink): [32 tokens][128 rows]
                // shared by the 4 epilogue warps; each token's 256 B of this CTA's rows
                // leave by one bulk copy
                constexpr int TOK_PER_WARP = 32 / P_EPI_WARPS;
                if (lane < TOK_PER_WARP) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                asm volatile("bar.sync 1, %0;" ::"n"(P_EPI_WARPS * 32) : "memory");
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    float f = __uint_as_float(v[jj]);
                    if (args.silu) f = silu_fast(f);
                    *reinterpret_cast<__nv_bfloat16*>(stage + jj * 256 + (mrow + lane) * 2) =
                        __float2bfloat16_rn(f);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, %0;" ::"n"(P_EPI_WARPS * 32) : "memory");
                const int jj = ew * TOK_PER_WARP + lane;
                if (lane < TOK_PER_WARP && j0 + jj < tile.count) {
                    const int p = tile.pos + j0 + jj;
                    __nv_bfloat16* dst = (args.row_dst ? reinterpret_cast<__nv_bfloat16*>(
                                                             args.row_dst[args.row_ids ? args.row_ids[p] : p])
                                                       : args.out + (size_t)p * args.M) +
                                         row_base;
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;" ::"l"(
                                     reinterpret_cast<uint64_t>(dst)),
                                 "r"(smem_u32(stage + jj * 256))
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader[buf]);
        }
    }

    if (warp >= EPI_WARP0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // the peer's MMAs / arrivals into this CTA are done
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS));
    }
}

CUtensorMap make_map_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                        uint32_t box_cols, uint64_t row_stride = 0) {
    return make_tma_map_2d(base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sizeof(__nv_bfloat16), rows, cols,
                           box_rows, box_cols, CU_TENSOR_MAP_SWIZZLE_128B, row_stride);
}

}  // namespace

int grouped_gemm_tile_rows() { return NT; }
int grouped_gemm_tile_rows_large() { return 256; }

void launch_grouped_gemm_bf16(scmoe_ctx* c, const __nv_bfloat16* W, size_t n_experts, size_t M,
                              size_t K, const __nv_bfloat16* X, size_t x_rows, const int* x_row_ids,
                              __nv_bfloat16* out, int silu, const TokenTile* tiles,
                              const int* n_tiles_dev, size_t max_tiles, int tile_rows,
                              const uint64_t* row_dst, const int* row_ids, size_t x_ld,
                              int causal_rows, int causal_k) {
    if (max_tiles == 0 || n_experts == 0) return;
    SCMOE_CHECK_ARG(tile_rows == 128 || tile_rows == 192 || tile_rows == 256, SCMOE_ERR_INTERNAL,
                    "gemm: tile rows must be 128, 192 or 256");
    SCMOE_CHECK_ARG(M % BM == 0 && K % BK == 0, SCMOE_ERR_DIMENSION,
                    "gemm: M must be a multiple of 256 and K of 64");
    // W in the blocked layout (internal.cuh wblk_index): a 2-D view of rows of BK elements
    const CUtensorMap mw = make_map_2d(W, n_experts * M * K / BK, BK, 128, BK);
    // X: tiled boxes of 128 permuted rows, or single-row boxes for tile::gather4
    const CUtensorMap mx =
        make_map_2d(X, std::max<size_t>(x_rows, 1), K, x_row_ids ? 1 : 64, BK, x_ld);
    // contiguous output: tensor map for the epilogue warps' [32 tokens x 32 rows]
    // stores (SWIZZLE_NONE: each warp's staging tile is dense, 64 B per token)
    static const bool tma_store_on = [] {
        const char* e = getenv("SCMOE_GEMM_TMA_STORE");
        return !(e && atoi(e) == 0);
    }();
    const bool use_tma_store = tma_store_on && row_dst == nullptr;
    const CUtensorMap mo =
        use_tma_store ? make_tma_map_2d(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sizeof(__nv_bfloat16),
                                        std::max<size_t>(max_tiles * tile_rows, 1), M, 32, 32,
                                        CU_TENSOR_MAP_SWIZZLE_NONE)
                      : mw;
    // epilogue of contiguous outputs: SCMOE_GEMM_EPI=direct -> per-token coalesced
    // st.global from the TMEM registers; default: per-warp TMA tensor stores
    static const int epi_direct = [] {
        const char* e = getenv("SCMOE_GEMM_EPI");
        return e && std::string(e) == "direct" ? 1 : 0;
    }();
    GemmArgs a;
    a.tma_store = use_tma_store ? (epi_direct ? 2 : 1) : 0;
    a.tiles = tiles;
    a.n_tiles = n_tiles_dev;
    a.x_rows = x_row_ids;
    a.x = X;
    a.out = out;
    a.row_dst = row_dst;
    a.row_ids = row_ids;
    a.M = (int)M;
    a.K = (int)K;
    a.silu = silu;
    a.causal_rows = causal_rows;
    a.causal_k = causal_k;
    static const int dbg = getenv("SCMOE_GEMM_DEBUG") ? atoi(getenv("SCMOE_GEMM_DEBUG")) : 0;
    a.debug = dbg;
    const size_t units_max = max_tiles * (M / BM);
    const int grid = (int)std::min<size_t>(
        units_max, (size_t)(c->gemm_sms > 0 ? std::min(c->gemm_sms, c->num_sms) : c->num_sms));
    // 256-token tiles: two 128-row slabs per unit (default; measured faster at
    // the EP x4 shard shape: 2.97 vs 3.16 ms) or, SCMOE_GEMM_SLABS=1, one slab
    // with double-buffered TMEM accumulators
    static const int slabs256 = [] {
        const char* e = getenv("SCMOE_GEMM_SLABS");
        return e && atoi(e) == 1 ? 1 : 2;
    }();
    auto go = [&](auto kern, int smem, int threads, int bm) {
        const size_t units = max_tiles * (M / bm);
        const int g = (int)std::min<size_t>(
            units, (size_t)(c->gemm_sms > 0 ? std::min(c->gemm_sms, c->num_sms) : c->num_sms));
        ensure_max_dynamic_smem(reinterpret_cast<const void*>(kern), smem, c->device);
        kern<<<g, threads, smem, c->stream>>>(mw, mx, mo, a);
    };
    (void)grid;
    // CTA-pair kernel (default; SCMOE_GEMM_2SM=0 selects the single-CTA one)
    static const bool pair_on = [] {
        const char* e = getenv("SCMOE_GEMM_2SM");
        return !(e && atoi(e) == 0);
    }();
    if (pair_on && x_row_ids == nullptr && (tile_rows == 192 || tile_rows == 256) &&
        K % (P_KS * BK) == 0) {
        const CUtensorMap mx32 = make_map_2d(X, std::max<size_t>(x_rows, 1), K, P_BOX, BK, x_ld);
        auto go2 = [&](auto kern, int smem) {
            const size_t units = max_tiles * (M / BM);
            const int sms = c->gemm_sms > 0 ? std::min(c->gemm_sms, c->num_sms) : c->num_sms;
            const int pairs = (int)std::min<size_t>(units, (size_t)std::max(1, sms / 2));
            ensure_max_dynamic_smem(reinterpret_cast<const void*>(kern), smem, c->device);
            kern<<<2 * pairs, P_THREADS, smem, c->stream>>>(mw, mx32, mo, a);
        };
        // ring stages of the 192-token variant (the one beside the router):
        // SCMOE_PAIR_STAGES = "AB" digits, default 33
        static const int st = [] {
            const char* e = getenv("SCMOE_PAIR_STAGES");
            return e ? atoi(e) : 33;
        }();
        if (tile_rows == 256 && c->corun_gemm)  // 177 KB: fits beside the 25 KB router
            go2(grouped_gemm_pair_kernel<256, 3, 2>, gemm_pair_smem_bytes<256, 3, 2>());
        else if (tile_rows == 256)
            go2(grouped_gemm_pair_kernel<256, 3, 3>, gemm_pair_smem_bytes<256, 3, 3>());
        else if (st == 32)
            go2(grouped_gemm_pair_kernel<192, 3, 2>, gemm_pair_smem_bytes<192, 3, 2>());
        else if (st == 22)
            go2(grouped_gemm_pair_kernel<192, 2, 2>, gemm_pair_smem_bytes<192, 2, 2>());
        else
            go2(grouped_gemm_pair_kernel<192, 3, 3>, gemm_pair_smem_bytes<192, 3, 3>());
        SCMOE_LAUNCH_CHECK(c);
        return;
    }
    if (tile_rows == 128) {
        go(grouped_gemm_kernel<128>, gemm_smem_bytes<128>(), NUM_THREADS, BM);
    } else if (tile_rows == 256 && slabs256 == 1) {
        // (per-warp stores work for any BM)
        go(grouped_gemm_kernel<256, 1>, gemm_smem_bytes<256, 1>(), 32 * (EPI_WARP0 + 4), 128);
    } else if (tile_rows == 256) {
        go(grouped_gemm_kernel<256, 2>, gemm_smem_bytes<256, 2>(), NUM_THREADS, BM);
    } else {
        go(grouped_gemm_kernel<192>, gemm_smem_bytes<192>(), NUM_THREADS, BM);
    }
    SCMOE_LAUNCH_CHECK(c);
}

}  // namespace scmoe
