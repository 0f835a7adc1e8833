// f32x2.cuh -- packed two-lane fp32 arithmetic (FMUL2 / FADD2, sm_100a) with
// the rounding of two separate IEEE fp32 operations: every product and every
// sum is rounded to nearest-even, nothing is fused.
//
// ptxas contracts a mul.rn.f32x2 feeding an add.rn.f32x2 into FFMA2 -- even
// with the explicit .rn and --fmad=false (checked with ptxas 12.9) -- which
// would change the result.  Adding the product HALF-SWAPPED (accumulator pair
// (c1, c0) += (p1, p0) swapped) blocks the contraction and costs nothing: the
// swap is an operand modifier of FADD2 (.F32x2.LO_HI).  build.py asserts that
// the kernels using these helpers contain no FFMA/FFMA2.
#pragma once
#include <cstdint>

namespace scmoe {

// (a, a) * (b0, b1): FMUL2 with a broadcast scalar operand (.F32).
__device__ __forceinline__ uint64_t f2_mul_bcast(float a, uint64_t b) {
    uint64_t r, ad;
    asm("mov.b64 %0, {%1, %1};" : "=l"(ad) : "f"(a));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ad), "l"(b));
    return r;
}
// acc + swap(p): acc's low lane accumulates p's high lane and vice versa.
__device__ __forceinline__ uint64_t f2_add_swapped(uint64_t acc, uint64_t p) {
    uint64_t r;
    asm("{.reg .b32 l, h; .reg .b64 s; mov.b64 {l, h}, %2; mov.b64 s, {h, l};"
        " add.rn.f32x2 %0, %1, s;}"
        : "=l"(r)
        : "l"(acc), "l"(p));
    return r;
}
__device__ __forceinline__ float f2_lo(uint64_t a) { return __uint_as_float((uint32_t)a); }
__device__ __forceinline__ float f2_hi(uint64_t a) { return __uint_as_float((uint32_t)(a >> 32)); }

}  // namespace scmoe
