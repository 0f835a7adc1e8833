// libm_port.h -- bit-exact restatement of glibc 2.39 expf (FMA ifunc variant).
//
// The reference computes softmax_rows (tensor.hpp:183) and the SiLU logistic
// (graph.hpp:529-533) with std::exp(float), i.e. glibc's expf, which on an
// FMA-capable x86 host dispatches to the variant compiled with -mfma.  Its
// algorithm (sysdeps/ieee754/flt-32/e_expf.c, ARM optimized-routines; table
// __exp2f_data, EXP2F_TABLE_BITS = 5) is restated here with every FMA that
// GCC contracts in that build written as an explicit fused multiply-add and
// every other operation as a separately rounded double op, so nvcc cannot
// re-contract anything.  SURVEY.md 8(a) a3 records the exhaustive probe;
// tests/test_libm_port.py re-checks all 2^31 negative floats on the host and
// the GPU test checks the device instantiation against host libm.
//
// Usable from host C/C++ (compile with -ffp-contract=off) and CUDA.
#pragma once
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SCMOE_HD __host__ __device__ __forceinline__
#else
#define SCMOE_HD static inline
#include <math.h>
#endif

// T[i] = bits(2^(i/32)) - (i << 47): 2^(i/32) rounded to nearest double,
// with the exponent contribution of i/32 removed (glibc __exp2f_data.tab).
#define SCMOE_EXP2F_TAB                                                                             \
    {0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,   \
     0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,   \
     0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,   \
     0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,   \
     0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,   \
     0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,   \
     0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,   \
     0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL}

#if defined(__CUDACC__)
__device__ __constant__ static const uint64_t scmoe_exp2f_tab_dev[32] = SCMOE_EXP2F_TAB;
#endif
static const uint64_t scmoe_exp2f_tab_host[32] = SCMOE_EXP2F_TAB;

SCMOE_HD uint32_t scmoe_f2u(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
SCMOE_HD double scmoe_u2d(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}
SCMOE_HD uint64_t scmoe_d2u(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}

#if defined(__CUDA_ARCH__)
#define SCMOE_FMA(a, b, c) __fma_rn((a), (b), (c))
#define SCMOE_DMUL(a, b) __dmul_rn((a), (b))
#define SCMOE_DSUB(a, b) __dsub_rn((a), (b))
#define SCMOE_TAB(i) scmoe_exp2f_tab_dev[(i)]
#define SCMOE_D2F(x) __double2float_rn(x)
#else
#define SCMOE_FMA(a, b, c) fma((a), (b), (c))
#define SCMOE_DMUL(a, b) ((a) * (b))
#define SCMOE_DSUB(a, b) ((a) - (b))
#define SCMOE_TAB(i) scmoe_exp2f_tab_host[(i)]
#define SCMOE_D2F(x) ((float)(x))
#endif

// glibc 2.39 __expf, FMA build.
SCMOE_HD float scmoe_expf(float x) {
    const double kInvLn2N = 0x1.71547652b82fep+0 * 32;  // N/ln2
    const double kShift = 0x1.8p+52;
    const double kC0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
    const double kC1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
    const double kC2 = 0x1.62e42ff0c52d6p-1 / 32;
    const uint32_t ux = scmoe_f2u(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {                       // |x| >= 88 or non-finite
        if (ux == 0xff800000u) return 0.0f;      // -inf
        if (abstop >= 0x7f8) return x + x;       // +inf or nan
        if (x > 0x1.62e42ep6f) return __builtin_huge_valf();  // overflow
        if (x < -0x1.9fe368p6f) return 0.0f;     // underflow (x < log(2^-150))
    }
    const double xd = (double)x;
    double kd = SCMOE_FMA(kInvLn2N, xd, kShift);  // z + SHIFT, contracted
    const uint64_t ki = scmoe_d2u(kd);
    kd = SCMOE_DSUB(kd, kShift);
    const double r = SCMOE_FMA(kInvLn2N, xd, -kd);  // z - kd, contracted
    uint64_t t = SCMOE_TAB(ki % 32);
    t += ki << 47;
    const double s = scmoe_u2d(t);
    const double z = SCMOE_FMA(kC0, r, kC1);
    const double r2 = SCMOE_DMUL(r, r);
    double y = SCMOE_FMA(kC2, r, 1.0);
    y = SCMOE_FMA(z, r2, y);
    y = SCMOE_DMUL(y, s);
    return SCMOE_D2F(y);
}

#if defined(__CUDACC__)
// graph.hpp:529-533 in S = float: sign-branched logistic.
__device__ __forceinline__ float scmoe_sigmoidf(float x) {
    if (x >= 0.0f) return __fdiv_rn(1.0f, __fadd_rn(1.0f, scmoe_expf(-x)));
    const float e = scmoe_expf(x);
    return __fdiv_rn(e, __fadd_rn(1.0f, e));
}
// graph.hpp:133-135: silu(v) = v * sigmoid(v)
__device__ __forceinline__ float scmoe_siluf(float v) { return __fmul_rn(v, scmoe_sigmoidf(v)); }
#endif
