/*
 * scmoe_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithm for the ScMoE hot
 * path (moelab, /root/reference/proj/include/moelab).  It is the checker the
 * parity tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * compare the CUDA path against.  Nothing in the product (libscmoe.so, the
 * Python package, the compat headers) may link or call this file.
 *
 * Parity pin: every function below is checked in tests/test_oracle_*.py
 * against (a) the golden vectors of the reference's own Catch2 tests
 * (tests/test_router.cpp, tests/test_blocks.cpp, tests/test_core.cpp) and
 * (b) the reference itself, compiled from its headers into
 * oracle/_ref/libmoelab_ref.so by oracle/Makefile (oracle/ref_shim.cpp).
 *
 * Build flags matter: compile with -O2/-O3 and
 * -ffp-contract=off and WITHOUT -march=native, exactly like the reference's
 * CMake Release build.  Floating-point operations are written in the same
 * order as the reference so results are bitwise identical.
 *
 * Error codes mirror the reference's exception taxonomy (common.hpp:11-33):
 *   0 ok, 1 ConfigError, 2 DimensionError, 3 StateError, 4 ParameterError.
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_CONFIG 1
#define ORC_DIMENSION 2
#define ORC_STATE 3
#define ORC_PARAMETER 4

#define ORC_NZ(x) ((x) > 0 ? (size_t)(x) : (size_t)1)

/* ------------------------------------------------------------------------
 * Counter RNG -- rng.hpp:15-64
 * ---------------------------------------------------------------------- */

/* rng.hpp:19-26 */
uint64_t orc_mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

/* rng.hpp:28-30 */
uint64_t orc_hash2(uint64_t seed, uint64_t ctr) {
    return orc_mix64(orc_mix64(seed + 0x9e3779b97f4a7c15ULL) ^ orc_mix64(ctr + 0xbf58476d1ce4e5b9ULL));
}

/* rng.hpp:35 -- CounterRng::stream(id) returns a generator seeded with this */
uint64_t orc_stream_seed(uint64_t seed, uint64_t id) { return orc_hash2(seed, id ^ 0xa5a5a5a5a5a5a5a5ULL); }

/* rng.hpp:40-42 */
double orc_uniform01_at(uint64_t seed, uint64_t ctr) {
    return ((double)(orc_hash2(seed, ctr) >> 11) + 1.0) * 0x1.0p-53;
}

/* rng.hpp:51-55 (Box-Muller on counters 2c, 2c+1) */
double orc_normal_at(uint64_t seed, uint64_t ctr) {
    const double u1 = orc_uniform01_at(seed, 2 * ctr);
    const double u2 = orc_uniform01_at(seed, 2 * ctr + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* router.hpp:357-360: x.data[i] = (S) batch_rng.normal_at(i), counters offset by `first` */
void orc_fill_normal_f32(uint64_t seed, uint64_t first, uint64_t n, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)orc_normal_at(seed, first + i);
}
void orc_fill_normal_f64(uint64_t seed, uint64_t first, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_normal_at(seed, first + i);
}

/* rng.hpp:89-94: Uniform init, element i drawn from counter i */
int orc_seeded_uniform_f32(uint64_t seed, uint64_t first, uint64_t n, double variance, float* out) {
    if (variance < 0.0) return ORC_PARAMETER;
    if (variance == 0.0) {
        memset(out, 0, n * sizeof(float));
        return ORC_OK;
    }
    const double half_width = sqrt(3.0 * variance);
    for (uint64_t i = 0; i < n; ++i) {
        const double u = orc_uniform01_at(seed, first + i);
        out[i] = (float)((2.0 * u - 1.0) * half_width);
    }
    return ORC_OK;
}

/* rng.hpp:95-111: TruncatedNormal init (64 rejection attempts per element) */
int orc_seeded_tn_f64(uint64_t seed, uint64_t n, double variance, double* out) {
    if (variance < 0.0) return ORC_PARAMETER;
    if (variance == 0.0) {
        memset(out, 0, n * sizeof(double));
        return ORC_OK;
    }
    const double scale = sqrt(variance / 0.77374201465191098);
    for (uint64_t i = 0; i < n; ++i) {
        double z = 0.0;
        int ok = 0;
        for (uint64_t attempt = 0; attempt < 64; ++attempt) {
            z = orc_normal_at(seed, (i << 6) | attempt);
            if (z >= -2.0 && z <= 2.0) {
                ok = 1;
                break;
            }
        }
        if (!ok) z = 0.0;
        out[i] = z * scale;
    }
    return ORC_OK;
}
int orc_seeded_tn_f32(uint64_t seed, uint64_t n, double variance, float* out) {
    if (variance < 0.0) return ORC_PARAMETER;
    double* tmp = (double*)malloc(ORC_NZ(n) * sizeof(double));
    int rc = orc_seeded_tn_f64(seed, n, variance, tmp);
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)tmp[i];
    free(tmp);
    return rc;
}

/* ------------------------------------------------------------------------
 * Fixed-order kernels -- tensor.hpp:95-112 (mm_into), :174-192 (softmax_rows)
 * Generated for S = float and S = double.
 * ---------------------------------------------------------------------- */

#define ORC_DEFINE_KERNELS(S, SUF, EXPF, SQRTF)                                                    \
    /* tensor.hpp:95-112: c[i,j] = sum_p a[i,p]*b[p,j], p ascending, separate mul/add */           \
    void orc_mm_##SUF(const S* a, const S* b, S* c, size_t m, size_t k, size_t n) {                \
        for (size_t i = 0; i < m; ++i) {                                                           \
            S* crow = c + i * n;                                                                   \
            for (size_t j = 0; j < n; ++j) crow[j] = (S)0;                                         \
            for (size_t p = 0; p < k; ++p) {                                                       \
                const S av = a[i * k + p];                                                         \
                const S* brow = b + p * n;                                                         \
                for (size_t j = 0; j < n; ++j) crow[j] += av * brow[j];                            \
            }                                                                                      \
        }                                                                                          \
    }                                                                                              \
    /* tensor.hpp:174-192: row max, exp(in-mx), sequential sum, divide */                          \
    void orc_softmax_rows_##SUF(const S* x, S* y, size_t rows, size_t cols) {                      \
        for (size_t r = 0; r < rows; ++r) {                                                        \
            const S* in = x + r * cols;                                                            \
            S* out = y + r * cols;                                                                 \
            S mx = in[0];                                                                          \
            for (size_t j = 1; j < cols; ++j) mx = in[j] > mx ? in[j] : mx;                        \
            S sum = (S)0;                                                                          \
            for (size_t j = 0; j < cols; ++j) {                                                    \
                out[j] = EXPF(in[j] - mx);                                                         \
                sum += out[j];                                                                     \
            }                                                                                      \
            for (size_t j = 0; j < cols; ++j) out[j] /= sum;                                       \
        }                                                                                          \
    }                                                                                              \
    /* graph.hpp:529-533: sign-branched logistic */                                                \
    S orc_sigmoid_##SUF(S x) {                                                                     \
        if (x >= (S)0) return (S)1 / ((S)1 + EXPF(-x));                                            \
        const S e = EXPF(x);                                                                       \
        return e / ((S)1 + e);                                                                     \
    }                                                                                              \
    /* graph.hpp:322-335: s2 += x*x (j ascending); inv = 1/sqrt(s2/d + eps); out = x*inv*g */      \
    void orc_rmsnorm_##SUF(const S* x, const S* gain, size_t rows, size_t d, S eps, S* out) {      \
        for (size_t r = 0; r < rows; ++r) {                                                        \
            const S* xr = x + r * d;                                                               \
            S s2 = (S)0;                                                                           \
            for (size_t j = 0; j < d; ++j) s2 += xr[j] * xr[j];                                    \
            const S inv = (S)1 / SQRTF(s2 / (S)d + eps);                                           \
            for (size_t j = 0; j < d; ++j) out[r * d + j] = xr[j] * inv * gain[j];                 \
        }                                                                                          \
    }

ORC_DEFINE_KERNELS(float, f32, expf, sqrtf)
ORC_DEFINE_KERNELS(double, f64, exp, sqrt)

float orc_expf(float x) { return expf(x); }
/* libm expf over consecutive bit patterns (checker for the device port) */
void orc_expf_range(uint32_t first_bits, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) {
        const uint32_t u = first_bits + (uint32_t)i;
        float x;
        memcpy(&x, &u, 4);
        out[i] = expf(x);
    }
}

/* ------------------------------------------------------------------------
 * Router -- router.hpp:50-141
 * ---------------------------------------------------------------------- */

/* router.hpp:50-61 RouterState::validate */
int orc_router_validate(size_t n_ffn, size_t n_zero, size_t top_k, size_t k_expected, double mu,
                        const double* b) {
    const size_t e = n_ffn + n_zero;
    if (top_k > e) return ORC_CONFIG;
    if (k_expected < 1 || k_expected > top_k) return ORC_CONFIG;
    if (n_zero > 0 && k_expected >= top_k) return ORC_CONFIG;
    if (n_zero < top_k - k_expected) return ORC_CONFIG;
    if (mu < 0.0) return ORC_CONFIG;
    if (b)
        for (size_t i = n_ffn; i < e; ++i)
            if (b[i] != 0.0) return ORC_CONFIG;
    return ORC_OK;
}

/* router.hpp:90-104: K largest of double(p)+b, ordered (score desc, index asc).
 * The comparator is a strict total order, so repeated arg-max extraction gives
 * the same sequence as std::partial_sort. */
#define ORC_DEFINE_SELECT(S, SUF)                                                                  \
    void orc_select_topk_row_##SUF(const S* probs, const double* bias, size_t n_experts, size_t k, \
                                   uint32_t* out_idx) {                                            \
        unsigned char stack_taken[1024];                                                           \
        unsigned char* taken = n_experts <= sizeof(stack_taken) ? stack_taken                      \
                                                                : (unsigned char*)malloc(n_experts); \
        memset(taken, 0, n_experts);                                                               \
        for (size_t s = 0; s < k; ++s) {                                                           \
            size_t best = (size_t)-1;                                                              \
            double best_score = 0.0;                                                               \
            for (size_t i = 0; i < n_experts; ++i) {                                               \
                if (taken[i]) continue;                                                            \
                const double sc = (double)probs[i] + bias[i];                                      \
                if (best == (size_t)-1 || sc > best_score) {                                       \
                    best = i;                                                                      \
                    best_score = sc;                                                               \
                }                                                                                  \
            }                                                                                      \
            taken[best] = 1;                                                                       \
            out_idx[s] = (uint32_t)best;                                                           \
        }                                                                                          \
        if (taken != stack_taken) free(taken);                                                     \
    }                                                                                              \
    /* router.hpp:107-130 */                                                                       \
    int orc_route_from_probs_##SUF(const S* probs, size_t t_count, size_t n_ffn, size_t n_zero,    \
                                   size_t top_k, size_t k_expected, double mu, const double* bias, \
                                   uint32_t* indices, double* gates, uint32_t* ffn_count) {        \
        int rc = orc_router_validate(n_ffn, n_zero, top_k, k_expected, mu, bias);                  \
        if (rc) return rc;                                                                         \
        const size_t e = n_ffn + n_zero;                                                           \
        for (size_t t = 0; t < t_count; ++t) {                                                     \
            uint32_t* idx = indices + t * top_k;                                                   \
            orc_select_topk_row_##SUF(probs + t * e, bias, e, top_k, idx);                         \
            uint32_t ffn = 0;                                                                      \
            for (size_t s = 0; s < top_k; ++s) {                                                   \
                gates[t * top_k + s] = (double)probs[t * e + idx[s]];                              \
                if (idx[s] < n_ffn) ++ffn;                                                         \
            }                                                                                      \
            ffn_count[t] = ffn;                                                                    \
        }                                                                                          \
        return ORC_OK;                                                                             \
    }                                                                                              \
    /* router.hpp:133-141: logits = mm(x, w); probs = softmax_rows(logits); route_from_probs */   \
    int orc_route_topk_##SUF(const S* x, size_t t_count, size_t d, const S* w, size_t n_ffn,       \
                             size_t n_zero, size_t top_k, size_t k_expected, double mu,            \
                             const double* bias, uint32_t* indices, double* gates,                 \
                             uint32_t* ffn_count, S* probs_out) {                                  \
        const size_t e = n_ffn + n_zero;                                                           \
        S* logits = (S*)malloc(ORC_NZ(t_count * e) * sizeof(S));                       \
        S* probs = probs_out ? probs_out : (S*)malloc(ORC_NZ(t_count * e) * sizeof(S)); \
        orc_mm_##SUF(x, w, logits, t_count, d, e);                                                 \
        orc_softmax_rows_##SUF(logits, probs, t_count, e);                                         \
        int rc = orc_route_from_probs_##SUF(probs, t_count, n_ffn, n_zero, top_k, k_expected, mu,  \
                                            bias, indices, gates, ffn_count);                      \
        free(logits);                                                                              \
        if (!probs_out) free(probs);                                                               \
        return rc;                                                                                 \
    }

ORC_DEFINE_SELECT(float, f32)
ORC_DEFINE_SELECT(double, f64)

/* router.hpp:144-150: slot-counted, zero experts included */
void orc_accumulate_counters(const uint32_t* indices, size_t t_count, size_t top_k,
                             uint64_t* tokens_routed, uint64_t* tokens_seen) {
    for (size_t t = 0; t < t_count; ++t)
        for (size_t s = 0; s < top_k; ++s) ++tokens_routed[indices[t * top_k + s]];
    *tokens_seen += t_count;
}

/* Routing statistics: RoutingDecision::mean_ffn / std_ffn
 * (router.hpp:73-86), per-expert slot load (stats.hpp:64-67) and the
 * slot-counted LB group frequencies lb_group_frequencies (router.hpp:193-216).
 * load may be NULL; lb may be NULL (else groups + (n_zero > 0) entries). */
int orc_routing_stats(const uint32_t* indices, const uint32_t* ffn_count, size_t t_count,
                      size_t top_k, size_t n_ffn, size_t n_zero, size_t k_expected,
                      size_t groups, double* mean, double* std_out, double* load, double* lb) {
    const size_t e = n_ffn + n_zero;
    if (lb && (groups == 0 || n_ffn % groups != 0)) return ORC_CONFIG;
    double m = 0.0, sd = 0.0;
    if (t_count) {
        double s = 0.0;
        for (size_t t = 0; t < t_count; ++t) s += ffn_count[t];
        m = s / (double)t_count;
        double s2 = 0.0;
        for (size_t t = 0; t < t_count; ++t) s2 += (ffn_count[t] - m) * (ffn_count[t] - m);
        sd = sqrt(s2 / (double)t_count);
    }
    *mean = m;
    *std_out = sd;
    if (load) {
        for (size_t i = 0; i < e; ++i) load[i] = 0.0;
        for (size_t i = 0; i < t_count * top_k; ++i) load[indices[i]] += 1.0;
        for (size_t i = 0; i < e; ++i) load[i] /= (double)(t_count * top_k);
    }
    if (lb) {
        const size_t gsz = n_ffn / groups;
        const int has_zero = n_zero > 0;
        const double tc = (double)t_count;
        for (size_t j = 0; j < groups + (size_t)has_zero; ++j) lb[j] = 0.0;
        for (size_t i = 0; i < t_count * top_k; ++i) {
            const uint32_t x = indices[i];
            if (x < n_ffn)
                lb[x / gsz] += 1.0;
            else
                lb[groups] += 1.0;
        }
        const size_t slack = top_k - k_expected;
        for (size_t j = 0; j < groups; ++j)
            lb[j] *= (double)groups / ((double)k_expected * tc);
        if (has_zero) lb[groups] /= (double)slack * tc;
    }
    return ORC_OK;
}

/* router.hpp:155-176: PID-style bias controller tick */
int orc_bias_update(size_t n_ffn, size_t n_zero, size_t top_k, size_t k_expected, double* mu,
                    double mu_decay, double* b, uint64_t* tokens_routed, uint64_t* tokens_seen,
                    double* delta) {
    const size_t e = n_ffn + n_zero;
    if (*tokens_seen == 0) return ORC_STATE;
    const double t_all = (double)*tokens_seen;
    uint64_t total = 0;
    for (size_t i = 0; i < e; ++i) total += tokens_routed[i];
    if (total != (uint64_t)top_k * *tokens_seen) return ORC_STATE;
    const double target = (double)k_expected / ((double)top_k * (double)n_ffn);
    for (size_t i = 0; i < e; ++i) delta[i] = 0.0;
    for (size_t i = 0; i < n_ffn; ++i) {
        const double load = (double)tokens_routed[i] / ((double)top_k * t_all);
        delta[i] = *mu * (target - load);
        b[i] += delta[i];
    }
    *mu *= mu_decay;
    for (size_t i = 0; i < e; ++i) tokens_routed[i] = 0;
    *tokens_seen = 0;
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * MoE -- blocks.hpp:226-394
 *
 * moe_forward (blocks.hpp:372-394) = index check, rebuilt probs[t,idx] =
 * (S) gate, moe_block (:341-369) with renormalize=false.  Each expert row
 * y = silu(x_t W_in[e]) W_out[e] depends only on its own token row (mm is
 * row independent, tensor.hpp:95-112), so computing it per slot is bitwise
 * the same as the reference's gathered sub-batch.  The combine follows
 * moe_combine (:226-274): FFN slots in rank order out += (g_ffn*w)*y,
 * zero slots zero_w += w, then out += (g_zero*zero_w)*x if zero_w != 0.
 * `renorm` reproduces moe_block(..., renormalize=true) with probs equal to
 * (S)gates at the selected entries (denominator in rank order, :240-247).
 * ---------------------------------------------------------------------- */
#define ORC_DEFINE_MOE(S, SUF)                                                                     \
    void orc_expert_row_##SUF(const S* xrow, size_t d, const S* w_in, const S* w_out,              \
                              size_t inter, S* h, S* y) {                                          \
        orc_mm_##SUF(xrow, w_in, h, 1, d, inter);                                                  \
        for (size_t i = 0; i < inter; ++i) h[i] = h[i] * orc_sigmoid_##SUF(h[i]);                  \
        orc_mm_##SUF(h, w_out, y, 1, inter, d);                                                    \
    }                                                                                              \
    int orc_moe_forward_##SUF(const S* x, size_t t_count, size_t d, const uint32_t* indices,       \
                              const double* gates, size_t top_k, size_t n_ffn, size_t n_zero,      \
                              const S* const* w_in, const S* const* w_out, size_t inter,           \
                              double gamma_ffn_d, double gamma_zero_d, int renorm, S* out) {       \
        const size_t e_total = n_ffn + n_zero;                                                     \
        for (size_t i = 0; i < t_count * top_k; ++i)                                               \
            if (indices[i] >= e_total) return ORC_STATE;                                           \
        const S gamma_ffn = (S)gamma_ffn_d, gamma_zero = (S)gamma_zero_d;                          \
        S* h = (S*)malloc(ORC_NZ(inter) * sizeof(S));                                        \
        S* y = (S*)malloc(ORC_NZ(d) * sizeof(S));                                                \
        for (size_t t = 0; t < t_count; ++t) {                                                     \
            S* orow = out + t * d;                                                                 \
            const S* xrow = x + t * d;                                                             \
            for (size_t j = 0; j < d; ++j) orow[j] = (S)0;                                         \
            S denom = (S)1;                                                                        \
            if (renorm) {                                                                          \
                S s = (S)0;                                                                        \
                for (size_t sl = 0; sl < top_k; ++sl) s += (S)gates[t * top_k + sl];              \
                denom = s;                                                                         \
            }                                                                                      \
            S zero_w = (S)0;                                                                       \
            for (size_t sl = 0; sl < top_k; ++sl) {                                                \
                const uint32_t e = indices[t * top_k + sl];                                        \
                const S w = (S)gates[t * top_k + sl] / denom;                                      \
                if (e < n_ffn) {                                                                   \
                    orc_expert_row_##SUF(xrow, d, w_in[e], w_out[e], inter, h, y);                 \
                    const S coeff = gamma_ffn * w;                                                 \
                    for (size_t j = 0; j < d; ++j) orow[j] += coeff * y[j];                        \
                } else {                                                                           \
                    zero_w += w;                                                                   \
                }                                                                                  \
            }                                                                                      \
            if (zero_w != (S)0) {                                                                  \
                const S coeff = gamma_zero * zero_w;                                               \
                for (size_t j = 0; j < d; ++j) orow[j] += coeff * xrow[j];                         \
            }                                                                                      \
        }                                                                                          \
        free(h);                                                                                   \
        free(y);                                                                                   \
        return ORC_OK;                                                                             \
    }

ORC_DEFINE_MOE(float, f32)
ORC_DEFINE_MOE(double, f64)

/* blocks.hpp:349-359: expert_tokens[e] ascending t, slot_row = position in it (-1 for zero). */
void orc_permutation(const uint32_t* indices, size_t t_count, size_t top_k, size_t n_ffn,
                     size_t n_zero, uint64_t* counts /*[n_ffn+n_zero]*/, int32_t* slot_row) {
    for (size_t e = 0; e < n_ffn + n_zero; ++e) counts[e] = 0;
    for (size_t t = 0; t < t_count; ++t)
        for (size_t s = 0; s < top_k; ++s) {
            const uint32_t e = indices[t * top_k + s];
            slot_row[t * top_k + s] = e < n_ffn ? (int32_t)counts[e] : -1;
            counts[e]++;
        }
}

/* model.hpp:390-391 (ScMoE dense shortcut branch) with ffn_block
 * (blocks.hpp:397-402): dd = a1 + silu(rmsnorm(a1, g) W_in) W_out. */
int orc_dense_branch_f32(const float* a1, const float* gain, size_t t_count, size_t d,
                         const float* w_in, const float* w_out, size_t inter, float* out) {
    float* xn = (float*)malloc(sizeof(float) * (d + inter + d));
    if (!xn) return ORC_PARAMETER;
    float *h = xn + d, *y = h + inter;
    for (size_t t = 0; t < t_count; ++t) {
        orc_rmsnorm_f32(a1 + t * d, gain, 1, d, 1e-6f, xn);
        orc_expert_row_f32(xn, d, w_in, w_out, inter, h, y);
        for (size_t j = 0; j < d; ++j) out[t * d + j] = a1[t * d + j] + y[j];
    }
    free(xn);
    return ORC_OK;
}

/* model.hpp:394-400 (ScMoE wiring, MoE branch): hmoe = rmsnorm(a1, g);
 * probs = softmax(hmoe W_r); d = route_from_probs(probs); out = a3 + moe(hmoe). */
int orc_scmoe_layer_f32(const float* a1, const float* a3, const float* gain, size_t t_count,
                        size_t d, const float* w_router, size_t n_ffn, size_t n_zero, size_t top_k,
                        size_t k_expected, double mu, const double* bias, const float* const* w_in,
                        const float* const* w_out, size_t inter, double gamma_ffn,
                        double gamma_zero, int renorm, uint32_t* indices, double* gates,
                        uint32_t* ffn_count, float* out) {
    const size_t e = n_ffn + n_zero;
    float* hmoe = (float*)malloc(ORC_NZ(t_count * d) * sizeof(float));
    float* moe = (float*)malloc(ORC_NZ(t_count * d) * sizeof(float));
    float* probs = (float*)malloc(ORC_NZ(t_count * e) * sizeof(float));
    orc_rmsnorm_f32(a1, gain, t_count, d, 1e-6f, hmoe);
    int rc = orc_route_topk_f32(hmoe, t_count, d, w_router, n_ffn, n_zero, top_k, k_expected, mu,
                                bias, indices, gates, ffn_count, probs);
    if (!rc)
        rc = orc_moe_forward_f32(hmoe, t_count, d, indices, gates, top_k, n_ffn, n_zero, w_in,
                                 w_out, inter, gamma_ffn, gamma_zero, renorm, moe);
    if (!rc)
        for (size_t i = 0; i < t_count * d; ++i) out[i] = a3[i] + moe[i];
    free(hmoe);
    free(moe);
    free(probs);
    return rc;
}

/* router.hpp:349-369 simulate_bias_control, S = float, with the router
 * projection given; mean/std per step out (RoutingDecision::mean_ffn/std_ffn,
 * router.hpp:76-86). */
int orc_simulate_bias_control_f32(const float* w, size_t d, size_t n_ffn, size_t n_zero,
                                  size_t top_k, size_t k_expected, double* mu, double mu_decay,
                                  double* b, uint64_t rng_seed, size_t batch_tokens, size_t steps,
                                  double* mean_ffn, double* std_ffn) {
    const size_t e = n_ffn + n_zero;
    float* x = (float*)malloc(batch_tokens * d * sizeof(float));
    uint32_t* idx = (uint32_t*)malloc(batch_tokens * top_k * sizeof(uint32_t));
    double* gates = (double*)malloc(batch_tokens * top_k * sizeof(double));
    uint32_t* cnt = (uint32_t*)malloc(batch_tokens * sizeof(uint32_t));
    uint64_t* routed = (uint64_t*)calloc(e, sizeof(uint64_t));
    double* delta = (double*)malloc(e * sizeof(double));
    uint64_t seen = 0;
    int rc = ORC_OK;
    for (size_t step = 0; step < steps && !rc; ++step) {
        const uint64_t s = orc_stream_seed(rng_seed, step);
        orc_fill_normal_f32(s, 0, batch_tokens * d, x);
        rc = orc_route_topk_f32(x, batch_tokens, d, w, n_ffn, n_zero, top_k, k_expected, *mu, b,
                                idx, gates, cnt, NULL);
        if (rc) break;
        orc_accumulate_counters(idx, batch_tokens, top_k, routed, &seen);
        double m = 0.0;
        for (size_t t = 0; t < batch_tokens; ++t) m += cnt[t];
        m /= (double)batch_tokens;
        double v = 0.0;
        for (size_t t = 0; t < batch_tokens; ++t) v += (cnt[t] - m) * (cnt[t] - m);
        mean_ffn[step] = m;
        std_ffn[step] = sqrt(v / (double)batch_tokens);
        rc = orc_bias_update(n_ffn, n_zero, top_k, k_expected, mu, mu_decay, b, routed, &seen,
                             delta);
    }
    free(x);
    free(idx);
    free(gates);
    free(cnt);
    free(routed);
    free(delta);
    return rc;
}

/* ------------------------------------------------------------------------
 * MLA, S = float -- blocks.hpp:19-26 (mla_scale_factors), :38-58 (MlaParams),
 * :73-102 (mla_block forward value), :129-181 (mla_infer_step);
 * tensor.hpp:197-224 (rope_apply); graph.hpp:396-434 (attention forward).
 * w[8] = w_dq [d,dq], w_uq [dq,H*dhc], w_qr [dq,H*dhr], w_dkv [d,dkv],
 * w_uk [dkv,H*dhc], w_uv [dkv,H*dhc], w_kr [d,dhr], w_o [H*dhc,d].
 * ---------------------------------------------------------------------- */
static int orc_mla_check(size_t d, size_t dq, size_t dkv, size_t heads, size_t dhr) {
    if (d == 0 || dq == 0 || dkv == 0) return ORC_PARAMETER; /* blocks.hpp:21-22 */
    if (heads == 0) return ORC_DIMENSION;                    /* tensor.hpp:202 */
    if (dhr % 2 != 0) return ORC_DIMENSION;                  /* tensor.hpp:204 */
    return ORC_OK;
}

/* rope_apply rows of x [rows, heads*hd] in place at positions pos[r]. */
static void orc_rope_f32(float* x, size_t ld, size_t rows, size_t heads, size_t hd,
                         const size_t* pos, double base) {
    for (size_t r = 0; r < rows; ++r) {
        const double p0 = (double)pos[r];
        float* row = x + r * ld;
        for (size_t h = 0; h < heads; ++h)
            for (size_t p = 0; p < hd / 2; ++p) {
                const double theta = p0 * pow(base, -2.0 * (double)p / (double)hd);
                const float c = (float)cos(theta), s = (float)sin(theta);
                const float a = row[h * hd + 2 * p], b = row[h * hd + 2 * p + 1];
                row[h * hd + 2 * p] = a * c - b * s;
                row[h * hd + 2 * p + 1] = a * s + b * c;
            }
    }
}

/* The per-row projections shared by both paths: cq, ckv (scaled), qc, qr
 * (rotated), kr (rotated), at positions pos[r]. */
static void orc_mla_project(const float* const* w, size_t d, size_t dq, size_t dkv, size_t heads,
                            size_t dhc, size_t dhr, double base, int va, const float* h,
                            size_t rows, const size_t* pos, float* ckv, float* qc, float* qr,
                            float* kr) {
    const float aq = va ? (float)sqrt((double)d / (double)dq) : 1.0f;
    const float akv = va ? (float)sqrt((double)d / (double)dkv) : 1.0f;
    float* cq = (float*)malloc(ORC_NZ(rows * dq) * sizeof(float));
    orc_mm_f32(h, w[0], cq, rows, d, dq);
    for (size_t i = 0; i < rows * dq; ++i) cq[i] *= aq;
    orc_mm_f32(h, w[3], ckv, rows, d, dkv);
    for (size_t i = 0; i < rows * dkv; ++i) ckv[i] *= akv;
    orc_mm_f32(cq, w[1], qc, rows, dq, heads * dhc);
    orc_mm_f32(cq, w[2], qr, rows, dq, heads * dhr);
    orc_rope_f32(qr, heads * dhr, rows, heads, dhr, pos, base);
    orc_mm_f32(h, w[6], kr, rows, d, dhr);
    orc_rope_f32(kr, dhr, rows, 1, dhr, pos, base);
    free(cq);
}

/* Causal attention of query rows (absolute positions q0+i) against keys
 * 0..q0+i of one sequence, head by head, into merged [nq, H*dhc]
 * (graph.hpp:396-434; identical arithmetic in blocks.hpp:155-179). */
static void orc_mla_attend(size_t heads, size_t dhc, size_t dhr, const float* qc, const float* qr,
                           size_t nq, size_t q0, const float* kc, const float* vv,
                           const float* kr, float* merged) {
    const float scale = (float)(1.0 / sqrt((double)(dhc + dhr)));
    float* att = (float*)malloc(ORC_NZ(q0 + nq) * sizeof(float));
    for (size_t i = 0; i < nq; ++i)
        for (size_t h = 0; h < heads; ++h) {
            const size_t n = q0 + i + 1;
            float mx = 0.0f;
            for (size_t j = 0; j < n; ++j) {
                float acc = 0.0f;
                for (size_t t = 0; t < dhc; ++t)
                    acc += qc[i * heads * dhc + h * dhc + t] * kc[j * heads * dhc + h * dhc + t];
                for (size_t t = 0; t < dhr; ++t)
                    acc += qr[i * heads * dhr + h * dhr + t] * kr[j * dhr + t];
                att[j] = acc * scale;
                mx = (j == 0 || att[j] > mx) ? att[j] : mx;
            }
            float denom = 0.0f;
            for (size_t j = 0; j < n; ++j) {
                att[j] = expf(att[j] - mx);
                denom += att[j];
            }
            float* o = merged + i * heads * dhc + h * dhc;
            for (size_t t = 0; t < dhc; ++t) o[t] = 0.0f;
            for (size_t j = 0; j < n; ++j) {
                const float wj = att[j] / denom;
                for (size_t t = 0; t < dhc; ++t) o[t] += wj * vv[j * heads * dhc + h * dhc + t];
            }
        }
    free(att);
}

/* mla_block forward value over packed sequences of seq_len rows. */
int orc_mla_forward_f32(size_t d, size_t dq, size_t dkv, size_t heads, size_t dhc, size_t dhr,
                        double base, int va, const float* const* w, const float* h, size_t rows,
                        size_t seq_len, float* out) {
    int rc = orc_mla_check(d, dq, dkv, heads, dhr);
    if (rc) return rc;
    if (seq_len == 0 || rows % seq_len != 0) return ORC_DIMENSION; /* graph.hpp:404 */
    size_t* pos = (size_t*)malloc(ORC_NZ(rows) * sizeof(size_t));
    for (size_t r = 0; r < rows; ++r) pos[r] = r % seq_len; /* blocks.hpp:64-68 */
    float* ckv = (float*)malloc(ORC_NZ(rows * dkv) * sizeof(float));
    float* qc = (float*)malloc(ORC_NZ(rows * heads * dhc) * sizeof(float));
    float* qr = (float*)malloc(ORC_NZ(rows * heads * dhr) * sizeof(float));
    float* kr = (float*)malloc(ORC_NZ(rows * dhr) * sizeof(float));
    float* kc = (float*)malloc(ORC_NZ(rows * heads * dhc) * sizeof(float));
    float* vv = (float*)malloc(ORC_NZ(rows * heads * dhc) * sizeof(float));
    float* merged = (float*)malloc(ORC_NZ(rows * heads * dhc) * sizeof(float));
    orc_mla_project(w, d, dq, dkv, heads, dhc, dhr, base, va, h, rows, pos, ckv, qc, qr, kr);
    orc_mm_f32(ckv, w[4], kc, rows, dkv, heads * dhc);
    orc_mm_f32(ckv, w[5], vv, rows, dkv, heads * dhc);
    for (size_t s0 = 0; s0 < rows; s0 += seq_len)
        orc_mla_attend(heads, dhc, dhr, qc + s0 * heads * dhc, qr + s0 * heads * dhr, seq_len, 0,
                       kc + s0 * heads * dhc, vv + s0 * heads * dhc, kr + s0 * dhr,
                       merged + s0 * heads * dhc);
    orc_mm_f32(merged, w[7], out, rows, heads * dhc, d);
    free(pos); free(ckv); free(qc); free(qr); free(kr); free(kc); free(vv); free(merged);
    return ORC_OK;
}

/* mla_infer_step for positions 0..T-1 of one sequence: out [T,d] and the
 * final cache (c_kv [T,dkv], k_r [T,dhr]).  Each step re-expands the whole
 * cache as the reference does (blocks.hpp:149-150). */
int orc_mla_infer_f32(size_t d, size_t dq, size_t dkv, size_t heads, size_t dhc, size_t dhr,
                      double base, int va, const float* const* w, const float* h, size_t T,
                      float* out, float* c_kv, float* k_r) {
    int rc = orc_mla_check(d, dq, dkv, heads, dhr);
    if (rc) return rc;
    float* qc = (float*)malloc(ORC_NZ(heads * dhc) * sizeof(float));
    float* qr = (float*)malloc(ORC_NZ(heads * dhr) * sizeof(float));
    float* kc = (float*)malloc(ORC_NZ(T * heads * dhc) * sizeof(float));
    float* vv = (float*)malloc(ORC_NZ(T * heads * dhc) * sizeof(float));
    float* merged = (float*)malloc(ORC_NZ(heads * dhc) * sizeof(float));
    for (size_t t = 0; t < T; ++t) {
        orc_mla_project(w, d, dq, dkv, heads, dhc, dhr, base, va, h + t * d, 1, &t,
                        c_kv + t * dkv, qc, qr, k_r + t * dhr);
        orc_mm_f32(c_kv, w[4], kc, t + 1, dkv, heads * dhc);
        orc_mm_f32(c_kv, w[5], vv, t + 1, dkv, heads * dhc);
        orc_mla_attend(heads, dhc, dhr, qc, qr, 1, t, kc, vv, k_r, merged);
        orc_mm_f32(merged, w[7], out + t * d, 1, heads * dhc, d);
    }
    free(qc); free(qr); free(kc); free(vv); free(merged);
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * moe_forward (blocks.hpp:372-394) for a token sample of a bank that does not
 * fit host RAM (configs B/C: 512 experts x 100 MB in fp32).  TEST
 * INFRASTRUCTURE: the parity tests call this at the headline shapes.
 *
 * Expert e's weights are regenerated from the synthetic recipe (SURVEY.md
 * 8d): w_in = seeded_init Uniform of CounterRng(seed).stream(stream0 + 2e),
 * w_out = stream(stream0 + 2e + 1) (rng.hpp:89-94), rounded to bf16 (RNE)
 * when `bf16` is set, as the device bank stores them.  Every slot row
 * y = silu(x_t W_in) W_out is computed with orc_mm_f32 over the sampled rows
 * routed to e (row independent, tensor.hpp:95-112, so bitwise the per-slot
 * orc_expert_row_f32), experts spread over `threads` workers; then the
 * rank-order combine of ORC_DEFINE_MOE (moe_combine, blocks.hpp:251-274).
 * ---------------------------------------------------------------------- */
typedef struct {
    const float* x;
    size_t t_count, d, top_k, n_ffn, inter;
    const uint32_t* indices;
    uint64_t seed, stream0;
    double variance;
    int bf16;
    float* y; /* [t_count * top_k][d] per-slot expert rows */
    atomic_size_t next;
    atomic_int rc;
} OrcStreamJob;

static float orc_bf16_rne(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    memcpy(&v, &u, 4);
    return v;
}

static void* orc_stream_worker(void* arg) {
    OrcStreamJob* j = (OrcStreamJob*)arg;
    const size_t d = j->d, I = j->inter, n_slots = j->t_count * j->top_k;
    float* w_in = (float*)malloc(d * I * sizeof(float));
    float* w_out = (float*)malloc(d * I * sizeof(float));
    size_t* slots = (size_t*)malloc(ORC_NZ(n_slots) * sizeof(size_t));
    float* xs = (float*)malloc(ORC_NZ(n_slots) * d * sizeof(float));
    float* hs = (float*)malloc(ORC_NZ(n_slots) * I * sizeof(float));
    float* ys = (float*)malloc(ORC_NZ(n_slots) * d * sizeof(float));
    if (!w_in || !w_out || !slots || !xs || !hs || !ys) {
        atomic_store(&j->rc, ORC_PARAMETER);
    } else {
        for (;;) {
            const size_t e = atomic_fetch_add(&j->next, 1);
            if (e >= j->n_ffn) break;
            size_t m = 0;
            for (size_t s = 0; s < n_slots; ++s)
                if (j->indices[s] == e) slots[m++] = s;
            if (m == 0) continue;
            orc_seeded_uniform_f32(orc_stream_seed(j->seed, j->stream0 + 2 * e), 0, d * I,
                                   j->variance, w_in);
            orc_seeded_uniform_f32(orc_stream_seed(j->seed, j->stream0 + 2 * e + 1), 0, d * I,
                                   j->variance, w_out);
            if (j->bf16)
                for (size_t i = 0; i < d * I; ++i) {
                    w_in[i] = orc_bf16_rne(w_in[i]);
                    w_out[i] = orc_bf16_rne(w_out[i]);
                }
            for (size_t r = 0; r < m; ++r)
                memcpy(xs + r * d, j->x + (slots[r] / j->top_k) * d, d * sizeof(float));
            orc_mm_f32(xs, w_in, hs, m, d, I);
            for (size_t i = 0; i < m * I; ++i) hs[i] = hs[i] * orc_sigmoid_f32(hs[i]);
            orc_mm_f32(hs, w_out, ys, m, I, d);
            for (size_t r = 0; r < m; ++r)
                memcpy(j->y + slots[r] * d, ys + r * d, d * sizeof(float));
        }
    }
    free(w_in); free(w_out); free(slots); free(xs); free(hs); free(ys);
    return NULL;
}

int orc_moe_forward_streamed_f32(const float* x, size_t t_count, size_t d, const uint32_t* indices,
                                 const double* gates, size_t top_k, size_t n_ffn, size_t n_zero,
                                 size_t inter, uint64_t seed, uint64_t stream0, double variance,
                                 int bf16, double gamma_ffn_d, double gamma_zero_d, int renorm,
                                 int threads, float* out) {
    const size_t e_total = n_ffn + n_zero, n_slots = t_count * top_k;
    for (size_t i = 0; i < n_slots; ++i)
        if (indices[i] >= e_total) return ORC_STATE;
    float* y = (float*)malloc(ORC_NZ(n_slots) * d * sizeof(float));
    if (!y) return ORC_PARAMETER;
    OrcStreamJob job = {x, t_count, d, top_k, n_ffn, inter, indices, seed, stream0, variance,
                        bf16, y};
    atomic_init(&job.next, 0);
    atomic_init(&job.rc, ORC_OK);
    if (threads < 1) threads = 1;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 0; i < threads; ++i) pthread_create(&tid[i], NULL, orc_stream_worker, &job);
    for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
    free(tid);
    int rc = atomic_load(&job.rc);
    if (!rc) {
        const float gamma_ffn = (float)gamma_ffn_d, gamma_zero = (float)gamma_zero_d;
        for (size_t t = 0; t < t_count; ++t) {
            float* orow = out + t * d;
            const float* xrow = x + t * d;
            for (size_t j = 0; j < d; ++j) orow[j] = 0.0f;
            float denom = 1.0f;
            if (renorm) {
                float s = 0.0f;
                for (size_t sl = 0; sl < top_k; ++sl) s += (float)gates[t * top_k + sl];
                denom = s;
            }
            float zero_w = 0.0f;
            for (size_t sl = 0; sl < top_k; ++sl) {
                const uint32_t e = indices[t * top_k + sl];
                const float w = (float)gates[t * top_k + sl] / denom;
                if (e < n_ffn) {
                    const float coeff = gamma_ffn * w;
                    const float* yr = y + (t * top_k + sl) * d;
                    for (size_t j = 0; j < d; ++j) orow[j] += coeff * yr[j];
                } else {
                    zero_w += w;
                }
            }
            if (zero_w != 0.0f) {
                const float coeff = gamma_zero * zero_w;
                for (size_t j = 0; j < d; ++j) orow[j] += coeff * xrow[j];
            }
        }
    }
    free(y);
    return rc;
}
