// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the reference's own templates, compiled from the
// headers where they lie (/root/reference/proj/include, never copied) into
// oracle/_ref/libmoelab_ref.so by oracle/Makefile.  Used (a) to pin the C
// restatement oracle/scmoe_oracle.c, (b) as bench.py's `--impl reference` arm
// and cpu_baseline ("kind": "reference"), token-sharded across host threads
// (routing, expert rows and combine are per-token independent, so sharding is
// bitwise identical to one monolithic call).
//
// Error codes: 0 ok, 1 ConfigError, 2 DimensionError, 3 StateError,
// 4 ParameterError, 5 other.

#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "moelab/blocks.hpp"
#include "moelab/graph.hpp"
#include "moelab/param.hpp"
#include "moelab/rng.hpp"
#include "moelab/router.hpp"
#include "moelab/tensor.hpp"

using namespace moelab;

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (const DimensionError&) {
        return 2;
    } catch (const StateError&) {
        return 3;
    } catch (const ParameterError&) {
        return 4;
    } catch (...) {
        return 5;
    }
}

template <typename S>
Tensor<S> wrap(const S* p, std::size_t r, std::size_t c) {
    return Tensor<S>({r, c}, std::vector<S>(p, p + r * c));
}

template <typename S>
RouterState<S> make_state(const S* w, std::size_t d, std::size_t n, std::size_t z, std::size_t k,
                          std::size_t ke, double mu, double decay, const double* b) {
    RouterState<S> st(w ? wrap(w, d, n + z) : Tensor<S>{}, n, z, k, ke, mu, decay);
    if (b) st.b.assign(b, b + n + z);
    return st;
}

void export_decision(const RoutingDecision& d, uint32_t* idx, double* gates, uint32_t* cnt) {
    std::memcpy(idx, d.indices.data(), d.indices.size() * sizeof(uint32_t));
    std::memcpy(gates, d.gates.data(), d.gates.size() * sizeof(double));
    std::memcpy(cnt, d.ffn_count.data(), d.ffn_count.size() * sizeof(uint32_t));
}

// Runs fn(t0, t1) over [0, T) in `threads` contiguous shards.
template <typename F>
int sharded(std::size_t T, int threads, F&& fn) {
    if (threads < 1) threads = 1;
    if ((std::size_t)threads > T) threads = T ? (int)T : 1;
    std::vector<int> rcs(threads, 0);
    std::vector<std::thread> pool;
    const std::size_t per = (T + threads - 1) / threads;
    for (int i = 0; i < threads; ++i) {
        const std::size_t t0 = i * per, t1 = std::min(T, t0 + per);
        pool.emplace_back([&, i, t0, t1] {
            if (t0 < t1) rcs[i] = guarded([&] { fn(t0, t1); });
        });
    }
    for (auto& th : pool) th.join();
    for (int rc : rcs)
        if (rc) return rc;
    return 0;
}

}  // namespace

extern "C" {

uint64_t ref_hash2(uint64_t seed, uint64_t ctr) { return CounterRng::hash2(seed, ctr); }
uint64_t ref_stream_seed(uint64_t seed, uint64_t id) { return CounterRng(seed).stream(id).seed(); }
double ref_normal_at(uint64_t seed, uint64_t ctr) { return CounterRng(seed).normal_at(ctr); }

int ref_seeded_init_f32(uint64_t seed, uint64_t n, int truncated_normal, double variance,
                        float* out) {
    return guarded([&] {
        auto t = seeded_init<float>({n},
                                    truncated_normal ? InitDistribution::TruncatedNormal
                                                     : InitDistribution::Uniform,
                                    variance, CounterRng(seed));
        std::memcpy(out, t.data.data(), n * sizeof(float));
    });
}

int ref_seeded_init_f64(uint64_t seed, uint64_t n, int truncated_normal, double variance,
                        double* out) {
    return guarded([&] {
        auto t = seeded_init<double>({n},
                                     truncated_normal ? InitDistribution::TruncatedNormal
                                                      : InitDistribution::Uniform,
                                     variance, CounterRng(seed));
        std::memcpy(out, t.data.data(), n * sizeof(double));
    });
}

int ref_mm_f32(const float* a, const float* b, float* c, std::size_t m, std::size_t k,
               std::size_t n) {
    return guarded([&] {
        auto r = mm(wrap(a, m, k), wrap(b, k, n));
        std::memcpy(c, r.data.data(), m * n * sizeof(float));
    });
}

int ref_softmax_rows_f32(const float* x, float* y, std::size_t rows, std::size_t cols) {
    return guarded([&] {
        auto r = softmax_rows(wrap(x, rows, cols));
        std::memcpy(y, r.data.data(), rows * cols * sizeof(float));
    });
}

float ref_expf(float x) { return std::exp(x); }

int ref_route_topk_f32(const float* x, std::size_t T, std::size_t d, const float* w, std::size_t n,
                       std::size_t z, std::size_t k, std::size_t ke, double mu, const double* b,
                       uint32_t* idx, double* gates, uint32_t* cnt, float* probs_out, int threads) {
    return guarded([&] { make_state(w, d, n, z, k, ke, mu, 1.0, b); }) ?: sharded(T, threads, [&](std::size_t t0, std::size_t t1) {
        RouterState<float> st = make_state(w, d, n, z, k, ke, mu, 1.0, b);
        Tensor<float> probs;
        auto dd = route_topk(wrap(x + t0 * d, t1 - t0, d), st, probs_out ? &probs : nullptr);
        export_decision(dd, idx + t0 * k, gates + t0 * k, cnt + t0);
        if (probs_out)
            std::memcpy(probs_out + t0 * (n + z), probs.data.data(), probs.data.size() * sizeof(float));
    });
}

// route_topk with S = double (RouterState<double>): libm exp in the softmax
int ref_route_topk_f64(const double* x, std::size_t T, std::size_t d, const double* w,
                       std::size_t n, std::size_t z, std::size_t k, std::size_t ke, double mu,
                       const double* b, uint32_t* idx, double* gates, uint32_t* cnt,
                       double* probs_out, int threads) {
    return guarded([&] { make_state(w, d, n, z, k, ke, mu, 1.0, b); }) ?: sharded(T, threads, [&](std::size_t t0, std::size_t t1) {
        RouterState<double> st = make_state(w, d, n, z, k, ke, mu, 1.0, b);
        Tensor<double> probs;
        auto dd = route_topk(wrap(x + t0 * d, t1 - t0, d), st, probs_out ? &probs : nullptr);
        export_decision(dd, idx + t0 * k, gates + t0 * k, cnt + t0);
        if (probs_out)
            std::memcpy(probs_out + t0 * (n + z), probs.data.data(), probs.data.size() * sizeof(double));
    });
}

#define REF_ROUTE_FROM_PROBS(S, SUF)                                                               \
    int ref_route_from_probs_##SUF(const S* probs, std::size_t T, std::size_t n, std::size_t z,    \
                                   std::size_t k, std::size_t ke, double mu, const double* b,      \
                                   uint32_t* idx, double* gates, uint32_t* cnt) {                  \
        return guarded([&] {                                                                       \
            RouterState<S> st = make_state<S>(nullptr, 0, n, z, k, ke, mu, 1.0, b);                \
            auto dd = route_from_probs(wrap(probs, T, n + z), st);                                 \
            export_decision(dd, idx, gates, cnt);                                                  \
        });                                                                                        \
    }
REF_ROUTE_FROM_PROBS(float, f32)
REF_ROUTE_FROM_PROBS(double, f64)

int ref_bias_update(std::size_t n, std::size_t z, std::size_t k, std::size_t ke, double* mu,
                    double mu_decay, double* b, uint64_t* routed, uint64_t* seen, double* delta) {
    return guarded([&] {
        RouterState<double> st(Tensor<double>{}, n, z, k, ke, *mu, mu_decay);
        st.b.assign(b, b + n + z);
        st.tokens_routed.assign(routed, routed + n + z);
        st.tokens_seen = *seen;
        auto dl = bias_update(st);
        std::memcpy(delta, dl.data(), dl.size() * sizeof(double));
        std::memcpy(b, st.b.data(), st.b.size() * sizeof(double));
        std::memcpy(routed, st.tokens_routed.data(), st.tokens_routed.size() * sizeof(uint64_t));
        *seen = st.tokens_seen;
        *mu = st.mu;
    });
}

int ref_accumulate_counters(const uint32_t* idx, std::size_t T, std::size_t n, std::size_t z,
                            std::size_t k, uint64_t* routed, uint64_t* seen) {
    return guarded([&] {
        RouterState<double> st(Tensor<double>{}, n, z, k, k > 1 ? k - 1 : 1, 0.0, 1.0);
        st.tokens_routed.assign(routed, routed + n + z);
        st.tokens_seen = *seen;
        RoutingDecision dd;
        dd.top_k = k;
        dd.n_ffn = n;
        dd.indices.assign(idx, idx + T * k);
        dd.ffn_count.assign(T, 0);
        accumulate_counters(st, dd);
        std::memcpy(routed, st.tokens_routed.data(), (n + z) * sizeof(uint64_t));
        *seen = st.tokens_seen;
    });
}

// Routing statistics: RoutingDecision::mean_ffn/std_ffn (router.hpp:73-86),
// per-expert load as routing_stats_for_tokens computes it (stats.hpp:64-67),
// lb_group_frequencies (router.hpp:193-216).
int ref_routing_stats(const uint32_t* idx, const uint32_t* cnt, std::size_t T, std::size_t k,
                      std::size_t n, std::size_t z, std::size_t ke, std::size_t groups,
                      double* mean, double* sd, double* load, double* lb) {
    return guarded([&] {
        RoutingDecision d;
        d.top_k = k;
        d.n_ffn = n;
        d.indices.assign(idx, idx + T * k);
        d.ffn_count.assign(cnt, cnt + T);
        *mean = d.mean_ffn();
        *sd = d.std_ffn();
        if (load) {
            std::vector<double> l(n + z, 0.0);
            for (auto i : d.indices) l[i] += 1.0;
            for (double& v : l) v /= static_cast<double>(d.indices.size());
            std::memcpy(load, l.data(), l.size() * sizeof(double));
        }
        if (lb) {
            const std::vector<double> f = lb_group_frequencies(d, LbLossConfig{1.0, groups}, n, z, ke);
            std::memcpy(lb, f.data(), f.size() * sizeof(double));
        }
    });
}

// moe_forward (blocks.hpp:372).  Experts whose w_in[e] is NULL are passed as
// empty Parameters (never touched unless routed to, which would throw).
#define REF_MOE_FORWARD(S, SUF)                                                                    \
    int ref_moe_forward_##SUF(const S* x, std::size_t T, std::size_t d, const uint32_t* idx,       \
                              const double* gates, std::size_t k, std::size_t n, std::size_t z,    \
                              const S* const* w_in, const S* const* w_out, std::size_t inter,      \
                              std::size_t m, int gamma_mode, S* out, int threads) {                \
        return sharded(T, threads, [&](std::size_t t0, std::size_t t1) {                           \
            const std::size_t tc = t1 - t0;                                                        \
            std::vector<char> hit(n, 0);                                                           \
            for (std::size_t i = t0 * k; i < t1 * k; ++i)                                          \
                if (idx[i] < n) hit[idx[i]] = 1;                                                   \
            std::vector<Parameter<S>> store(2 * n);                                                \
            ExpertBank<S> bank;                                                                    \
            bank.m = m;                                                                            \
            bank.gamma_mode = gamma_mode == 0 ? GammaMode::FfnOnly                                 \
                              : gamma_mode == 1 ? GammaMode::All : GammaMode::Off;                 \
            for (std::size_t e = 0; e < n; ++e) {                                                  \
                if (hit[e]) {                                                                      \
                    store[2 * e].value = wrap(w_in[e], d, inter);                                  \
                    store[2 * e + 1].value = wrap(w_out[e], inter, d);                             \
                }                                                                                  \
                bank.w_in.push_back(&store[2 * e]);                                                \
                bank.w_out.push_back(&store[2 * e + 1]);                                           \
            }                                                                                      \
            RoutingDecision dd;                                                                    \
            dd.top_k = k;                                                                          \
            dd.n_ffn = n;                                                                          \
            dd.indices.assign(idx + t0 * k, idx + t1 * k);                                         \
            dd.gates.assign(gates + t0 * k, gates + t1 * k);                                       \
            dd.ffn_count.assign(tc, 0);                                                            \
            auto o = moe_forward(wrap(x + t0 * d, tc, d), dd, bank, z);                            \
            std::memcpy(out + t0 * d, o.data.data(), tc * d * sizeof(S));                          \
        });                                                                                        \
    }
REF_MOE_FORWARD(float, f32)
REF_MOE_FORWARD(double, f64)

// Graph::rmsnorm forward (graph.hpp:322-335).
int ref_rmsnorm_f32(const float* x, const float* gain, std::size_t rows, std::size_t d, float* out) {
    return guarded([&] {
        Graph<float> g;
        auto xv = g.input(wrap(x, rows, d));
        auto gv = g.input(Tensor<float>({d}, std::vector<float>(gain, gain + d)));
        auto o = g.rmsnorm(xv, gv);
        std::memcpy(out, g.val(o).data.data(), rows * d * sizeof(float));
    });
}

int ref_simulate_bias_control_f32(const float* w, std::size_t d, std::size_t n, std::size_t z,
                                  std::size_t k, std::size_t ke, double* mu, double mu_decay,
                                  double* b, uint64_t seed, std::size_t T, std::size_t steps,
                                  double* mean_ffn, double* std_ffn) {
    return guarded([&] {
        RouterState<float> st = make_state(w, d, n, z, k, ke, *mu, mu_decay, b);
        auto tr = simulate_bias_control(st, d, T, steps, CounterRng(seed));
        std::memcpy(mean_ffn, tr.mean_ffn.data(), steps * sizeof(double));
        std::memcpy(std_ffn, tr.std_ffn.data(), steps * sizeof(double));
        std::memcpy(b, st.b.data(), (n + z) * sizeof(double));
        *mu = st.mu;
    });
}

// ---- MLA (blocks.hpp:38-181), S = float ---------------------------------------
// w[8] = w_dq, w_uq, w_qr, w_dkv, w_uk, w_uv, w_kr, w_o (row-major Parameter values).
struct RefMla {
    std::vector<Parameter<float>> store;
    MlaParams<float> p;
    RefMla(std::size_t d, std::size_t dq, std::size_t dkv, std::size_t H, std::size_t dhc,
           std::size_t dhr, double base, int va, const float* const* w) {
        p.d_model = d; p.d_q = dq; p.d_kv = dkv; p.n_heads = H; p.d_head_c = dhc;
        p.d_head_r = dhr; p.rope_base = base; p.variance_alignment = va != 0;
        const std::size_t shp[8][2] = {{d, dq}, {dq, H * dhc}, {dq, H * dhr}, {d, dkv},
                                       {dkv, H * dhc}, {dkv, H * dhc}, {d, dhr}, {H * dhc, d}};
        store.reserve(8);
        for (int i = 0; i < 8; ++i)
            store.emplace_back("w", ParamClass::Hidden, wrap(w[i], shp[i][0], shp[i][1]));
        p.w_dq = &store[0]; p.w_uq = &store[1]; p.w_qr = &store[2]; p.w_dkv = &store[3];
        p.w_uk = &store[4]; p.w_uv = &store[5]; p.w_kr = &store[6]; p.w_o = &store[7];
    }
};

// mla_block forward value (blocks.hpp:73-102) over packed sequences; sequences
// are independent, so `threads` shards them (bitwise the monolithic call).
int ref_mla_forward_f32(std::size_t d, std::size_t dq, std::size_t dkv, std::size_t H,
                        std::size_t dhc, std::size_t dhr, double base, int va,
                        const float* const* w, const float* h, std::size_t rows,
                        std::size_t seq_len, float* out, int threads) {
    auto run = [&](std::size_t s0, std::size_t n_rows) {
        RefMla m(d, dq, dkv, H, dhc, dhr, base, va, w);
        Graph<float> g;
        auto hv = g.input(wrap(h + s0 * d, n_rows, d));
        MlaVars<float> v{g.input(m.p.w_dq->value), g.input(m.p.w_uq->value),
                         g.input(m.p.w_qr->value), g.input(m.p.w_dkv->value),
                         g.input(m.p.w_uk->value), g.input(m.p.w_uv->value),
                         g.input(m.p.w_kr->value), g.input(m.p.w_o->value)};
        auto u = mla_block(g, hv, m.p, v, seq_len);
        std::memcpy(out + s0 * d, g.val(u).data.data(), n_rows * d * sizeof(float));
    };
    // malformed packing: one monolithic call raises the reference's own error
    if (seq_len == 0 || rows % seq_len != 0) return guarded([&] { run(0, rows); });
    return sharded(rows / seq_len, threads, [&](std::size_t s0, std::size_t s1) {
        run(s0 * seq_len, (s1 - s0) * seq_len);
    });
}

// mla_infer_step (blocks.hpp:129-181) for positions 0..T-1 of one sequence;
// returns every step's output and the final compressed cache.
int ref_mla_infer_f32(std::size_t d, std::size_t dq, std::size_t dkv, std::size_t H,
                      std::size_t dhc, std::size_t dhr, double base, int va,
                      const float* const* w, const float* h, std::size_t T, float* out,
                      float* c_kv, float* k_r) {
    return guarded([&] {
        RefMla m(d, dq, dkv, H, dhc, dhr, base, va, w);
        MlaCache<float> cache;
        for (std::size_t t = 0; t < T; ++t) {
            auto u = mla_infer_step(m.p, cache, wrap(h + t * d, 1, d), t);
            std::memcpy(out + t * d, u.data.data(), d * sizeof(float));
        }
        if (c_kv && T) std::memcpy(c_kv, cache.c_kv.data.data(), T * dkv * sizeof(float));
        if (k_r && T && dhr) std::memcpy(k_r, cache.k_r.data.data(), T * dhr * sizeof(float));
    });
}

// One mla_infer_step with a cache of `cache_len` rows (the StateError check).
int ref_mla_infer_position_check(std::size_t cache_len, std::size_t position) {
    return guarded([&] {
        const float* w[8] = {nullptr};
        std::vector<float> z(64 * 64, 0.0f);
        for (auto& p : w) p = z.data();
        RefMla m(8, 4, 4, 1, 4, 2, 1.0e4, 1, w);
        MlaCache<float> cache;
        for (std::size_t t = 0; t < cache_len; ++t)
            mla_infer_step(m.p, cache, Tensor<float>({1, 8}), t);
        mla_infer_step(m.p, cache, Tensor<float>({1, 8}), position);
    });
}

}  // extern "C"
