// moelab_b200/moelab.hpp -- C++ drop-in for the reference's ScMoE hot path.
//
// Mirrors the API of the CPU reference (moelab, proj/include/moelab) for the
// path this project accelerates -- same namespace, type names, function
// signatures, argument meanings and exception types -- and executes it on a
// B200 through the C ABI (include/scmoe.h, libscmoe.so):
//
//   Tensor<S>, Parameter<S>         tensor.hpp:16-87, param.hpp:25-38 (data holders)
//   CounterRng, seeded_init         rng.hpp:15-113 (host, for inputs/weights)
//   RouterState<S>, RoutingDecision router.hpp:20-87
//   select_topk_row                 router.hpp:90-104
//   route_from_probs                router.hpp:107-130
//   route_topk                      router.hpp:133-141       (S = float, double)
//   accumulate_counters             router.hpp:144-150
//   bias_update                     router.hpp:155-176
//   simulate_bias_control           router.hpp:349-369       (S = float)
//   GammaMode, ExpertBank<S>        blocks.hpp:185-213
//   moe_forward                     blocks.hpp:372-394       (S = float, double)
//
// Results equal the reference's bit for bit (fp32 path).  Errors are thrown
// as the reference throws them (ConfigError from RouterState, StateError for
// bad indices / counters, DimensionError for shape mismatches).  Device
// residency: router weights and expert banks are uploaded once per (object,
// weights pointer, version) and cached per thread; call
// moelab::b200::invalidate() after mutating weights in place.
//
// Build: g++ -std=c++17 -I<repo>/include app.cpp -L<repo>/paper_2509_01322_b200 -lscmoe
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../scmoe.h"

namespace moelab {

// ---- errors (common.hpp:11-37) ---------------------------------------------
struct DimensionError : std::runtime_error {
    explicit DimensionError(const std::string& m) : std::runtime_error(m) {}
};
struct ParameterError : std::invalid_argument {
    explicit ParameterError(const std::string& m) : std::invalid_argument(m) {}
};
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct StateError : std::runtime_error {
    explicit StateError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};
inline void check(bool cond, const std::string& msg) {
    if (!cond) throw DimensionError(msg);
}

// ---- data holders ---------------------------------------------------------------
template <typename S>
struct Tensor {
    std::vector<std::size_t> shape;
    std::vector<S> data;
    Tensor() = default;
    explicit Tensor(std::vector<std::size_t> shp) : shape(std::move(shp)) {
        data.assign(numel_of(shape), S(0));
    }
    Tensor(std::vector<std::size_t> shp, std::vector<S> values)
        : shape(std::move(shp)), data(std::move(values)) {
        if (numel_of(shape) != data.size()) throw DimensionError("tensor: shape/data size mismatch");
    }
    static std::size_t numel_of(const std::vector<std::size_t>& s) {
        std::size_t n = 1;
        for (auto v : s) n *= v;
        return n;
    }
    static Tensor row(std::vector<S> v) {
        const std::size_t n = v.size();
        return Tensor({1, n}, std::move(v));
    }
    std::size_t numel() const { return data.size(); }
    std::size_t ndim() const { return shape.size(); }
    std::size_t rows() const {
        check(ndim() == 2, "tensor: rows() on non-2d tensor");
        return shape[0];
    }
    std::size_t cols() const {
        check(ndim() == 2, "tensor: cols() on non-2d tensor");
        return shape[1];
    }
    S& at(std::size_t r, std::size_t c) { return data[r * shape[1] + c]; }
    const S& at(std::size_t r, std::size_t c) const { return data[r * shape[1] + c]; }
    const S* row_ptr(std::size_t r) const { return data.data() + r * shape[1]; }
};

template <typename S>
struct Parameter {
    std::string name;
    Tensor<S> value;
    Tensor<S> grad;
    Parameter() = default;
    Parameter(std::string n, Tensor<S> v) : name(std::move(n)), value(std::move(v)), grad(value.shape) {}
};

// ---- counter RNG (rng.hpp:15-64) ---------------------------------------------
class CounterRng {
  public:
    explicit CounterRng(std::uint64_t seed) : seed_(seed) {}
    static std::uint64_t mix64(std::uint64_t x) {
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdULL;
        x ^= x >> 33;
        x *= 0xc4ceb9fe1a85ec53ULL;
        x ^= x >> 33;
        return x;
    }
    static std::uint64_t hash2(std::uint64_t s, std::uint64_t c) {
        return mix64(mix64(s + 0x9e3779b97f4a7c15ULL) ^ mix64(c + 0xbf58476d1ce4e5b9ULL));
    }
    std::uint64_t seed() const { return seed_; }
    CounterRng stream(std::uint64_t id) const {
        return CounterRng(hash2(seed_, id ^ 0xa5a5a5a5a5a5a5a5ULL));
    }
    std::uint64_t at(std::uint64_t c) const { return hash2(seed_, c); }
    double uniform01_at(std::uint64_t c) const {
        return (static_cast<double>(at(c) >> 11) + 1.0) * 0x1.0p-53;
    }
    double normal_at(std::uint64_t c) const {
        const double u1 = uniform01_at(2 * c), u2 = uniform01_at(2 * c + 1);
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
    }

  private:
    std::uint64_t seed_;
};

enum class InitDistribution { Uniform, TruncatedNormal };

// rng.hpp:82-113 (host; the device bank initialiser reproduces the Uniform case)
template <typename S>
Tensor<S> seeded_init(std::vector<std::size_t> shape, InitDistribution dist, double variance,
                      const CounterRng& rng) {
    if (variance < 0.0) throw ParameterError("seeded_init: variance must be >= 0");
    Tensor<S> t(std::move(shape));
    if (variance == 0.0) return t;
    if (dist == InitDistribution::Uniform) {
        const double hw = std::sqrt(3.0 * variance);
        for (std::size_t i = 0; i < t.numel(); ++i)
            t.data[i] = static_cast<S>((2.0 * rng.uniform01_at(i) - 1.0) * hw);
    } else {
        const double scale = std::sqrt(variance / 0.77374201465191098);
        for (std::size_t i = 0; i < t.numel(); ++i) {
            double z = 0.0;
            bool ok = false;
            for (std::uint64_t a = 0; a < 64; ++a) {
                z = rng.normal_at((static_cast<std::uint64_t>(i) << 6) | a);
                if (z >= -2.0 && z <= 2.0) {
                    ok = true;
                    break;
                }
            }
            t.data[i] = static_cast<S>((ok ? z : 0.0) * scale);
        }
    }
    return t;
}

// ---- device plumbing ---------------------------------------------------------------
namespace b200 {

[[noreturn]] inline void raise(int rc, const char* msg) {
    const std::string m = msg ? msg : "scmoe call failed";
    switch (rc) {
        case SCMOE_ERR_CONFIG: throw ConfigError(m);
        case SCMOE_ERR_DIMENSION: throw DimensionError(m);
        case SCMOE_ERR_STATE: throw StateError(m);
        case SCMOE_ERR_PARAMETER: throw ParameterError(m);
        default: throw DeviceError(m);
    }
}

// One context per thread (the C ABI's threading contract), device from SCMOE_DEVICE.
struct Device {
    scmoe_ctx* ctx = nullptr;
    std::map<const void*, std::pair<std::uint64_t, scmoe_router*>> routers;
    std::map<const void*, std::pair<std::uint64_t, scmoe_bank*>> banks;
    Device() {
        const char* dv = std::getenv("SCMOE_DEVICE");
        const int rc = scmoe_ctx_create(dv ? std::atoi(dv) : 0, &ctx);
        if (rc) raise(rc, "scmoe_ctx_create failed (no B200?)");
    }
    ~Device() {
        for (auto& kv : routers) scmoe_router_destroy(ctx, kv.second.second);
        for (auto& kv : banks) scmoe_bank_destroy(ctx, kv.second.second);
        scmoe_ctx_destroy(ctx);
    }
    void ok(int rc) const {
        if (rc) raise(rc, scmoe_last_error(ctx));
    }
};

inline Device& device() {
    thread_local Device d;
    return d;
}

// Drops every cached device copy (call after mutating weights in place).
inline void invalidate() {
    Device& d = device();
    for (auto& kv : d.routers) scmoe_router_destroy(d.ctx, kv.second.second);
    for (auto& kv : d.banks) scmoe_bank_destroy(d.ctx, kv.second.second);
    d.routers.clear();
    d.banks.clear();
}

inline std::uint64_t fingerprint(const void* p, std::size_t bytes) {
    // identity of the weight buffer: address, size and a hash of EVERY byte, so
    // an in-place update anywhere re-uploads (~2 ms for the 18.9 MB LongCat W_r)
    std::uint64_t h = reinterpret_cast<std::uintptr_t>(p) ^ (bytes * 0x9e3779b97f4a7c15ULL);
    const unsigned char* c = static_cast<const unsigned char*>(p);
    std::size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        std::uint64_t w;
        std::memcpy(&w, c + i, 8);
        h = (h ^ w) * 0x100000001b3ULL;
        h ^= h >> 29;
    }
    for (; i < bytes; ++i) h = (h ^ c[i]) * 0x100000001b3ULL;
    return h;
}

}  // namespace b200

// ---- router (router.hpp:20-176) ------------------------------------------------------
template <typename S>
struct RouterState {
    Tensor<S> w;
    std::vector<double> b;
    std::size_t n_ffn = 0, n_zero = 0, top_k = 0, k_expected = 0;
    double mu = 0.0, mu_decay = 1.0;
    std::vector<std::uint64_t> tokens_routed;
    std::uint64_t tokens_seen = 0;

    RouterState() = default;
    RouterState(Tensor<S> weights, std::size_t n, std::size_t z, std::size_t k, std::size_t ke,
                double mu_, double mu_decay_)
        : w(std::move(weights)), b(n + z, 0.0), n_ffn(n), n_zero(z), top_k(k), k_expected(ke),
          mu(mu_), mu_decay(mu_decay_), tokens_routed(n + z, 0) {
        validate();
    }
    std::size_t n_experts() const { return n_ffn + n_zero; }
    void validate() const {
        if (top_k > n_experts()) throw ConfigError("router: top_k exceeds expert count");
        if (k_expected < 1 || k_expected > top_k)
            throw ConfigError("router: need 1 <= k_expected <= top_k");
        if (n_zero > 0 && k_expected >= top_k)
            throw ConfigError("router: k_expected must be < top_k when zero experts exist");
        if (n_zero < top_k - k_expected)
            throw ConfigError("router: too few zero experts to absorb top_k - k_expected slack");
        if (mu < 0.0) throw ConfigError("router: mu must be >= 0");
        for (std::size_t i = n_ffn; i < b.size(); ++i)
            if (b[i] != 0.0) throw ConfigError("router: zero-expert bias must stay 0");
    }
};

struct RoutingDecision {
    std::size_t top_k = 0;
    std::size_t n_ffn = 0;
    std::vector<std::uint32_t> indices;
    std::vector<double> gates;
    std::vector<std::uint32_t> ffn_count;
    std::size_t tokens() const { return ffn_count.size(); }
    double mean_ffn() const {
        if (ffn_count.empty()) return 0.0;
        double s = 0.0;
        for (auto c : ffn_count) s += c;
        return s / static_cast<double>(ffn_count.size());
    }
    double std_ffn() const {
        if (ffn_count.empty()) return 0.0;
        const double m = mean_ffn();
        double s = 0.0;
        for (auto c : ffn_count) s += (c - m) * (c - m);
        return std::sqrt(s / static_cast<double>(ffn_count.size()));
    }
};

namespace b200 {
// Device mirror of a RouterState: created per state object, weights re-uploaded
// when their fingerprint changes; bias, mu and counters synced every call.
template <typename S>
scmoe_router* router_of(const RouterState<S>& st) {
    Device& d = device();
    const std::size_t dm = st.w.ndim() == 2 ? st.w.rows() : 0;
    // the mirror is keyed on the state's address AND its shape: a state at a
    // reused stack address with another (n_ffn, n_zero, top_k, k_expected, d,
    // S) must never reuse a mirror sized for the previous one
    std::uint64_t fp = dm ? fingerprint(st.w.data.data(), st.w.data.size() * sizeof(S)) : 0x5eed;
    for (std::uint64_t v : {std::uint64_t(st.n_ffn), std::uint64_t(st.n_zero),
                            std::uint64_t(st.top_k), std::uint64_t(st.k_expected),
                            std::uint64_t(dm), std::uint64_t(sizeof(S))})
        fp = CounterRng::hash2(fp, v);
    auto it = d.routers.find(&st);
    scmoe_router* r = nullptr;
    if (it != d.routers.end() && it->second.first == fp) {
        r = it->second.second;
    } else {
        if (it != d.routers.end()) scmoe_router_destroy(d.ctx, it->second.second);
        d.ok(scmoe_router_create(d.ctx, dm, st.n_ffn, st.n_zero, st.top_k, st.k_expected, st.mu,
                                 st.mu_decay, &r));
        if (dm) {
            if constexpr (std::is_same_v<S, float>) {
                d.ok(scmoe_router_set_weights_host(d.ctx, r, st.w.data.data()));
            } else {
                std::vector<float> w32(st.w.data.begin(), st.w.data.end());
                d.ok(scmoe_router_set_weights_host(d.ctx, r, w32.data()));
            }
        }
        d.routers[&st] = {fp, r};
    }
    d.ok(scmoe_router_set_bias_host(d.ctx, r, st.b.data()));
    d.ok(scmoe_router_set_mu(d.ctx, r, st.mu, st.mu_decay));
    d.ok(scmoe_router_set_counters_host(d.ctx, r, st.tokens_routed.data(), st.tokens_seen));
    return r;
}
}  // namespace b200

// router.hpp:90-104
template <typename S>
void select_topk_row(const S* probs, const std::vector<double>& bias, std::size_t n_experts,
                     std::size_t k, std::uint32_t* out_idx) {
    RouterState<S> st(Tensor<S>{}, n_experts, 0, k, k, 0.0, 1.0);
    st.b.assign(bias.begin(), bias.begin() + n_experts);
    Tensor<S> p({1, n_experts}, std::vector<S>(probs, probs + n_experts));
    auto& d = b200::device();
    scmoe_router* r = b200::router_of(st);
    std::vector<double> g(k);
    std::uint32_t c = 0;
    if constexpr (std::is_same_v<S, double>)
        d.ok(scmoe_route_from_probs_f64_host(d.ctx, r, p.data.data(), 1, out_idx, g.data(), &c));
    else
        d.ok(scmoe_route_from_probs_f32_host(d.ctx, r, p.data.data(), 1, out_idx, g.data(), &c));
    scmoe_router_destroy(d.ctx, r);
    d.routers.erase(&st);
}

// router.hpp:107-130
template <typename S>
RoutingDecision route_from_probs(const Tensor<S>& probs, const RouterState<S>& state) {
    state.validate();
    const std::size_t T = probs.rows(), E = state.n_experts();
    check(probs.cols() == E, "route: probs width mismatch");
    RoutingDecision dd;
    dd.top_k = state.top_k;
    dd.n_ffn = state.n_ffn;
    dd.indices.resize(T * state.top_k);
    dd.gates.resize(T * state.top_k);
    dd.ffn_count.resize(T);
    auto& d = b200::device();
    scmoe_router* r = b200::router_of(state);
    if constexpr (std::is_same_v<S, double>)
        d.ok(scmoe_route_from_probs_f64_host(d.ctx, r, probs.data.data(), T, dd.indices.data(),
                                             dd.gates.data(), dd.ffn_count.data()));
    else
        d.ok(scmoe_route_from_probs_f32_host(d.ctx, r, probs.data.data(), T, dd.indices.data(),
                                             dd.gates.data(), dd.ffn_count.data()));
    return dd;
}

// router.hpp:133-141 (S = float: the fp32 hot path; S = double: the projection
// in double and the glibc exp(double) restatement; both bit-exact)
template <typename S>
RoutingDecision route_topk(const Tensor<S>& x, const RouterState<S>& state,
                           Tensor<S>* probs_out = nullptr) {
    check(x.ndim() == 2 && state.w.ndim() == 2, "matmul: operands must be 2-d");
    if (x.cols() != state.w.rows()) throw DimensionError("matmul: inner dims disagree");
    state.validate();
    const std::size_t T = x.rows(), E = state.n_experts();
    RoutingDecision dd;
    dd.top_k = state.top_k;
    dd.n_ffn = state.n_ffn;
    dd.indices.resize(T * state.top_k);
    dd.gates.resize(T * state.top_k);
    dd.ffn_count.resize(T);
    auto& d = b200::device();
    scmoe_router* r = b200::router_of(state);
    Tensor<S> probs;
    if (probs_out) probs = Tensor<S>({T, E});
    if constexpr (std::is_same_v<S, double>)
        d.ok(scmoe_route_topk_f64_host(d.ctx, r, x.data.data(), T, state.w.data.data(),
                                       dd.indices.data(), dd.gates.data(), dd.ffn_count.data(),
                                       probs_out ? probs.data.data() : nullptr));
    else
        d.ok(scmoe_route_topk_host(d.ctx, r, x.data.data(), T, dd.indices.data(), dd.gates.data(),
                                   dd.ffn_count.data(), probs_out ? probs.data.data() : nullptr));
    if (probs_out) *probs_out = std::move(probs);
    return dd;
}

// router.hpp:144-150 (device histogram)
template <typename S>
void accumulate_counters(RouterState<S>& state, const RoutingDecision& dd) {
    auto& d = b200::device();
    scmoe_router* r = b200::router_of(state);
    d.ok(scmoe_accumulate_counters_host(d.ctx, r, dd.indices.data(), dd.tokens()));
    d.ok(scmoe_router_get_counters_host(d.ctx, r, state.tokens_routed.data(), &state.tokens_seen));
}

// router.hpp:155-176 (device controller)
template <typename S>
std::vector<double> bias_update(RouterState<S>& state) {
    if (state.tokens_seen == 0) throw StateError("bias_update: empty batch");
    auto& d = b200::device();
    scmoe_router* r = b200::router_of(state);
    std::vector<double> delta(state.n_experts());
    d.ok(scmoe_bias_update(d.ctx, r, delta.data()));
    d.ok(scmoe_router_get_bias_host(d.ctx, r, state.b.data()));
    d.ok(scmoe_router_get_mu(d.ctx, r, &state.mu, nullptr));
    d.ok(scmoe_router_get_counters_host(d.ctx, r, state.tokens_routed.data(), &state.tokens_seen));
    return delta;
}

struct BiasControlTrace {
    std::vector<double> mean_ffn, std_ffn;
    std::vector<std::vector<double>> bias_history;
};

// router.hpp:349-369
template <typename S>
BiasControlTrace simulate_bias_control(RouterState<S>& state, std::size_t d_model,
                                       std::size_t batch_tokens, std::size_t steps,
                                       const CounterRng& rng, bool keep_bias_history = false) {
    BiasControlTrace tr;
    for (std::size_t step = 0; step < steps; ++step) {
        Tensor<S> x({batch_tokens, d_model});
        scmoe_rng_fill_normal_host(rng.stream(step).seed(), 0, x.numel(), x.data.data(), 8);
        RoutingDecision dd = route_topk(x, state);
        accumulate_counters(state, dd);
        tr.mean_ffn.push_back(dd.mean_ffn());
        tr.std_ffn.push_back(dd.std_ffn());
        bias_update(state);
        if (keep_bias_history) tr.bias_history.push_back(state.b);
    }
    return tr;
}

// ---- MoE (blocks.hpp:185-394) ------------------------------------------------------------
enum class GammaMode { FfnOnly, All, Off };

template <typename S>
struct ExpertBank {
    std::size_t m = 1;
    GammaMode gamma_mode = GammaMode::FfnOnly;
    std::vector<Parameter<S>*> w_in;   // [d_model, inter] each
    std::vector<Parameter<S>*> w_out;  // [inter, d_model] each
    std::size_t n_experts() const { return w_in.size(); }
    double gamma_ffn() const { return gamma_mode == GammaMode::Off ? 1.0 : static_cast<double>(m); }
    double gamma_zero() const { return gamma_mode == GammaMode::All ? static_cast<double>(m) : 1.0; }
};

namespace b200 {
template <typename S>
scmoe_bank* bank_of(const ExpertBank<S>& bank, int precision) {
    Device& d = device();
    const std::size_t n = bank.n_experts();
    check(n > 0, "moe_block: empty expert bank");
    const std::size_t dm = bank.w_in[0]->value.rows(), I = bank.w_in[0]->value.cols();
    std::uint64_t fp = static_cast<std::uint64_t>(precision) * 31 + bank.m * 7 +
                       static_cast<std::uint64_t>(bank.gamma_mode);
    for (std::size_t e = 0; e < n; ++e) {
        fp = CounterRng::hash2(fp, fingerprint(bank.w_in[e]->value.data.data(),
                                               bank.w_in[e]->value.data.size() * sizeof(S)));
        fp = CounterRng::hash2(fp, fingerprint(bank.w_out[e]->value.data.data(),
                                               bank.w_out[e]->value.data.size() * sizeof(S)));
    }
    auto it = d.banks.find(&bank);
    if (it != d.banks.end() && it->second.first == fp) return it->second.second;
    if (it != d.banks.end()) scmoe_bank_destroy(d.ctx, it->second.second);
    scmoe_bank* b = nullptr;
    d.ok(scmoe_bank_create(d.ctx, n, dm, I, precision, bank.m, static_cast<int>(bank.gamma_mode), &b));
    for (std::size_t e = 0; e < n; ++e) {
        const auto& wi = bank.w_in[e]->value;
        const auto& wo = bank.w_out[e]->value;
        check(wi.rows() == dm && wi.cols() == I && wo.rows() == I && wo.cols() == dm,
              "moe_block: expert weight shapes disagree");
        if constexpr (std::is_same_v<S, float>) {
            d.ok(scmoe_bank_set_expert_host(d.ctx, b, e, wi.data.data(), wo.data.data()));
        } else {
            d.ok(scmoe_bank_set_expert_f64_host(d.ctx, b, e, wi.data.data(), wo.data.data()));
        }
    }
    d.banks[&bank] = {fp, b};
    return b;
}
}  // namespace b200

// blocks.hpp:372-394.  S = float: precision SCMOE_PREC_F32_EXACT (bit-exact,
// default) or SCMOE_PREC_BF16 (tcgen05 tensor cores, rel-L2 <= 2e-2);
// S = double: the fp64 bank (bit-exact moe_forward<double>).
template <typename S>
Tensor<S> moe_forward(const Tensor<S>& x, const RoutingDecision& dd, const ExpertBank<S>& bank,
                      std::size_t n_zero, int precision = SCMOE_PREC_F32_EXACT) {
    if constexpr (std::is_same_v<S, double>) precision = SCMOE_PREC_F64_EXACT;
    const std::size_t e_total = bank.n_experts() + n_zero;
    for (auto i : dd.indices)
        if (i >= e_total) throw StateError("moe_forward: expert index out of range");
    check(dd.n_ffn == bank.n_experts(), "moe_block: decision/bank FFN count mismatch");
    const std::size_t T = x.rows(), dm = x.cols();
    Tensor<S> out({T, dm});
    auto& d = b200::device();
    scmoe_bank* b = b200::bank_of(bank, precision);
    if constexpr (std::is_same_v<S, double>)
        d.ok(scmoe_moe_forward_f64_host(d.ctx, b, x.data.data(), T, dd.indices.data(),
                                        dd.gates.data(), dd.top_k, n_zero, 0, nullptr,
                                        out.data.data()));
    else
        d.ok(scmoe_moe_forward_host(d.ctx, b, x.data.data(), T, dd.indices.data(), dd.gates.data(),
                                    dd.top_k, n_zero, 0, nullptr, out.data.data()));
    return out;
}

// ---- multi-head latent attention (blocks.hpp:19-181), S = float ----------------
inline std::pair<double, double> mla_scale_factors(std::size_t d_model, std::size_t d_q,
                                                   std::size_t d_kv) {
    if (d_model == 0 || d_q == 0 || d_kv == 0)
        throw ParameterError("mla_scale_factors: dims must be positive");
    return {std::sqrt(static_cast<double>(d_model) / static_cast<double>(d_q)),
            std::sqrt(static_cast<double>(d_model) / static_cast<double>(d_kv))};
}

template <typename S>
struct MlaParams {
    std::size_t d_model = 0, d_q = 0, d_kv = 0;
    std::size_t n_heads = 0, d_head_c = 0, d_head_r = 0;
    double rope_base = 1.0e6;
    bool variance_alignment = true;
    Parameter<S>* w_dq = nullptr;   // [d_model, d_q]
    Parameter<S>* w_uq = nullptr;   // [d_q, n_heads*d_head_c]
    Parameter<S>* w_qr = nullptr;   // [d_q, n_heads*d_head_r]
    Parameter<S>* w_dkv = nullptr;  // [d_model, d_kv]
    Parameter<S>* w_uk = nullptr;   // [d_kv, n_heads*d_head_c]
    Parameter<S>* w_uv = nullptr;   // [d_kv, n_heads*d_head_c]
    Parameter<S>* w_kr = nullptr;   // [d_model, d_head_r]
    Parameter<S>* w_o = nullptr;    // [n_heads*d_head_c, d_model]
    double alpha_q() const {
        return variance_alignment ? mla_scale_factors(d_model, d_q, d_kv).first : 1.0;
    }
    double alpha_kv() const {
        return variance_alignment ? mla_scale_factors(d_model, d_q, d_kv).second : 1.0;
    }
};

namespace b200 {
// Device copy of an MlaParams<float>, keyed on its address + a weight fingerprint.
inline scmoe_mla* mla_of(const MlaParams<float>& p) {
    static thread_local std::map<const void*, std::pair<std::uint64_t, scmoe_mla*>> cache;
    Device& d = device();
    Parameter<float>* const ws[8] = {p.w_dq, p.w_uq, p.w_qr, p.w_dkv, p.w_uk, p.w_uv, p.w_kr, p.w_o};
    std::uint64_t fp = CounterRng::hash2(p.d_model * 131 + p.d_q * 17 + p.d_kv,
                                         p.n_heads * 1009 + p.d_head_c * 31 + p.d_head_r);
    fp = CounterRng::hash2(fp, static_cast<std::uint64_t>(p.rope_base) * 2 + p.variance_alignment);
    for (auto* w : ws) {
        check(w != nullptr, "mla: missing weight");
        fp = CounterRng::hash2(fp, fingerprint(w->value.data.data(),
                                               w->value.data.size() * sizeof(float)));
    }
    auto it = cache.find(&p);
    if (it != cache.end() && it->second.first == fp) return it->second.second;
    if (it != cache.end()) scmoe_mla_destroy(d.ctx, it->second.second);
    scmoe_mla* m = nullptr;
    d.ok(scmoe_mla_create(d.ctx, p.d_model, p.d_q, p.d_kv, p.n_heads, p.d_head_c, p.d_head_r,
                          p.rope_base, p.variance_alignment ? 1 : 0, &m));
    for (int i = 0; i < 8; ++i) d.ok(scmoe_mla_set_weight_host(d.ctx, m, i, ws[i]->value.data.data()));
    cache[&p] = {fp, m};
    return m;
}
}  // namespace b200

// Value of mla_block (blocks.hpp:73-102) over packed sequences of seq_len rows
// -- what a forward-only caller of the Graph op gets, bitwise.
inline Tensor<float> mla_forward(const MlaParams<float>& p, const Tensor<float>& h,
                                 std::size_t seq_len) {
    check(h.ndim() == 2 && h.cols() == p.d_model, "mla_block: bad input shape");
    Tensor<float> out({h.rows(), p.d_model});
    auto& d = b200::device();
    d.ok(scmoe_mla_forward_host(d.ctx, b200::mla_of(p), h.data.data(), h.rows(), seq_len,
                                out.data.data()));
    return out;
}

// MlaCache (blocks.hpp:106-112): the host mirror of the compressed stream plus
// the device-resident cache the steps run on.
template <typename S>
struct MlaCache {
    Tensor<S> c_kv;  // [n, d_kv]
    Tensor<S> k_r;   // [n, d_head_r], already rotated
    std::shared_ptr<scmoe_mla_cache> dev;
    std::size_t length() const { return c_kv.ndim() == 2 ? c_kv.rows() : 0; }
};

// One decode step at `position` (blocks.hpp:129-181); the cache must hold
// exactly `position` rows.
inline Tensor<float> mla_infer_step(const MlaParams<float>& p, MlaCache<float>& cache,
                                    const Tensor<float>& h_t, std::size_t position) {
    check(h_t.ndim() == 2 && h_t.rows() == 1 && h_t.cols() == p.d_model,
          "mla_infer_step: bad input shape");
    if (cache.length() != position)
        throw StateError("mla_infer_step: cache holds " + std::to_string(cache.length()) +
                         " rows but position is " + std::to_string(position));
    auto& d = b200::device();
    scmoe_mla* m = b200::mla_of(p);
    if (!cache.dev) {
        check(position == 0, "mla_infer_step: cache was filled elsewhere");
        scmoe_mla_cache* k = nullptr;
        d.ok(scmoe_mla_cache_create(d.ctx, m, 256, &k));
        scmoe_ctx* ctx = d.ctx;
        cache.dev = std::shared_ptr<scmoe_mla_cache>(k, [ctx](scmoe_mla_cache* q) {
            scmoe_mla_cache_destroy(ctx, q);
        });
    }
    Tensor<float> out({1, p.d_model});
    d.ok(scmoe_mla_infer_step_host(d.ctx, m, cache.dev.get(), h_t.data.data(), position,
                                   out.data.data()));
    const std::size_t n = position + 1;
    Tensor<float> ckv({n, p.d_kv}), kr({n, p.d_head_r});
    d.ok(scmoe_mla_cache_read_host(d.ctx, m, cache.dev.get(), ckv.data.data(), kr.data.data()));
    cache.c_kv = std::move(ckv);
    cache.k_r = std::move(kr);
    return out;
}

}  // namespace moelab
