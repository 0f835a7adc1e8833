// The reference's own unit-test cases for the hot path (tests/test_router.cpp,
// tests/test_blocks.cpp), restated against the C++ drop-in header
// include/moelab_b200/moelab.hpp so they run on the B200 through libscmoe.
// Same inputs, same expectations; a tiny CHECK shim replaces Catch2.
// Exit status = number of failed checks.
#include <cmath>
#include <cstdio>

#include "moelab_b200/moelab.hpp"

using namespace moelab;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (cond) {                                                          \
            ++g_pass;                                                        \
        } else {                                                             \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
        }                                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                             \
    do {                                                                     \
        bool thrown = false;                                                 \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const T&) {                                                 \
            thrown = true;                                                   \
        }                                                                    \
        CHECK(thrown);                                                       \
    } while (0)

static RouterState<double> make_state(std::size_t n, std::size_t z, std::size_t k, std::size_t ke,
                                      double mu = 0.1, double decay = 1.0) {
    return RouterState<double>(Tensor<double>{}, n, z, k, ke, mu, decay);
}

static void selection_is_biased_gates_are_not() {  // test_router.cpp:26-51
    auto st = make_state(2, 1, 2, 1);
    auto d = route_from_probs(Tensor<double>::row({0.5, 0.3, 0.2}), st);
    CHECK((d.indices == std::vector<std::uint32_t>{0, 1}));
    CHECK((d.gates == std::vector<double>{0.5, 0.3}));
    CHECK((d.ffn_count == std::vector<std::uint32_t>{2}));
    st.b = {-0.4, 0.0, 0.0};
    d = route_from_probs(Tensor<double>::row({0.5, 0.3, 0.2}), st);
    CHECK((d.indices == std::vector<std::uint32_t>{1, 2}));
    CHECK((d.gates == std::vector<double>{0.3, 0.2}));
    CHECK((d.ffn_count == std::vector<std::uint32_t>{1}));
    st.b = {0.0, 1e9, 0.0};
    d = route_from_probs(Tensor<double>::row({0.5, 0.3, 0.2}), st);
    CHECK(d.indices[0] == 1 && d.gates[0] == 0.3);
    st.b = {0.0, 0.0, 0.0};
    d = route_from_probs(Tensor<double>::row({0.4, 0.4, 0.2}), st);
    CHECK((d.indices == std::vector<std::uint32_t>{0, 1}));
}

static void route_topk_double_full_path() {  // test_router.cpp:53-71 (RouterState<double>)
    CounterRng rng(3);
    const std::size_t d_model = 8, n = 3, z = 2;
    RouterState<double> st(seeded_init<double>({d_model, n + z}, InitDistribution::TruncatedNormal,
                                               0.25, rng.stream(0)),
                           n, z, 3, 2, 0.1, 1.0);
    Tensor<double> x({5, d_model});
    for (std::size_t i = 0; i < x.numel(); ++i) x.data[i] = rng.normal_at(100 + i);
    Tensor<double> probs;
    auto d = route_topk(x, st, &probs);
    auto d2 = route_from_probs(probs, st);
    CHECK(d.indices == d2.indices);
    CHECK(d.gates == d2.gates);
    for (std::size_t t = 0; t < 5; ++t) {
        double s = 0.0;
        for (std::size_t e = 0; e < n + z; ++e) s += probs.at(t, e);
        CHECK(std::fabs(s - 1.0) <= 1e-12);
    }
}

static void config_errors() {  // test_router.cpp:88-92
    CHECK_THROWS_AS(make_state(2, 1, 4, 1), ConfigError);
    CHECK_THROWS_AS(make_state(2, 0, 2, 1), ConfigError);
    CHECK_THROWS_AS(make_state(2, 1, 2, 2), ConfigError);
}

static void bias_update_rules() {  // test_router.cpp:94-134
    {
        auto st = make_state(2, 1, 2, 1, 0.1);
        st.tokens_routed = {50, 50, 100};
        st.tokens_seen = 100;
        auto delta = bias_update(st);
        CHECK(delta[0] == 0.0 && delta[1] == 0.0 && delta[2] == 0.0);
    }
    {
        auto st = make_state(2, 1, 2, 1, 0.1);
        st.tokens_routed = {80, 70, 50};
        st.tokens_seen = 100;
        auto delta = bias_update(st);
        CHECK(std::fabs(delta[0] + 0.015) < 1e-15);
        CHECK(std::fabs(delta[1] + 0.010) < 1e-15);
        CHECK(delta[2] == 0.0);
        CHECK(std::fabs(st.b[0] + 0.015) < 1e-15);
        CHECK(st.b[2] == 0.0);
        CHECK(st.tokens_seen == 0 && st.tokens_routed[0] == 0);
    }
    {
        auto st = make_state(2, 1, 2, 1, 0.1, 0.5);
        st.tokens_routed = {50, 50, 100};
        st.tokens_seen = 100;
        bias_update(st);
        CHECK(std::fabs(st.mu - 0.05) < 1e-15);
    }
    {
        auto st = make_state(2, 1, 2, 1);
        CHECK_THROWS_AS(bias_update(st), StateError);
    }
    {
        auto st = make_state(2, 1, 2, 1);
        st.tokens_routed = {10, 10, 10};
        st.tokens_seen = 100;
        CHECK_THROWS_AS(bias_update(st), StateError);
    }
}

struct BankFixture {  // test_blocks.cpp:214-248 (fp32, Uniform init)
    std::vector<Parameter<float>> store;
    ExpertBank<float> bank;
    BankFixture(std::size_t n, std::size_t d, std::size_t inter, std::uint64_t seed) {
        store.reserve(2 * n);
        for (std::size_t e = 0; e < n; ++e) {
            store.emplace_back("in", seeded_init<float>({d, inter}, InitDistribution::Uniform,
                                                         1.0 / d, CounterRng(seed).stream(2 * e)));
            store.emplace_back("out", seeded_init<float>({inter, d}, InitDistribution::Uniform,
                                                          1.0 / d, CounterRng(seed).stream(2 * e + 1)));
        }
        for (std::size_t e = 0; e < n; ++e) {
            bank.w_in.push_back(&store[2 * e]);
            bank.w_out.push_back(&store[2 * e + 1]);
        }
    }
};

static Tensor<float> random_tensor(std::vector<std::size_t> shape, std::uint64_t seed) {
    CounterRng rng(seed);
    Tensor<float> t(std::move(shape));
    for (std::size_t i = 0; i < t.numel(); ++i) t.data[i] = static_cast<float>(rng.normal_at(i));
    return t;
}

static void moe_cases() {  // test_blocks.cpp:250-304
    BankFixture fx(2, 8, 4, 7);
    {
        const Tensor<float> x = random_tensor({3, 8}, 11);
        RoutingDecision d;
        d.top_k = 1;
        d.n_ffn = 2;
        d.indices = {2, 3, 2};
        d.gates = {1.0, 1.0, 1.0};
        d.ffn_count = {0, 0, 0};
        Tensor<float> out = moe_forward(x, d, fx.bank, 2);
        bool same = true;
        for (std::size_t i = 0; i < x.numel(); ++i) same = same && out.data[i] == x.data[i];
        CHECK(same);  // zero-expert identity is bitwise
    }
    {
        const Tensor<float> x = random_tensor({1, 8}, 12);
        RoutingDecision d;
        d.top_k = 2;
        d.n_ffn = 2;
        d.indices = {2, 3};
        d.gates = {0.25, 0.5};
        d.ffn_count = {0};
        Tensor<float> out = moe_forward(x, d, fx.bank, 2);
        bool close = true;
        for (std::size_t i = 0; i < x.numel(); ++i)
            close = close && std::fabs(out.data[i] - 0.75f * x.data[i]) < 1e-6f;
        CHECK(close);
    }
    {
        const Tensor<float> x = random_tensor({1, 8}, 14);
        RoutingDecision d;
        d.top_k = 1;
        d.n_ffn = 2;
        d.indices = {4};
        d.gates = {1.0};
        d.ffn_count = {0};
        CHECK_THROWS_AS(moe_forward(x, d, fx.bank, 1), StateError);
    }
}

static void moe_cases_double() {  // test_blocks.cpp:250-275 with ExpertBank<double>
    std::vector<Parameter<double>> store;
    store.reserve(4);
    ExpertBank<double> bank;
    for (std::size_t e = 0; e < 2; ++e) {
        store.emplace_back("in", seeded_init<double>({8, 4}, InitDistribution::Uniform, 1.0 / 8,
                                                     CounterRng(7).stream(2 * e)));
        store.emplace_back("out", seeded_init<double>({4, 8}, InitDistribution::Uniform, 1.0 / 8,
                                                      CounterRng(7).stream(2 * e + 1)));
    }
    for (std::size_t e = 0; e < 2; ++e) {
        bank.w_in.push_back(&store[2 * e]);
        bank.w_out.push_back(&store[2 * e + 1]);
    }
    CounterRng rng(11);
    Tensor<double> x({3, 8});
    for (std::size_t i = 0; i < x.numel(); ++i) x.data[i] = rng.normal_at(i);
    RoutingDecision d;
    d.top_k = 1;
    d.n_ffn = 2;
    d.indices = {2, 3, 2};
    d.gates = {1.0, 1.0, 1.0};
    d.ffn_count = {0, 0, 0};
    Tensor<double> out = moe_forward(x, d, bank, 2);
    CHECK(out.data == x.data);  // zero-expert identity is bitwise
    Tensor<double> x1({1, 8});
    for (std::size_t i = 0; i < 8; ++i) x1.data[i] = rng.normal_at(100 + i);
    d.top_k = 2;
    d.indices = {2, 3};
    d.gates = {0.25, 0.5};
    d.ffn_count = {0};
    out = moe_forward(x1, d, bank, 2);
    bool close = true;
    for (std::size_t i = 0; i < 8; ++i) close = close && std::fabs(out.data[i] - 0.75 * x1.data[i]) < 1e-12;
    CHECK(close);
}

static void closed_loop_controller() {  // test_router.cpp:269-283 (fp32 router)
    RouterState<float> st(seeded_init<float>({64, 24}, InitDistribution::TruncatedNormal,
                                             1.0 / 64, CounterRng(7)),
                          16, 8, 6, 4, 0.05, 0.999);
    auto trace = simulate_bias_control(st, 64, 512, 220, CounterRng(99));
    double tail = 0.0;
    for (std::size_t i = trace.mean_ffn.size() - 60; i < trace.mean_ffn.size(); ++i)
        tail += trace.mean_ffn[i];
    tail /= 60.0;
    CHECK(std::fabs(tail - 4.0) / 4.0 < 0.05);
    CHECK(trace.std_ffn.back() > 0.25);
    bool zero_fixed = true;
    for (std::size_t i = 16; i < 24; ++i) zero_fixed = zero_fixed && st.b[i] == 0.0;
    CHECK(zero_fixed);
    std::printf("closed loop: tail mean %.4f (target 4)\n", tail);
}

struct MlaFixtureF {  // test_blocks.cpp:27-66, S = float
    std::vector<Parameter<float>> store;
    MlaParams<float> p;
    MlaFixtureF(std::size_t d, std::size_t dq, std::size_t dkv, std::size_t H, std::size_t dhc,
                std::size_t dhr, std::uint64_t seed, bool zero = false) {
        p.d_model = d; p.d_q = dq; p.d_kv = dkv; p.n_heads = H; p.d_head_c = dhc; p.d_head_r = dhr;
        p.rope_base = 1.0e4;
        const std::vector<std::vector<std::size_t>> shp = {{d, dq}, {dq, H * dhc}, {dq, H * dhr},
                                                           {d, dkv}, {dkv, H * dhc}, {dkv, H * dhc},
                                                           {d, dhr}, {H * dhc, d}};
        store.reserve(8);
        for (std::size_t i = 0; i < 8; ++i)
            store.emplace_back("w", zero ? Tensor<float>(shp[i])
                                         : seeded_init<float>(shp[i], InitDistribution::TruncatedNormal,
                                                              1.0 / d, CounterRng(seed).stream(i)));
        p.w_dq = &store[0]; p.w_uq = &store[1]; p.w_qr = &store[2]; p.w_dkv = &store[3];
        p.w_uk = &store[4]; p.w_uv = &store[5]; p.w_kr = &store[6]; p.w_o = &store[7];
    }
};

static void mla_cases() {  // test_blocks.cpp:139-209 with MlaParams<float>
    {
        auto [aq, akv] = mla_scale_factors(6144, 1536, 512);
        CHECK(std::fabs(aq - 2.0) <= 1e-15 && std::fabs(akv - std::sqrt(12.0)) <= 1e-12);
        CHECK_THROWS_AS(mla_scale_factors(0, 1, 1), ParameterError);
    }
    {
        MlaFixtureF fx(32, 8, 4, 4, 8, 4, 0, /*zero=*/true);
        auto u = mla_forward(fx.p, random_tensor({4, 32}, 9), 4);
        bool zero = u.shape == std::vector<std::size_t>{4, 32};
        for (float v : u.data) zero = zero && v == 0.0f;
        CHECK(zero);
    }
    {
        // cached incremental decode == packed forward, bitwise in fp32
        MlaFixtureF fx(16, 8, 4, 2, 6, 4, 3);
        const Tensor<float> h = random_tensor({5, 16}, 1);
        const Tensor<float> want = mla_forward(fx.p, h, 5);
        MlaCache<float> cache;
        bool same = true;
        for (std::size_t t = 0; t < 5; ++t) {
            Tensor<float> row({1, 16});
            for (std::size_t j = 0; j < 16; ++j) row.data[j] = h.at(t, j);
            Tensor<float> u = mla_infer_step(fx.p, cache, row, t);
            for (std::size_t j = 0; j < 16; ++j) same = same && u.data[j] == want.at(t, j);
        }
        CHECK(same);
        CHECK(cache.length() == 5);
        CHECK_THROWS_AS(mla_forward(fx.p, h, 3), DimensionError);
    }
    {
        MlaFixtureF fx(8, 4, 4, 1, 4, 2, 5);
        MlaCache<float> cache;
        Tensor<float> row({1, 8});
        mla_infer_step(fx.p, cache, row, 0);
        CHECK_THROWS_AS(mla_infer_step(fx.p, cache, row, 0), StateError);
        CHECK_THROWS_AS(mla_infer_step(fx.p, cache, row, 5), StateError);
    }
}

// Two weightless states of different shapes, in successive scopes (the second
// may sit at the first's stack address): the device mirror must follow the
// shape, not the address (make_state(2,1,2,1) then make_state(4,2,3,2), as the
// reference's test_router.cpp builds them in separate TEST_CASEs).
static void successive_states_of_different_shape() {
    {
        auto st = make_state(2, 1, 2, 1);
        auto d = route_from_probs(Tensor<double>::row({0.5, 0.3, 0.2}), st);
        CHECK((d.indices == std::vector<std::uint32_t>{0, 1}));
    }
    {
        auto st = make_state(4, 2, 3, 2);
        auto d = route_from_probs(Tensor<double>::row({0.1, 0.3, 0.2, 0.05, 0.25, 0.1}), st);
        CHECK(d.indices.size() == 3);
        CHECK((d.indices == std::vector<std::uint32_t>{1, 4, 2}));
        CHECK((d.gates == std::vector<double>{0.3, 0.25, 0.2}));
        CHECK((d.ffn_count == std::vector<std::uint32_t>{2}));
    }
    {
        auto st = make_state(2, 1, 2, 1);
        auto d = route_from_probs(Tensor<double>::row({0.2, 0.3, 0.5}), st);
        CHECK((d.indices == std::vector<std::uint32_t>{2, 1}));
    }
}

int main() {
    successive_states_of_different_shape();
    route_topk_double_full_path();
    moe_cases_double();
    selection_is_biased_gates_are_not();
    config_errors();
    bias_update_rules();
    moe_cases();
    closed_loop_controller();
    mla_cases();
    std::printf("compat: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
