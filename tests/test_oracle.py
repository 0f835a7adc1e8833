"""CPU tests: pin the oracle (oracle/scmoe_oracle.c) to the reference.

(a) the reference's own golden vectors and known answers
    (tests/test_router.cpp, tests/test_blocks.cpp, tests/test_core.cpp);
(b) the reference itself, compiled from its headers (oracle/_ref), bitwise on
    seeded inputs at the tiny config and at LongCat router width;
(c) the committed golden fixtures (tests/golden/, made by make_golden.py).
"""
import os
import subprocess

import numpy as np
import pytest

import _oracle as O
from _oracle import ptr, ptr_array

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def route_from_probs_f64(orc, probs, n, z, k, ke, b=None, mu=0.1):
    probs = np.ascontiguousarray(probs, np.float64)
    T = probs.shape[0]
    b = np.zeros(n + z) if b is None else np.asarray(b, np.float64)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k, np.float64)
    c = np.empty(T, np.uint32)
    rc = orc.orc_route_from_probs_f64(ptr(probs), T, n, z, k, ke, mu, ptr(b), ptr(idx), ptr(g),
                                      ptr(c))
    return rc, idx, g, c


# ---- (a) reference golden vectors -------------------------------------------------
def test_selection_is_biased_gates_are_not(orc):
    # tests/test_router.cpp:26-51
    p = np.array([[0.5, 0.3, 0.2]])
    rc, idx, g, c = route_from_probs_f64(orc, p, 2, 1, 2, 1)
    assert rc == 0 and idx.tolist() == [0, 1] and g.tolist() == [0.5, 0.3] and c.tolist() == [2]
    rc, idx, g, c = route_from_probs_f64(orc, p, 2, 1, 2, 1, b=[-0.4, 0.0, 0.0])
    assert idx.tolist() == [1, 2] and g.tolist() == [0.3, 0.2] and c.tolist() == [1]
    rc, idx, g, c = route_from_probs_f64(orc, p, 2, 1, 2, 1, b=[0.0, 1e9, 0.0])
    assert idx[0] == 1 and g[0] == 0.3
    rc, idx, g, c = route_from_probs_f64(orc, np.array([[0.4, 0.4, 0.2]]), 2, 1, 2, 1)
    assert idx.tolist() == [0, 1]


def test_config_errors(orc):
    # tests/test_router.cpp:88-92
    assert orc.orc_router_validate(2, 1, 4, 1, 0.1, None) == 1
    assert orc.orc_router_validate(2, 0, 2, 1, 0.1, None) == 1
    assert orc.orc_router_validate(2, 1, 2, 2, 0.1, None) == 1
    assert orc.orc_router_validate(2, 1, 2, 1, 0.1, None) == 0
    b = np.array([0.0, 0.0, 0.5])
    assert orc.orc_router_validate(2, 1, 2, 1, 0.1, ptr(b)) == 1  # zero-expert bias


def _bias_update(orc, routed, seen, mu=0.1, decay=1.0, n=2, z=1, k=2, ke=1, b=None):
    E = n + z
    b = np.zeros(E) if b is None else np.array(b, np.float64)
    r = np.array(routed, np.uint64)
    s = np.array([seen], np.uint64)
    m = np.array([mu])
    delta = np.zeros(E)
    rc = orc.orc_bias_update(n, z, k, ke, ptr(m), decay, ptr(b), ptr(r), ptr(s), ptr(delta))
    return rc, delta, b, r, s[0], m[0]


def test_bias_update_rules(orc):
    # tests/test_router.cpp:94-134
    rc, delta, *_ = _bias_update(orc, [50, 50, 100], 100)
    assert rc == 0 and delta.tolist() == [0.0, 0.0, 0.0]
    rc, delta, b, r, s, _ = _bias_update(orc, [80, 70, 50], 100)
    assert abs(delta[0] - -0.015) < 1e-15 and abs(delta[1] - -0.010) < 1e-15 and delta[2] == 0
    assert abs(b[0] - -0.015) < 1e-15 and b[2] == 0.0 and s == 0 and r[0] == 0
    rc, *_, mu = _bias_update(orc, [50, 50, 100], 100, decay=0.5)
    assert abs(mu - 0.05) < 1e-15
    assert _bias_update(orc, [0, 0, 0], 0)[0] == 3  # empty batch -> StateError
    assert _bias_update(orc, [10, 10, 10], 100)[0] == 3  # counters mismatch -> StateError


def test_mm_matches_triple_loop_bitwise(orc):
    # tests/test_core.cpp:53-60 (f64, normal_at inputs)
    a = O.normal_f64(0, 12).reshape(3, 4)
    b = O.normal_f64(1, 8).reshape(4, 2)
    c = np.empty((3, 2))
    orc.orc_mm_f64(ptr(a), ptr(b), ptr(c), 3, 4, 2)
    want = np.zeros((3, 2))
    for i in range(3):
        for j in range(2):
            acc = 0.0
            for k in range(4):
                acc += a[i, k] * b[k, j]
            want[i, j] = acc
    assert (c == want).all()


def test_softmax_basics(orc):
    # tests/test_core.cpp:68-84
    def sm(row):
        x = np.array([row], np.float64)
        y = np.empty_like(x)
        orc.orc_softmax_rows_f64(ptr(x), ptr(y), 1, x.shape[1])
        return y[0]
    assert np.allclose(sm([0.0, 0.0]), [0.5, 0.5], atol=1e-15)
    assert np.allclose(sm([1000.0, 0.0]), [1.0, 0.0], atol=1e-12)
    assert np.allclose(sm(np.log([1.0, 2.0, 3.0])), [1 / 6, 2 / 6, 3 / 6], rtol=1e-12)


def _bank(n, d, I, seed):
    w_in = [O.uniform_f32(O.stream_seed(seed, 2 * e), d * I, 1.0 / d).reshape(d, I) for e in range(n)]
    w_out = [O.uniform_f32(O.stream_seed(seed, 2 * e + 1), I * d, 1.0 / d).reshape(I, d)
             for e in range(n)]
    return w_in, w_out


def test_moe_zero_expert_identity_bitwise(orc):
    # tests/test_blocks.cpp:250-261
    w_in, w_out = _bank(2, 8, 4, 7)
    x = O.normal_f32(11, 24).reshape(3, 8)
    rc, out = O.orc_moe_forward(x, [2, 3, 2], [1.0, 1.0, 1.0], 1, 2, 2, w_in, w_out)
    assert rc == 0 and (out == x).all()


def test_moe_split_zero_gates(orc):
    # tests/test_blocks.cpp:263-275
    w_in, w_out = _bank(2, 8, 4, 7)
    x = O.normal_f32(12, 8).reshape(1, 8)
    rc, out = O.orc_moe_forward(x, [2, 3], [0.25, 0.5], 2, 2, 2, w_in, w_out)
    assert np.allclose(out, 0.75 * x, atol=1e-7)


def test_moe_single_expert_exact(orc):
    # tests/test_blocks.cpp:277-292: unit gate == silu(x W_in) W_out exactly
    w_in, w_out = _bank(2, 8, 4, 9)
    x = O.normal_f32(13, 8).reshape(1, 8)
    rc, out = O.orc_moe_forward(x, [1], [1.0], 1, 2, 0, w_in, w_out)
    h = np.empty((1, 4), np.float32)
    orc.orc_mm_f32(ptr(x), ptr(w_in[1]), ptr(h), 1, 8, 4)
    # sigmoid/silu via the oracle's expf path, computed through a 1-expert moe is the check
    # itself; here verify against the reference composition order with float32 numpy ops.
    hv = h[0].astype(np.float32)
    sig = np.array([np.float32(1) / (np.float32(1) + np.float32(orc.orc_expf(float(-v)))) if v >= 0
                    else np.float32(orc.orc_expf(float(v))) / (np.float32(1) + np.float32(orc.orc_expf(float(v))))
                    for v in hv], np.float32)
    hs = (hv * sig).astype(np.float32).reshape(1, 4)
    want = np.empty((1, 8), np.float32)
    orc.orc_mm_f32(ptr(hs), ptr(w_out[1]), ptr(want), 1, 4, 8)
    assert (out == want).all()


def test_moe_out_of_range_is_state_error(orc):
    # tests/test_blocks.cpp:294-304
    w_in, w_out = _bank(2, 8, 4, 9)
    x = O.normal_f32(14, 8).reshape(1, 8)
    rc, _ = O.orc_moe_forward(x, [4], [1.0], 1, 2, 1, w_in, w_out)
    assert rc == 3


def test_expf_port_matches_libm_strided():
    """The product's glibc-expf restatement vs this host's libm (every 61st
    bit pattern; the GPU test checks the device instantiation exhaustively
    over the softmax/SiLU domain)."""
    src = os.path.join(O.ROOT, "tests", "cpp", "check_expf_port.c")
    exe = os.path.join(O.ORACLE_DIR, "_ref", "check_expf_port")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off",
                    "-I" + os.path.join(O.ROOT, "paper_2509_01322_b200", "csrc"), src, "-o", exe,
                    "-lm"], check=True)
    out = subprocess.run([exe, "61"], capture_output=True, text=True)
    checked, bad, _ = out.stdout.split()
    assert int(checked) > 70_000_000 and int(bad) == 0, out.stdout


def test_exp_port_matches_libm_sampled():
    """The product's glibc-exp (double) restatement vs this host's libm:
    10^7 samples over the whole range, the softmax domain and tiny inputs,
    plus edge values (3e8 were checked when it was written)."""
    src = os.path.join(O.ROOT, "tests", "cpp", "check_exp_port.c")
    exe = os.path.join(O.ORACLE_DIR, "_ref", "check_exp_port")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off",
                    "-I" + os.path.join(O.ROOT, "paper_2509_01322_b200", "csrc"), src, "-o", exe,
                    "-lm"], check=True)
    out = subprocess.run([exe, "10000000"], capture_output=True, text=True)
    checked, bad, _ = out.stdout.split()
    assert int(checked) > 10_000_000 and int(bad) == 0, out.stdout


# ---- (b) oracle == reference, bitwise -------------------------------------------------
def test_rng_matches_reference(orc, ref):
    for s, c in [(0, 0), (7, 123456), (2024, 2**40 + 3)]:
        assert orc.orc_hash2(s, c) == ref.ref_hash2(s, c)
        assert orc.orc_stream_seed(s, c) == ref.ref_stream_seed(s, c)
        assert orc.orc_normal_at(s, c) == ref.ref_normal_at(s, c)
    a = O.uniform_f32(11, 257, 0.3)
    b = np.empty(257, np.float32)
    assert ref.ref_seeded_init_f32(11, 257, 0, 0.3, ptr(b)) == 0
    assert (a == b).all()
    a = np.empty(300)
    b = np.empty(300)
    orc.orc_seeded_tn_f64(3, 300, 1.0 / 64, ptr(a))
    ref.ref_seeded_init_f64(3, 300, 1, 1.0 / 64, ptr(b))
    assert (a == b).all()


def _ref_route_topk(ref, x, w, n, z, k, ke, b, threads=4):
    T, d = x.shape
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    probs = np.empty((T, n + z), np.float32)
    rc = ref.ref_route_topk_f32(ptr(x), T, d, ptr(w), n, z, k, ke, 0.0, ptr(b), ptr(idx), ptr(g),
                                ptr(c), ptr(probs), threads)
    return rc, idx, g, c, probs


@pytest.mark.parametrize("shape", [(512, 256, 8, 4, 2, 1), (64, 6144, 512, 256, 12, 8)])
def test_route_topk_oracle_equals_reference(orc, ref, shape):
    T, d, n, z, k, ke = shape
    x = O.normal_f32(O.stream_seed(99, 0), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(5, 0), d * (n + z), 1.0 / d).reshape(d, n + z)
    b = np.zeros(n + z)
    b[:n] = O.normal_f64(17, n) * 1e-3
    rc1, i1, g1, c1, p1 = O.orc_route_topk(x, w, n, z, k, ke, bias=b, want_probs=True)
    rc2, i2, g2, c2, p2 = _ref_route_topk(ref, x, w, n, z, k, ke, b)
    assert rc1 == rc2 == 0
    assert (i1 == i2).all() and (g1.view(np.uint64) == g2.view(np.uint64)).all()
    assert (c1 == c2).all() and (p1.view(np.uint32) == p2.view(np.uint32)).all()


@pytest.mark.parametrize("gm,m,renorm", [(0, 1, False), (1, 2, False), (2, 3, False)])
def test_moe_forward_oracle_equals_reference(orc, ref, gm, m, renorm):
    T, d, n, z, k, ke, I = 96, 256, 8, 4, 2, 1, 128
    x = O.normal_f32(O.stream_seed(99, 1), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(5, 0), d * (n + z), 1.0 / d).reshape(d, n + z)
    _, idx, g, _, _ = O.orc_route_topk(x, w, n, z, k, ke)
    w_in, w_out = _bank(n, d, I, 21)
    gf = 1.0 if gm == 2 else float(m)
    gz = float(m) if gm == 1 else 1.0
    rc1, o1 = O.orc_moe_forward(x, idx, g, k, n, z, w_in, w_out, gf, gz)
    o2 = np.empty_like(o1)
    rc2 = ref.ref_moe_forward_f32(ptr(x), T, d, ptr(idx), ptr(g), k, n, z, ptr_array(w_in),
                                  ptr_array(w_out), I, m, gm, ptr(o2), 4)
    assert rc1 == rc2 == 0
    assert (o1.view(np.uint32) == o2.view(np.uint32)).all()


@pytest.mark.parametrize("gm,m", [(0, 1), (1, 2), (2, 3)])
def test_moe_forward_f64_oracle_equals_reference(orc, ref, gm, m):
    """moe_forward<double> (ExpertBank<double>): oracle == reference, bitwise."""
    T, d, n, z, k, I = 40, 64, 6, 3, 3, 32
    x = O.normal_f64(41, T * d).reshape(T, d)
    rng = np.random.default_rng(7)
    idx = np.stack([rng.choice(n + z, k, replace=False) for _ in range(T)]).astype(np.uint32).ravel()
    g = rng.uniform(0.01, 0.5, T * k)
    w_in = [O.normal_f64(50 + e, d * I).reshape(d, I) / 8 for e in range(n)]
    w_out = [O.normal_f64(60 + e, I * d).reshape(I, d) / 8 for e in range(n)]
    gf = 1.0 if gm == 2 else float(m)
    gz = float(m) if gm == 1 else 1.0
    o1 = np.empty((T, d))
    assert orc.orc_moe_forward_f64(ptr(x), T, d, ptr(idx), ptr(g), k, n, z, ptr_array(w_in),
                                   ptr_array(w_out), I, gf, gz, 0, ptr(o1)) == 0
    o2 = np.empty_like(o1)
    assert ref.ref_moe_forward_f64(ptr(x), T, d, ptr(idx), ptr(g), k, n, z, ptr_array(w_in),
                                   ptr_array(w_out), I, m, gm, ptr(o2), 4) == 0
    assert (o1.view(np.uint64) == o2.view(np.uint64)).all()


def test_rmsnorm_oracle_equals_reference(orc, ref):
    x = O.normal_f32(3, 8 * 6144).reshape(8, 6144)
    g = O.uniform_f32(4, 6144, 0.1) + np.float32(1)
    o1 = np.empty_like(x)
    o2 = np.empty_like(x)
    orc.orc_rmsnorm_f32(ptr(x), ptr(g), 8, 6144, np.float32(1e-6), ptr(o1))
    assert ref.ref_rmsnorm_f32(ptr(x), ptr(g), 8, 6144, ptr(o2)) == 0
    assert (o1.view(np.uint32) == o2.view(np.uint32)).all()


def test_closed_loop_controller_oracle_equals_reference(orc, ref):
    # tests/test_router.cpp:269-283 shape (fp32 router, 40 steps)
    d, n, z, k, ke = 64, 16, 8, 6, 4
    w = np.empty(d * (n + z), np.float32)
    orc.orc_seeded_tn_f32(7, d * (n + z), 1.0 / 64, ptr(w))
    steps, T = 40, 512
    res = []
    for fn in (orc.orc_simulate_bias_control_f32, ref.ref_simulate_bias_control_f32):
        mu = np.array([0.05])
        b = np.zeros(n + z)
        mean = np.empty(steps)
        std = np.empty(steps)
        assert fn(ptr(w), d, n, z, k, ke, ptr(mu), 0.999, ptr(b), 99, T, steps, ptr(mean),
                  ptr(std)) == 0
        res.append((mean, std, b, mu))
    for a, b in zip(res[0], res[1]):
        assert (np.asarray(a).view(np.uint64) == np.asarray(b).view(np.uint64)).all()


# ---- (c) committed golden fixtures ------------------------------------------------------
def test_oracle_matches_committed_golden(orc):
    path = os.path.join(GOLDEN, "config_a.npz")
    if not os.path.exists(path):
        pytest.skip("golden fixture not generated")
    gd = np.load(path)
    cfg = {k: int(gd[k]) for k in ("T", "d", "n", "z", "k", "ke", "I", "seed_x", "seed_w",
                                   "seed_bank")}
    T, d, n, z, k, ke, I = (cfg[c] for c in ("T", "d", "n", "z", "k", "ke", "I"))
    x = O.normal_f32(O.stream_seed(cfg["seed_x"], 0), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(cfg["seed_w"], 0), d * (n + z), 1.0 / d).reshape(d, n + z)
    rc, idx, g, c, _ = O.orc_route_topk(x, w, n, z, k, ke)
    assert (idx == gd["indices"]).all() and (g == gd["gates"]).all() and (c == gd["ffn_count"]).all()
    w_in, w_out = _bank(n, d, I, cfg["seed_bank"])
    rc, out = O.orc_moe_forward(x, idx, g, k, n, z, w_in, w_out)
    assert (out.view(np.uint32) == gd["out"].view(np.uint32)).all()


def test_routing_stats_match_reference(orc):
    """mean/std activated FFN (router.hpp:73-86), per-expert
    load (stats.hpp:64-67), LB group frequencies (router.hpp:193-216)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = O.ref()
    for (T, k, n, z, ke, g) in [(1000, 12, 64, 32, 8, 8), (257, 6, 24, 12, 4, 3),
                                (5, 2, 8, 0, 2, 4), (0, 2, 8, 4, 1, 2)]:
        idx, cnt = O.random_decision(T + 1, T, k, n, z)
        a = O.routing_stats(orc.orc_routing_stats, idx, cnt, k, n, z, ke, g)
        b = O.routing_stats(ref.ref_routing_stats, idx, cnt, k, n, z, ke, g)
        assert a[0] == b[0] == 0
        assert np.float64(a[1]).tobytes() == np.float64(b[1]).tobytes()
        assert np.float64(a[2]).tobytes() == np.float64(b[2]).tobytes()
        assert a[3].tobytes() == b[3].tobytes() and a[4].tobytes() == b[4].tobytes()
    # LbLossConfig::validate: groups must divide n_ffn -> ConfigError
    idx, cnt = O.random_decision(1, 10, 2, 8, 4)
    assert O.routing_stats(orc.orc_routing_stats, idx, cnt, 2, 8, 4, 1, 3)[0] == 1
    assert O.routing_stats(ref.ref_routing_stats, idx, cnt, 2, 8, 4, 1, 3)[0] == 1


@pytest.mark.parametrize("shape", [(512, 256, 8, 4, 2, 1), (48, 6144, 512, 256, 12, 8)])
def test_route_topk_f64_oracle_equals_reference(orc, ref, shape):
    """RouterState<double>: projection in double, softmax with libm exp."""
    T, d, n, z, k, ke = shape
    x = O.normal_f64(O.stream_seed(98, 0), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(6, 0), d * (n + z), 1.0 / d).astype(np.float64).reshape(d, n + z)
    b = np.zeros(n + z)
    b[:n] = O.normal_f64(18, n) * 1e-3
    rc1, i1, g1, c1, p1 = O.orc_route_topk_f64(x, w, n, z, k, ke, bias=b)
    i2 = np.empty(T * k, np.uint32)
    g2 = np.empty(T * k)
    c2 = np.empty(T, np.uint32)
    p2 = np.empty((T, n + z))
    rc2 = ref.ref_route_topk_f64(ptr(x), T, d, ptr(w), n, z, k, ke, 0.0, ptr(b), ptr(i2), ptr(g2),
                                 ptr(c2), ptr(p2), 4)
    assert rc1 == rc2 == 0
    assert (i1 == i2).all() and (g1.view(np.uint64) == g2.view(np.uint64)).all()
    assert (c1 == c2).all() and (p1.view(np.uint64) == p2.view(np.uint64)).all()


@pytest.mark.parametrize("bf16,renorm,gm,m", [(False, False, 0, 1), (True, False, 0, 1),
                                               (False, True, 1, 2)])
def test_streamed_moe_oracle_equals_reference(orc, ref, bf16, renorm, gm, m):
    """The per-expert streamed moe_forward (the checker of the headline-shape
    GPU tests, whose 512-expert fp32 bank does not fit host RAM) is bitwise
    the reference's moe_forward on the same (bf16-rounded) weights."""
    T, d, n, z, k, ke, I, seed = 80, 256, 8, 4, 3, 2, 128, 41
    x = O.normal_f32(O.stream_seed(98, 1), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(5, 0), d * (n + z), 1.0 / d).reshape(d, n + z)
    _, idx, g, _, _ = O.orc_route_topk(x, w, n, z, k, ke)
    rnd = O.bf16_round if bf16 else (lambda a: a)
    w_in = [rnd(O.uniform_f32(O.stream_seed(seed, 100 + 2 * e), d * I, 1.0 / d)).reshape(d, I)
            for e in range(n)]
    w_out = [rnd(O.uniform_f32(O.stream_seed(seed, 101 + 2 * e), I * d, 1.0 / d)).reshape(I, d)
             for e in range(n)]
    gf = 1.0 if gm == 2 else float(m)
    gz = float(m) if gm == 1 else 1.0
    rc1, o1 = O.orc_moe_forward_streamed(x, idx, g, k, n, z, I, seed, bf16=bf16, gamma_ffn=gf,
                                         gamma_zero=gz, renorm=renorm, threads=3)
    rc2, o2 = O.orc_moe_forward(x, idx, g, k, n, z, w_in, w_out, gf, gz, renorm)
    assert rc1 == rc2 == 0
    assert (o1.view(np.uint32) == o2.view(np.uint32)).all()
    if not renorm:
        o3 = np.empty_like(o1)
        assert ref.ref_moe_forward_f32(ptr(x), T, d, ptr(idx), ptr(g), k, n, z, ptr_array(w_in),
                                       ptr_array(w_out), I, m, gm, ptr(o3), 4) == 0
        assert (o1.view(np.uint32) == o3.view(np.uint32)).all()
