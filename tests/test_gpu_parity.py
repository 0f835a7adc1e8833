"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): routing indices / gates / ffn_count and
per-expert counts bit-exact; fp32 layer outputs bit-exact as well (the fp32
kernels replay the reference's operation order; the stated tolerance rel-L2
<= 1e-5 is therefore met with zero error); bf16 tensor-core path rel-L2 <= 2e-2
against the oracle run on the same bf16-rounded weights/inputs widened to fp32.
"""
import os

import numpy as np
import pytest

import _oracle as O
from _oracle import ptr

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
BF16_TOL = 2e-2


def bits32(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def bits64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def make_router(P, d, n, z, k, ke, seed_w=5, sid=0, mu=0.0, decay=1.0, bias=None):
    w = O.uniform_f32(O.stream_seed(seed_w, sid), d * (n + z), 1.0 / d).reshape(d, n + z)
    st = P.RouterState(w, n, z, k, ke, mu, decay)
    if bias is not None:
        st.b = np.asarray(bias, np.float64).copy()
    return st


def make_bank_arrays(n, d, I, seed, bf16=False):
    w_in = [O.uniform_f32(O.stream_seed(seed, 2 * e), d * I, 1.0 / d).reshape(d, I) for e in range(n)]
    w_out = [O.uniform_f32(O.stream_seed(seed, 2 * e + 1), I * d, 1.0 / d).reshape(I, d)
             for e in range(n)]
    if bf16:
        w_in = [O.bf16_round(w) for w in w_in]
        w_out = [O.bf16_round(w) for w in w_out]
    return w_in, w_out


# ---------------------------------------------------------------------------
# glibc-expf restatement on the device, exhaustive over the softmax / SiLU
# domain: every float in [-104, -0] (plus +0 .. 89 and specials).
# ---------------------------------------------------------------------------
def test_device_expf_exhaustive(scmoe):
    P = scmoe
    import ctypes as C
    ctx = P.default_context()
    L = P.lib()
    chunk = 1 << 26
    dev = C.c_void_p()
    ctx._check(L.scmoe_device_alloc(ctx.handle, chunk * 4, C.byref(dev)))
    got = np.empty(chunk, np.float32)
    want = np.empty(chunk, np.float32)
    ranges = [(0x80000000, 0xC2D00000 + 1),  # -0 .. -104
              (0x00000000, 0x42B20000),      # +0 .. 89
              (0xFF800000, 0xFF800001), (0x7F800000, 0x7F800001), (0x7FC00000, 0x7FC00001)]
    bad = 0
    total = 0
    for lo, hi in ranges:
        for first in range(lo, hi, chunk):
            n = min(chunk, hi - first)
            ctx._check(L.scmoe_debug_expf_range(ctx.handle, first, dev, n))
            ctx._check(L.scmoe_copy_d2h(ctx.handle, ptr(got), dev, n * 4))
            O.orc().orc_expf_range(first, n, ptr(want))
            g, w = got[:n].view(np.uint32), want[:n].view(np.uint32)
            nan_both = np.isnan(got[:n]) & np.isnan(want[:n])
            bad += int(np.count_nonzero((g != w) & ~nan_both))
            total += n
    L.scmoe_device_free(ctx.handle, dev)
    assert total > 2_200_000_000
    assert bad == 0


# ---------------------------------------------------------------------------
# Router
# ---------------------------------------------------------------------------
def test_golden_selection_vectors(scmoe):
    # tests/test_router.cpp:26-51 through the device top-k kernel (f64 probs)
    P = scmoe
    st = P.RouterState(None, 2, 1, 2, 1, 0.1, 1.0)
    p = np.array([[0.5, 0.3, 0.2]])
    d = P.route_from_probs(p, st)
    assert d.indices.tolist() == [0, 1] and d.gates.tolist() == [0.5, 0.3]
    assert d.ffn_count.tolist() == [2]
    st.b = np.array([-0.4, 0.0, 0.0])
    d = P.route_from_probs(p, st)
    assert d.indices.tolist() == [1, 2] and d.gates.tolist() == [0.3, 0.2]
    assert d.ffn_count.tolist() == [1]
    st.b = np.array([0.0, 1e9, 0.0])
    d = P.route_from_probs(p, st)
    assert d.indices[0] == 1 and d.gates[0] == 0.3
    st.b = np.zeros(3)
    d = P.route_from_probs(np.array([[0.4, 0.4, 0.2]]), st)
    assert d.indices.tolist() == [0, 1]
    # select_topk_row: ties to lowest index, bias applied in double
    assert P.select_topk_row(np.array([0.2, 0.4, 0.4, 0.1]), [0, 0, 0, 0], 4, 3).tolist() == [1, 2, 0]


def test_config_errors_device(scmoe):
    P = scmoe
    for args in [(2, 1, 4, 1), (2, 0, 2, 1), (2, 1, 2, 2)]:
        with pytest.raises(P.ConfigError):
            P.RouterState(None, *args, 0.1, 1.0)
    import ctypes as C
    ctx = P.default_context()
    h = C.c_void_p()
    assert P.lib().scmoe_router_create(ctx.handle, 8, 2, 1, 4, 1, 0.1, 1.0, C.byref(h)) == 1
    st = P.RouterState(None, 2, 1, 2, 1, 0.1, 1.0)
    st.b = np.array([0.0, 0.0, 0.5])
    with pytest.raises(P.ConfigError):
        P.route_from_probs(np.array([[0.5, 0.3, 0.2]]), st)


@pytest.mark.parametrize("shape", [
    (512, 256, 8, 4, 2, 1),        # config A
    (300, 256, 8, 4, 2, 1),        # ragged token count
    (1, 256, 8, 4, 2, 1),
    (777, 6144, 512, 256, 12, 8),  # LongCat router width, ragged T
])
def test_route_topk_bitwise(scmoe, shape):
    P = scmoe
    T, d, n, z, k, ke = shape
    x = O.normal_f32(O.stream_seed(99, 0), T * d).reshape(T, d)
    bias = np.zeros(n + z)
    bias[:n] = O.normal_f64(17, n) * 1e-3
    st = make_router(P, d, n, z, k, ke, bias=bias)
    probs_l = []
    dg = P.route_topk(x, st, probs_l)
    rc, idx, g, c, probs = O.orc_route_topk(x, st.w, n, z, k, ke, bias=bias, want_probs=True)
    assert rc == 0
    assert (bits32(probs_l[0]) == bits32(probs)).all()
    assert (dg.indices == idx).all()
    assert (bits64(dg.gates) == bits64(g)).all()
    assert (dg.ffn_count == c).all()


def test_route_topk_golden_fixture_longcat(scmoe):
    P = scmoe
    gd = np.load(os.path.join(GOLDEN, "router_longcat.npz"))
    T, d, n, z, k, ke = (int(gd[c]) for c in ("T", "d", "n", "z", "k", "ke"))
    x = O.normal_f32(O.stream_seed(int(gd["seed_x"]), 1), T * d).reshape(T, d)
    st = make_router(P, d, n, z, k, ke, seed_w=int(gd["seed_w"]), sid=1, bias=gd["bias"])
    dg = P.route_topk(x, st)
    assert (dg.indices == gd["indices"]).all()
    assert (bits64(dg.gates) == bits64(gd["gates"])).all()
    assert (dg.ffn_count == gd["ffn_count"]).all()


def test_route_from_probs_f32_matches_oracle(scmoe):
    P = scmoe
    T, n, z, k, ke = 200, 64, 32, 6, 4
    logits = O.normal_f32(3, T * (n + z)).reshape(T, n + z)
    probs = np.empty_like(logits)
    O.orc().orc_softmax_rows_f32(ptr(logits), ptr(probs), T, n + z)
    b = np.zeros(n + z)
    b[:n] = O.normal_f64(5, n) * 1e-2
    st = P.RouterState(None, n, z, k, ke, 0.0, 1.0)
    st.b = b
    dg = P.route_from_probs(probs, st)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    assert O.orc().orc_route_from_probs_f32(ptr(probs), T, n, z, k, ke, 0.0, ptr(b), ptr(idx),
                                            ptr(g), ptr(c)) == 0
    assert (dg.indices == idx).all() and (bits64(dg.gates) == bits64(g)).all()
    assert (dg.ffn_count == c).all()


def test_counters_and_bias_update(scmoe):
    P = scmoe
    # tests/test_router.cpp:94-134 through the device controller
    st = P.RouterState(None, 2, 1, 2, 1, 0.1, 1.0)
    st.tokens_routed = np.array([80, 70, 50], np.uint64)
    st.tokens_seen = 100
    delta = P.bias_update(st)
    assert abs(delta[0] + 0.015) < 1e-15 and abs(delta[1] + 0.010) < 1e-15 and delta[2] == 0.0
    assert abs(st.b[0] + 0.015) < 1e-15 and st.b[2] == 0.0
    assert st.tokens_seen == 0 and int(st.tokens_routed[0]) == 0
    st = P.RouterState(None, 2, 1, 2, 1, 0.1, 0.5)
    st.tokens_routed = np.array([50, 50, 100], np.uint64)
    st.tokens_seen = 100
    assert (P.bias_update(st) == 0).all() and abs(st.mu - 0.05) < 1e-15
    with pytest.raises(P.StateError):
        P.bias_update(P.RouterState(None, 2, 1, 2, 1, 0.1, 1.0))
    st = P.RouterState(None, 2, 1, 2, 1, 0.1, 1.0)
    st.tokens_routed = np.array([10, 10, 10], np.uint64)
    st.tokens_seen = 100
    with pytest.raises(P.StateError):
        P.bias_update(st)
    # per-expert slot counts of a LongCat-width routing == oracle histogram
    T, d, n, z, k, ke = 512, 6144, 512, 256, 12, 8
    x = O.normal_f32(O.stream_seed(7, 3), T * d).reshape(T, d)
    st = make_router(P, d, n, z, k, ke)
    dg = P.route_topk(x, st)
    P.accumulate_counters(st, dg)
    routed = np.zeros(n + z, np.uint64)
    seen = np.zeros(1, np.uint64)
    O.orc().orc_accumulate_counters(ptr(dg.indices), T, k, ptr(routed), ptr(seen))
    assert (st.tokens_routed == routed).all() and st.tokens_seen == T


def test_closed_loop_controller_bitwise(scmoe):
    """simulate_bias_control (router.hpp:349-369) on the device vs the oracle:
    per-step mean/std ffn and the final bias vector, bit for bit."""
    P = scmoe
    d, n, z, k, ke = 64, 16, 8, 6, 4
    w = np.empty(d * (n + z), np.float32)
    O.orc().orc_seeded_tn_f32(7, d * (n + z), 1.0 / 64, ptr(w))
    w = w.reshape(d, n + z)
    steps, T = 60, 512
    st = P.RouterState(w, n, z, k, ke, 0.05, 0.999)
    tr = P.simulate_bias_control(st, d, T, steps, 99)
    mu = np.array([0.05])
    b = np.zeros(n + z)
    mean = np.empty(steps)
    std = np.empty(steps)
    assert O.orc().orc_simulate_bias_control_f32(ptr(w), d, n, z, k, ke, ptr(mu), 0.999, ptr(b),
                                                 99, T, steps, ptr(mean), ptr(std)) == 0
    assert (bits64(tr.mean_ffn) == bits64(mean)).all()
    assert (bits64(tr.std_ffn) == bits64(std)).all()
    assert (bits64(st.b) == bits64(b)).all() and st.mu == mu[0]
    assert (st.b[n:] == 0).all()


# ---------------------------------------------------------------------------
# MoE (exact fp32 path)
# ---------------------------------------------------------------------------
def test_moe_small_golden_cases(scmoe):
    P = scmoe
    w_in, w_out = make_bank_arrays(2, 8, 4, 7)
    bank = P.ExpertBank(w_in, w_out)
    x = O.normal_f32(11, 24).reshape(3, 8)
    d = P.RoutingDecision(1, 2, np.array([2, 3, 2], np.uint32), np.ones(3), np.zeros(3, np.uint32))
    out = P.moe_forward(x, d, bank, 2)
    assert (bits32(out) == bits32(x)).all()  # tests/test_blocks.cpp:250-261
    x1 = O.normal_f32(12, 8).reshape(1, 8)
    d = P.RoutingDecision(2, 2, np.array([2, 3], np.uint32), np.array([0.25, 0.5]),
                          np.zeros(1, np.uint32))
    out = P.moe_forward(x1, d, bank, 2)
    assert np.allclose(out, 0.75 * x1, atol=1e-7)  # :263-275
    d = P.RoutingDecision(1, 2, np.array([4], np.uint32), np.ones(1), np.zeros(1, np.uint32))
    with pytest.raises(P.StateError):  # :294-304
        P.moe_forward(x1, d, bank, 1)
    d = P.RoutingDecision(1, 2, np.array([1], np.uint32), np.ones(1), np.ones(1, np.uint32))
    out = P.moe_forward(x1, d, bank, 0)
    rc, want = O.orc_moe_forward(x1, [1], [1.0], 1, 2, 0, w_in, w_out)
    assert (bits32(out) == bits32(want)).all()  # :277-292


@pytest.mark.parametrize("gamma_mode,m,renorm", [(0, 1, False), (1, 2, False), (2, 3, True),
                                                 (0, 2, True)])
def test_moe_forward_exact_config_a(scmoe, gamma_mode, m, renorm):
    P = scmoe
    T, d, n, z, k, ke, I = 512, 256, 8, 4, 2, 1, 128
    x = O.normal_f32(O.stream_seed(99, 0), T * d).reshape(T, d)
    st = make_router(P, d, n, z, k, ke)
    dg = P.route_topk(x, st)
    w_in, w_out = make_bank_arrays(n, d, I, 21)
    bank = P.ExpertBank(w_in, w_out, m=m, gamma_mode=gamma_mode)
    out = P.moe_forward(x, dg, bank, z, renormalize=renorm)
    rc, want = O.orc_moe_forward(x, dg.indices, dg.gates, k, n, z, w_in, w_out,
                                 bank.gamma_ffn(), bank.gamma_zero(), renorm)
    assert rc == 0
    assert (bits32(out) == bits32(want)).all()


def test_moe_forward_config_a_golden_fixture(scmoe):
    P = scmoe
    gd = np.load(os.path.join(GOLDEN, "config_a.npz"))
    T, d, n, z, k, ke, I = (int(gd[c]) for c in ("T", "d", "n", "z", "k", "ke", "I"))
    x = O.normal_f32(O.stream_seed(int(gd["seed_x"]), 0), T * d).reshape(T, d)
    st = make_router(P, d, n, z, k, ke, seed_w=int(gd["seed_w"]))
    dg = P.route_topk(x, st)
    assert (dg.indices == gd["indices"]).all()
    w_in, w_out = make_bank_arrays(n, d, I, int(gd["seed_bank"]))
    out = P.moe_forward(x, dg, P.ExpertBank(w_in, w_out), z)
    assert (bits32(out) == bits32(gd["out"])).all()


def test_layer_forward_exact(scmoe):
    """ScMoE MoE branch (model.hpp:394-400): rmsnorm -> router -> moe -> +a3."""
    P = scmoe
    T, d, n, z, k, ke, I = 333, 256, 16, 8, 4, 2, 64
    a1 = O.normal_f32(41, T * d).reshape(T, d)
    a3 = O.normal_f32(42, T * d).reshape(T, d)
    gain = (O.uniform_f32(43, d, 0.05) + np.float32(1.0)).astype(np.float32)
    st = make_router(P, d, n, z, k, ke)
    w_in, w_out = make_bank_arrays(n, d, I, 44)
    bank = P.ExpertBank(w_in, w_out, m=2, gamma_mode=P.GammaMode.FfnOnly)
    out, dg = P.scmoe_layer_forward(a1, a3, gain, st, bank)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    want = np.empty((T, d), np.float32)
    rc = O.orc().orc_scmoe_layer_f32(ptr(a1), ptr(a3), ptr(gain), T, d, ptr(st.w), n, z, k, ke,
                                     0.0, ptr(st.b), O.ptr_array(w_in), O.ptr_array(w_out), I,
                                     2.0, 1.0, 0, ptr(idx), ptr(g), ptr(c), ptr(want))
    assert rc == 0
    assert (dg.indices == idx).all() and (dg.ffn_count == c).all()
    assert (bits32(out) == bits32(want)).all()


@pytest.mark.parametrize("T,n,z,k", [(131, 20, 12, 6), (40, 8, 4, 8), (333, 16, 8, 4)])
def test_layer_forward_small_front_edge_values(scmoe, T, n, z, k):
    """The fused small-batch front (rmsnorm + router + softmax / top-K in one
    launch, E <= 32) on edge values -- subnormal products, signed zeros, an
    all-zero row, large rows, non-zero biases with ties, K up to E - 4 --
    bit-exact against the reference composition."""
    P = scmoe
    d, ke, I = 256, max(1, k // 2), 64
    a1 = O.normal_f32(O.stream_seed(61, T), T * d).reshape(T, d)
    a3 = O.normal_f32(O.stream_seed(62, T), T * d).reshape(T, d)
    a1[::3] *= np.float32(2.0 ** -66)
    a1[5 % T] = 0.0
    a1[7 % T, ::2] = -0.0
    a1[9 % T] *= np.float32(2.0 ** 40)
    gain = (O.uniform_f32(63, d, 0.05) + np.float32(1.0)).astype(np.float32)
    bias = np.zeros(n + z)
    bias[:n] = np.round(np.random.default_rng(T).uniform(-0.02, 0.02, n), 3)  # ties
    st = make_router(P, d, n, z, k, ke, bias=bias)
    w_in, w_out = make_bank_arrays(n, d, I, 64)
    bank = P.ExpertBank(w_in, w_out)
    out, dg = P.scmoe_layer_forward(a1, a3, gain, st, bank)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    want = np.empty((T, d), np.float32)
    rc = O.orc().orc_scmoe_layer_f32(ptr(a1), ptr(a3), ptr(gain), T, d, ptr(st.w), n, z, k, ke,
                                     0.0, ptr(st.b), O.ptr_array(w_in), O.ptr_array(w_out), I,
                                     1.0, 1.0, 0, ptr(idx), ptr(g), ptr(c), ptr(want))
    assert rc == 0
    assert (dg.indices == idx).all() and (dg.ffn_count == c).all()
    assert (dg.gates.view(np.uint64) == g.view(np.uint64)).all()
    assert (bits32(out) == bits32(want)).all()


def test_empty_batch_is_a_noop(scmoe):
    P = scmoe
    st = make_router(P, 256, 8, 4, 2, 1)
    dg = P.route_topk(np.zeros((0, 256), np.float32), st)
    assert dg.tokens() == 0


# ---------------------------------------------------------------------------
# bf16 tcgen05 path
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shape", [
    (512, 512, 16, 8, 4, 2, 256),      # small: several tiles per expert
    (200, 1024, 64, 32, 6, 4, 512),    # ragged, many experts with few tokens
    (256, 6144, 8, 4, 3, 2, 2048),     # LongCat widths, K loops of 96 / 32 blocks
])
def test_moe_forward_bf16_tensor_cores(scmoe, shape):
    P = scmoe
    T, d, n, z, k, ke, I = shape
    x = O.bf16_round(O.normal_f32(O.stream_seed(7, 1), T * d)).reshape(T, d)
    st = make_router(P, d, n, z, k, ke)
    dg = P.route_topk(x, st)
    w_in, w_out = make_bank_arrays(n, d, I, 31, bf16=True)
    bank = P.ExpertBank(w_in, w_out, precision=P.PREC_BF16)
    out = P.moe_forward(x, dg, bank, z)
    rc, want = O.orc_moe_forward(x, dg.indices, dg.gates, k, n, z, w_in, w_out)
    assert rc == 0
    err = O.rel_l2(out, want)
    assert err <= BF16_TOL, err
    assert err < 5e-3  # expected ~1e-3 (SURVEY.md 8c measured 7.4e-4)


@pytest.mark.parametrize("T,n,z,k", [(333, 16, 8, 4), (1024, 48, 16, 6), (1, 8, 4, 2),
                                     (1025, 16, 8, 4), (4000, 64, 32, 8)])
def test_permutation_matches_oracle(scmoe, T, n, z, k):
    """moe_block's permutation (blocks.hpp:349-359) on the device -- the one-CTA
    path for small batches (T <= 1024, E <= 64) and the three-pass path --
    equals the oracle: per-expert slot counts and each slot's rank in its
    expert's token list."""
    import torch
    P = scmoe
    rng = np.random.default_rng(T + n)
    idx = np.stack([rng.permutation(n + z)[:k] for _ in range(T)]).astype(np.uint32).reshape(-1)
    ctx = P.default_context()
    idx_d = torch.from_numpy(idx.view(np.int32)).cuda()
    cnt_d = torch.empty(n + z, dtype=torch.int32, device="cuda")
    row_d = torch.empty(T * k, dtype=torch.int32, device="cuda")
    ctx._check(P.lib().scmoe_permutation(ctx.handle, idx_d.data_ptr(), T, k, n, z,
                                         cnt_d.data_ptr(), row_d.data_ptr()))
    ctx.synchronize()
    counts = np.empty(n + z, np.uint64)
    slot_row = np.empty(T * k, np.int32)
    O.orc().orc_permutation(ptr(idx), T, k, n, z, ptr(counts), ptr(slot_row))
    assert (cnt_d.cpu().numpy().astype(np.uint64) == counts).all()
    assert (row_d.cpu().numpy() == slot_row).all()


@pytest.mark.parametrize("case", ["one_expert", "zero_only", "single_token", "max_skew"])
def test_moe_forward_bf16_skewed_routing(scmoe, case):
    """Routing extremes on the tcgen05 path: every token on one expert (many
    token tiles of one expert, every other expert empty), every slot on zero
    experts (no FFN rows: the GEMMs see no tiles), a single token, and all
    tokens on the same K experts."""
    P = scmoe
    d, n, z, k, I = 512, 16, 8, 4, 256
    T = 1 if case == "single_token" else 700
    x = O.bf16_round(O.normal_f32(O.stream_seed(8, 3), T * d)).reshape(T, d)
    rng = np.random.default_rng(5)
    if case == "one_expert":  # slot 0 of every token: FFN expert 3; rest zero experts
        idx = np.stack([np.full(T, 3)] + [n + (np.arange(T) + s) % z for s in range(1, k)], 1)
    elif case == "zero_only":
        idx = np.stack([n + (np.arange(T) + s) % z for s in range(k)], 1)
    elif case == "max_skew":
        idx = np.tile(np.array([5, 9, 0, n + 1]), (T, 1))
    else:
        idx = rng.permutation(n + z)[:k][None, :]
    idx = idx.astype(np.uint32).reshape(-1)
    gates = rng.uniform(0.01, 0.3, T * k)
    dg = P.RoutingDecision(top_k=k, n_ffn=n, indices=idx, gates=gates,
                           ffn_count=(idx.reshape(T, k) < n).sum(1).astype(np.uint32))
    w_in, w_out = make_bank_arrays(n, d, I, 33, bf16=True)
    out = P.moe_forward(x, dg, P.ExpertBank(w_in, w_out, precision=P.PREC_BF16), z)
    rc, want = O.orc_moe_forward(x, idx, gates, k, n, z, w_in, w_out)
    assert rc == 0
    if case == "zero_only":  # identity terms only: exact
        assert out.tobytes() == want.tobytes()
    else:
        assert O.rel_l2(out, want) <= 5e-3, O.rel_l2(out, want)


def test_layer_forward_bf16_routing_exact(scmoe):
    """bf16 GEMM path: routing is still bit-exact (fp32 router), output within
    the bf16 tolerance."""
    P = scmoe
    T, d, n, z, k, ke, I = 384, 1024, 32, 16, 6, 4, 256
    a1 = O.normal_f32(51, T * d).reshape(T, d)
    a3 = O.normal_f32(52, T * d).reshape(T, d)
    st = make_router(P, d, n, z, k, ke)
    w_in, w_out = make_bank_arrays(n, d, I, 53, bf16=True)
    bank = P.ExpertBank(w_in, w_out, precision=P.PREC_BF16)
    out, dg = P.scmoe_layer_forward(a1, a3, None, st, bank)
    ones = np.ones(d, np.float32)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    want = np.empty((T, d), np.float32)
    # oracle on the bf16-rounded rmsnorm output is what the GEMM sees; the
    # identity term uses fp32 hmoe.  Compare the MoE part with a tolerance.
    rc = O.orc().orc_scmoe_layer_f32(ptr(a1), ptr(a3), ptr(ones), T, d, ptr(st.w), n, z, k, ke,
                                     0.0, ptr(st.b), O.ptr_array(w_in), O.ptr_array(w_out), I,
                                     1.0, 1.0, 0, ptr(idx), ptr(g), ptr(c), ptr(want))
    assert rc == 0
    assert (dg.indices == idx).all() and (bits64(dg.gates) == bits64(g)).all()
    err = O.rel_l2(out - a3, want - a3)
    assert err <= BF16_TOL, err


@pytest.mark.parametrize("shape", [(1000, 12, 64, 32, 8, 8), (8192, 12, 512, 256, 8, 16),
                                   (257, 6, 24, 12, 4, 3), (5, 2, 8, 0, 2, 4)])
def test_routing_stats_device_bitwise(scmoe, shape):
    """routing statistics from the device histogram and the
    device-side sequential moments equal the reference's bit for bit."""
    P = scmoe
    T, k, n, z, ke, g = shape
    idx, cnt = O.random_decision(T + 7, T, k, n, z)
    d = P.RoutingDecision(k, n, idx, np.zeros(T * k), cnt)
    st = P.routing_stats(d, z, ke, g)
    rc, mean, std, load, lb = O.routing_stats(O.orc().orc_routing_stats, idx, cnt, k, n, z, ke, g)
    assert rc == 0
    assert np.float64(st["mean_activated_ffn"]).tobytes() == np.float64(mean).tobytes()
    assert np.float64(st["std_activated_ffn"]).tobytes() == np.float64(std).tobytes()
    assert st["per_expert_load"].tobytes() == load.tobytes()
    assert st["lb_group_frequencies"].tobytes() == lb.tobytes()


def test_routing_stats_errors(scmoe):
    P = scmoe
    idx, cnt = O.random_decision(3, 10, 2, 8, 4)
    d = P.RoutingDecision(2, 8, idx, np.zeros(20), cnt)
    with pytest.raises(P.ConfigError):  # LbLossConfig::validate (router.hpp:184-188)
        P.routing_stats(d, 4, 1, 3)
    bad = idx.copy()
    bad[3] = 12
    with pytest.raises(P.StateError):
        P.routing_stats(P.RoutingDecision(2, 8, bad, np.zeros(20), cnt), 4, 1, 2)


@pytest.mark.parametrize("T,d,inter,gain", [(333, 256, 512, False), (200, 512, 256, True)])
def test_dense_ffn_bf16(scmoe, T, d, inter, gain):
    """dense shortcut branch dd = a1 + silu(rmsnorm(a1) W_in) W_out
    (model.hpp:390-391, blocks.hpp:397-402) on the tcgen05 GEMM, vs the oracle
    on the same bf16-rounded weights (rel-L2 of the FFN part <= 5e-3)."""
    import torch
    from paper_2509_01322_b200.layer import DenseFFN
    P = scmoe
    ctx = P.Context(0)
    w_in = O.bf16_round(O.uniform_f32(O.stream_seed(31, 0), d * inter, 1.0 / d)).reshape(d, inter)
    w_out = O.bf16_round(O.uniform_f32(O.stream_seed(31, 1), inter * d, 1.0 / d)).reshape(inter, d)
    a1 = O.normal_f32(O.stream_seed(32, 0), T * d).reshape(T, d)
    g = (1.0 + 0.1 * O.normal_f32(33, d)).astype(np.float32) if gain else None
    dense = DenseFFN(ctx, d, inter, w_in=w_in, w_out=w_out)
    a1_d = torch.from_numpy(a1).cuda()
    g_d = torch.from_numpy(g).cuda() if gain else None
    out_d = torch.empty_like(a1_d)
    dense.forward(a1_d.data_ptr(), g_d.data_ptr() if gain else None, T, out_d.data_ptr())
    ctx.synchronize()
    out = out_d.cpu().numpy()
    want = np.empty_like(a1)
    g_or = g if gain else np.ones(d, np.float32)  # NULL gain on the device = unit gain
    assert O.orc().orc_dense_branch_f32(O.ptr(a1), O.ptr(g_or), T, d, O.ptr(w_in), O.ptr(w_out),
                                        inter, O.ptr(want)) == 0
    err = O.rel_l2(out - a1, want - a1)
    assert err <= 5e-3, err
    with pytest.raises(P.ParameterError):  # not a one-expert bf16 bank
        ctx._check(P.lib().scmoe_dense_ffn(ctx.handle, None, a1_d.data_ptr(), None, T,
                                           out_d.data_ptr()))
    dense.close()


def test_longcat_prefill_full_shape_sampled_tokens(scmoe):
    """The bench workload itself (SURVEY config B: T=8192, d=6144, 512+256
    experts, top-12, bf16 GEMMs, device-initialised weights): the routing of
    sampled tokens is bit-exact and their layer output within the bf16
    tolerance of the oracle run on the same bf16-rounded expert weights
    (regenerated on the host from the same counter-based streams)."""
    import torch
    from paper_2509_01322_b200.layer import LONGCAT, DeviceLayer
    P = scmoe
    s, T, SW = LONGCAT, 8192, 11
    ctx = P.Context(0)
    layer = DeviceLayer(ctx, s, seed=SW)
    a1 = P.fill_normal(P.stream_seed(21, 0), T * s.d).reshape(T, s.d)
    a3 = P.fill_normal(P.stream_seed(22, 0), T * s.d).reshape(T, s.d)
    a1_d, a3_d = torch.from_numpy(a1).cuda(), torch.from_numpy(a3).cuda()
    idx = torch.empty(T * s.top_k, dtype=torch.int32, device="cuda")
    gates = torch.empty(T * s.top_k, dtype=torch.float64, device="cuda")
    cnt = torch.empty(T, dtype=torch.int32, device="cuda")
    out = torch.empty(T, s.d, device="cuda")
    layer.forward(a1_d.data_ptr(), a3_d.data_ptr(), None, T, idx.data_ptr(), gates.data_ptr(),
                  cnt.data_ptr(), out.data_ptr())
    ctx.synchronize()
    idx_h = idx.cpu().numpy().view(np.uint32).reshape(T, s.top_k)
    gates_h = gates.cpu().numpy().reshape(T, s.top_k)
    out_h = out.cpu().numpy()
    w_r = layer.router_weights()
    sample = np.array([0, T - 1])
    # oracle layer on the sampled rows; only the experts the device routed them
    # to are materialised (the routing is asserted bit-exact below)
    ones = np.ones(s.d, np.float32)
    probe_idx = np.empty(len(sample) * s.top_k, np.uint32)
    probe_g = np.empty(len(sample) * s.top_k)
    probe_c = np.empty(len(sample), np.uint32)
    w_in = [None] * s.n_ffn
    w_out = [None] * s.n_ffn
    for e in sorted(set(int(x) for x in idx_h[sample].ravel() if x < s.n_ffn)):
        w_in[e] = O.bf16_round(O.uniform_f32(O.stream_seed(SW, 100 + 2 * e), s.d * s.inter,
                                             1.0 / s.d)).reshape(s.d, s.inter)
        w_out[e] = O.bf16_round(O.uniform_f32(O.stream_seed(SW, 101 + 2 * e), s.inter * s.d,
                                              1.0 / s.d)).reshape(s.inter, s.d)
    want = np.empty((len(sample), s.d), np.float32)
    bias = np.zeros(s.E)
    rc = O.orc().orc_scmoe_layer_f32(
        ptr(np.ascontiguousarray(a1[sample])), ptr(np.ascontiguousarray(a3[sample])), ptr(ones),
        len(sample), s.d, ptr(w_r), s.n_ffn, s.n_zero, s.top_k, s.k_expected, 0.0, ptr(bias),
        O.ptr_array(w_in), O.ptr_array(w_out), s.inter, 1.0, 1.0, 0, ptr(probe_idx),
        ptr(probe_g), ptr(probe_c), ptr(want))
    assert rc == 0
    assert (probe_idx.reshape(-1, s.top_k) == idx_h[sample]).all()
    assert (bits64(probe_g.reshape(-1, s.top_k)) == bits64(gates_h[sample])).all()
    err = O.rel_l2(out_h[sample] - a3[sample], want - a3[sample])
    assert err <= 5e-3, err


@pytest.mark.parametrize("shape", [(512, 256, 8, 4, 2, 1), (301, 256, 8, 4, 2, 1),
                                   (200, 6144, 512, 256, 12, 8)])
def test_route_topk_f64_bitwise(scmoe, shape):
    """route_topk for RouterState<double> (S = double): projection in double,
    softmax with the device glibc exp(double) port -- probabilities, indices,
    gates and counts bitwise equal to the reference (oracle pinned on _ref)."""
    P = scmoe
    T, d, n, z, k, ke = shape
    x = O.normal_f64(O.stream_seed(98, 0), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(6, 0), d * (n + z), 1.0 / d).astype(np.float64).reshape(d, n + z)
    b = np.zeros(n + z)
    b[:n] = O.normal_f64(18, n) * 1e-3
    st = P.RouterState(w, n, z, k, ke, 0.0, 1.0)
    st.b[:] = b
    pl = []
    dg = P.route_topk(x, st, pl)
    rc, idx, g, c, probs = O.orc_route_topk_f64(x, w, n, z, k, ke, bias=b)
    assert rc == 0
    assert (pl[0].view(np.uint64) == probs.view(np.uint64)).all()
    assert (dg.indices == idx).all() and (bits64(dg.gates) == bits64(g)).all()
    assert (dg.ffn_count == c).all()


def test_device_exp_f64_matches_libm(scmoe):
    """The device instantiation of the glibc exp(double) port vs host libm on
    300k inputs over the whole range, the softmax domain and edge values."""
    import ctypes
    import torch
    P = scmoe
    libm = ctypes.CDLL("libm.so.6")
    libm.exp.restype = ctypes.c_double
    libm.exp.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-750, 750, 100_000), rng.uniform(-30, 10, 100_000),
                        -rng.uniform(0, 1e-3, 100_000),
                        [0.0, -0.0, 709.78, 709.79, -708.4, -745.13, -745.14, -746.0, 1e-300,
                         np.inf, -np.inf]])
    want = np.array([libm.exp(float(v)) for v in x])
    ctx = P.Context(0)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    ctx._check(P.lib().scmoe_debug_exp(ctx.handle, xd.data_ptr(), out.data_ptr(), x.size))
    ctx.synchronize()
    got = out.cpu().numpy()
    assert (got.view(np.uint64) == want.view(np.uint64)).all(), \
        int((got.view(np.uint64) != want.view(np.uint64)).sum())


@pytest.mark.parametrize("gamma_mode,m,renorm", [(0, 1, False), (1, 2, True), (2, 3, False)])
def test_moe_forward_f64_bitwise(scmoe, gamma_mode, m, renorm):
    """moe_forward<double> (ExpertBank<double>, S = double): the fp64 expert
    FFN (DMUL/DADD chains, logistic on the exp(double) port) and combine are
    bitwise equal to the reference's double path (oracle f64)."""
    P = scmoe
    T, d, n, z, k, ke, I = 96, 128, 8, 4, 2, 1, 64
    x = O.normal_f64(O.stream_seed(61, 0), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(62, 0), d * (n + z), 1.0 / d).astype(np.float64).reshape(d, n + z)
    st = P.RouterState(w, n, z, k, ke, 0.0, 1.0)
    dg = P.route_topk(x, st)
    w_in = [O.normal_f64(O.stream_seed(63, 2 * e), d * I).reshape(d, I) / np.sqrt(d)
            for e in range(n)]
    w_out = [O.normal_f64(O.stream_seed(63, 2 * e + 1), I * d).reshape(I, d) / np.sqrt(d)
             for e in range(n)]
    bank = P.ExpertBank(w_in, w_out, m=m, gamma_mode=gamma_mode, precision=P.PREC_F64_EXACT)
    out = P.moe_forward(x, dg, bank, z, renormalize=renorm)
    want = np.empty((T, d))
    rc = O.orc().orc_moe_forward_f64(ptr(x), T, d, ptr(np.ascontiguousarray(dg.indices, np.uint32)),
                                     ptr(np.ascontiguousarray(dg.gates)), k, n, z,
                                     O.ptr_array(w_in), O.ptr_array(w_out), I, bank.gamma_ffn(),
                                     bank.gamma_zero(), int(renorm), ptr(want))
    assert rc == 0
    assert (out.view(np.uint64) == want.view(np.uint64)).all(), \
        int((out.view(np.uint64) != want.view(np.uint64)).sum())
