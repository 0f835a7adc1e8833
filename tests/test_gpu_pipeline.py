"""GPU tests of the device tier: the pipelined multi-batch schedule
(scmoe_layer_forward_batches) gives bit-identical routing and outputs to
serial scmoe_layer_forward calls, and every router kernel variant (slab,
lean, tiled) is bit-exact against the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_pipelined_batches_equal_serial(scmoe):
    import torch
    from paper_2509_01322_b200.layer import DeviceLayer, LayerShape
    P = scmoe
    ctx = P.Context(0)
    shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=4, inter=512,
                       precision=P.PREC_BF16)
    layer = DeviceLayer(ctx, shape, seed=3)
    T, nb = 700, 5
    a1 = [torch.from_numpy(P.fill_normal(P.stream_seed(9, i), T * shape.d)).cuda() for i in range(nb)]
    a3 = [torch.from_numpy(P.fill_normal(P.stream_seed(10, i), T * shape.d)).cuda() for i in range(nb)]

    def bufs():
        return dict(idx=torch.empty(T * shape.top_k, dtype=torch.int32, device="cuda"),
                    gates=torch.empty(T * shape.top_k, dtype=torch.float64, device="cuda"),
                    cnt=torch.empty(T, dtype=torch.int32, device="cuda"),
                    out=torch.empty(T, shape.d, dtype=torch.float32, device="cuda"))

    ser = [bufs() for _ in range(nb)]
    for i in range(nb):
        layer.forward(a1[i].data_ptr(), a3[i].data_ptr(), None, T, ser[i]["idx"].data_ptr(),
                      ser[i]["gates"].data_ptr(), ser[i]["cnt"].data_ptr(), ser[i]["out"].data_ptr())
    ctx.synchronize()
    pip = [bufs() for _ in range(nb)]
    layer.forward_batches([a.data_ptr() for a in a1], [a.data_ptr() for a in a3], None, T,
                          [b["idx"].data_ptr() for b in pip], [b["gates"].data_ptr() for b in pip],
                          [b["cnt"].data_ptr() for b in pip], [b["out"].data_ptr() for b in pip])
    ctx.synchronize()
    for s, p in zip(ser, pip):
        for k in ("idx", "gates", "cnt", "out"):
            assert torch.equal(s[k], p[k]), k


@pytest.mark.parametrize("variant", ["tma", "corun", "slab", "lean", "tiled"])
def test_router_kernel_variants_bitwise(variant):
    """Each router projection kernel, selected with SCMOE_ROUTER, reproduces
    the reference's logits (via route_topk probabilities) bit for bit."""
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
import _oracle as O, paper_2509_01322_b200 as P
T, d, n, z, k, ke = 4200, 6144, 512, 256, 12, 8
x = O.normal_f32(O.stream_seed(77, 0), T * d).reshape(T, d)
w = O.uniform_f32(O.stream_seed(5, 0), d * (n + z), 1.0 / d).reshape(d, n + z)
st = P.RouterState(w, n, z, k, ke, 0.0, 1.0)
pl = []
dg = P.route_topk(x, st, pl)
sub = np.r_[0:300, 4000:4200]
rc, idx, g, c, probs = O.orc_route_topk(x[sub], w, n, z, k, ke, want_probs=True)
assert rc == 0
assert (pl[0][sub].view(np.uint32) == probs.view(np.uint32)).all()
assert (dg.indices.reshape(T, k)[sub].ravel() == idx).all()
print("ok")
"""
    env = dict(os.environ, SCMOE_ROUTER=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("variant", ["tma", "corun", "slab", "lean", "tiled", "small"])
def test_router_kernel_variants_edge_values(variant):
    """Subnormal products and sums, exact zeros, signed zeros, a ragged last
    slab and a partial expert width (E = 60 < 768): every router kernel (the
    slab kernel runs packed f32x2 FMUL2/FADD2) still matches the reference's
    sequential fp32 arithmetic bit for bit."""
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
import _oracle as O, paper_2509_01322_b200 as P
T, d, n, z, k, ke = 131, 256, 40, 20, 6, 4
x = O.normal_f32(O.stream_seed(3, 0), T * d).reshape(T, d)
w = O.uniform_f32(O.stream_seed(4, 0), d * (n + z), 1.0 / d).reshape(d, n + z)
x[::3] *= np.float32(2.0 ** -66)      # x*w products below 2^-126: subnormal
w[:, ::5] *= np.float32(2.0 ** -60)
x[5] = 0.0
x[7, ::2] = -0.0
w[:, 3] = 0.0
x[9] *= np.float32(2.0 ** 60)          # large products next to tiny ones
st = P.RouterState(w, n, z, k, ke, 0.0, 1.0)
pl = []
dg = P.route_topk(x, st, pl)
rc, idx, g, c, probs = O.orc_route_topk(x, w, n, z, k, ke, want_probs=True)
assert rc == 0
assert (pl[0].view(np.uint32) == probs.view(np.uint32)).all()
assert (dg.indices == idx).all() and (dg.gates.view(np.uint64) == g.view(np.uint64)).all()
print("ok")
"""
    env = dict(os.environ, SCMOE_ROUTER=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_host_batches_equal_serial_host_calls(scmoe):
    """scmoe_layer_forward_host_batches (copy-in / compute / copy-out of
    neighbouring batches overlapped) returns exactly what n serial
    scmoe_layer_forward_host calls return, including the routing outputs."""
    import torch
    from paper_2509_01322_b200.layer import DeviceLayer, LayerShape
    P = scmoe
    ctx = P.Context(0)
    shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=4, inter=512,
                       precision=P.PREC_BF16)
    layer = DeviceLayer(ctx, shape, seed=5)
    T, nb, d, K = 333, 5, shape.d, shape.top_k
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    a1 = [pin(P.fill_normal(P.stream_seed(21, i), T * d).reshape(T, d)) for i in range(nb)]
    a3 = [pin(P.fill_normal(P.stream_seed(22, i), T * d).reshape(T, d)) for i in range(nb)]

    def outs():
        return (np.zeros((T, d), np.float32), np.zeros(T * K, np.uint32), np.zeros(T * K),
                np.zeros(T, np.uint32))

    ser = [outs() for _ in range(nb)]
    for i in range(nb):
        o, ix, g, c = ser[i]
        layer.forward_host(a1[i], a3[i], None, T, ix, g, c, o)
    bat = [outs() for _ in range(nb)]
    layer.forward_host_batches(a1, a3, None, T, [b[1] for b in bat], [b[2] for b in bat],
                               [b[3] for b in bat], [b[0] for b in bat])
    for s, b in zip(ser, bat):
        for u, v in zip(s, b):
            assert u.tobytes() == v.tobytes()
    # routing outputs optional, a3 optional
    only = [np.zeros((T, d), np.float32) for _ in range(2)]
    layer.forward_host_batches(a1[:2], None, None, T, None, None, None, only)
    for i in range(2):
        o = np.zeros((T, d), np.float32)
        layer.forward_host(a1[i], None, None, T, None, None, None, o)
        assert o.tobytes() == only[i].tobytes()


def test_pipelined_batches_with_gain_and_renormalisation(scmoe):
    """The pipelined schedule with a norm gain vector and gate renormalisation
    (blocks.hpp:240-247) gives the serial results bit for bit."""
    import torch
    from paper_2509_01322_b200.layer import DeviceLayer, LayerShape
    P = scmoe
    ctx = P.Context(0)
    shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=4, inter=512,
                       precision=P.PREC_BF16, m=2, gamma_mode=1)
    layer = DeviceLayer(ctx, shape, seed=4)
    T, nb = 640, 3
    g = torch.from_numpy((1.0 + 0.1 * P.fill_normal(P.stream_seed(3, 9), shape.d)).astype(
        np.float32)).cuda()
    a1 = [torch.from_numpy(P.fill_normal(P.stream_seed(11, i), T * shape.d)).cuda() for i in range(nb)]
    a3 = [torch.from_numpy(P.fill_normal(P.stream_seed(12, i), T * shape.d)).cuda() for i in range(nb)]

    def bufs():
        return dict(idx=torch.empty(T * shape.top_k, dtype=torch.int32, device="cuda"),
                    gates=torch.empty(T * shape.top_k, dtype=torch.float64, device="cuda"),
                    cnt=torch.empty(T, dtype=torch.int32, device="cuda"),
                    out=torch.empty(T, shape.d, dtype=torch.float32, device="cuda"))

    ser = [bufs() for _ in range(nb)]
    for i in range(nb):
        layer.forward(a1[i].data_ptr(), a3[i].data_ptr(), g.data_ptr(), T, ser[i]["idx"].data_ptr(),
                      ser[i]["gates"].data_ptr(), ser[i]["cnt"].data_ptr(), ser[i]["out"].data_ptr(),
                      renormalize=True)
    ctx.synchronize()
    pip = [bufs() for _ in range(nb)]
    layer.forward_batches([a.data_ptr() for a in a1], [a.data_ptr() for a in a3], g.data_ptr(), T,
                          [b["idx"].data_ptr() for b in pip], [b["gates"].data_ptr() for b in pip],
                          [b["cnt"].data_ptr() for b in pip], [b["out"].data_ptr() for b in pip],
                          renormalize=True)
    ctx.synchronize()
    for s, p in zip(ser, pip):
        for k in ("idx", "gates", "cnt", "out"):
            assert torch.equal(s[k], p[k]), k
