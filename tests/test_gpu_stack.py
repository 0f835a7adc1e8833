"""BASELINE config 5: a 4-layer ScMoE stack with PID-controlled expert bias.

Teacher-forced check against the oracle at every step and layer: the oracle
routes the GPU's actual layer input (rmsnorm -> exact router) with its own
controller state, accumulates and ticks the controller; indices, counters and
bias vectors must match bit for bit, and the activated-FFN mean must move to
K_e (zero-expert fraction -> 1 - K_e/K)."""
import os

import numpy as np
import pytest

import _oracle as O
from _oracle import ptr

pytestmark = pytest.mark.gpu


def _route_ref(x, w, n, z, k, ke, mu, b):
    T, d = x.shape
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    if O.ref_available():  # the reference itself, token-sharded over the host cores
        rc = O.ref().ref_route_topk_f32(ptr(x), T, d, ptr(w), n, z, k, ke, mu, ptr(b), ptr(idx),
                                        ptr(g), ptr(c), None, os.cpu_count() or 4)
    else:
        rc = O.orc().orc_route_topk_f32(ptr(x), T, d, ptr(w), n, z, k, ke, mu, ptr(b), ptr(idx),
                                        ptr(g), ptr(c), None)
    assert rc == 0
    return idx, c


def test_pid_stack_teacher_forced_bitwise(scmoe):
    import torch
    from paper_2509_01322_b200.layer import LayerShape
    from paper_2509_01322_b200.stack import ScMoEStack
    P = scmoe
    shape = LayerShape(d=6144, n_ffn=512, n_zero=256, top_k=12, k_expected=6, inter=256,
                       precision=P.PREC_BF16)
    n_layers, T, steps, mu0, decay = 4, 512, 12, 0.2, 0.999
    stream = torch.cuda.Stream()
    ctx = P.Context(0)
    ctx.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        stack = ScMoEStack(ctx, shape, n_layers, seed=11, mu=mu0, mu_decay=decay)
        E = shape.E
        W = [l.router_weights() for l in stack.layers]
        ob = [np.zeros(E) for _ in range(n_layers)]
        omu = [np.array([mu0]) for _ in range(n_layers)]
        ones = np.ones(shape.d, np.float32)
        for step in range(steps):
            x = torch.from_numpy(P.fill_normal(P.stream_seed(99, step), T * shape.d)).cuda()
            idxs, inputs, _ = stack.step(x.view(T, shape.d), T, keep_inputs=True)
            routed = [np.zeros(E, np.uint64) for _ in range(n_layers)]
            seen = [np.zeros(1, np.uint64) for _ in range(n_layers)]
            for l in range(n_layers):
                a1 = inputs[l].cpu().numpy().reshape(T, shape.d)
                h = np.empty_like(a1)
                O.orc().orc_rmsnorm_f32(ptr(a1), ptr(ones), T, shape.d, np.float32(1e-6), ptr(h))
                want_idx, _ = _route_ref(h, W[l], shape.n_ffn, shape.n_zero, shape.top_k,
                                         shape.k_expected, float(omu[l][0]), ob[l])
                got_idx = idxs[l].cpu().numpy().view(np.uint32)
                assert (got_idx == want_idx).all(), f"step {step} layer {l}: routing differs"
                O.orc().orc_accumulate_counters(ptr(want_idx), T, shape.top_k, ptr(routed[l]),
                                                ptr(seen[l]))
            for l in range(n_layers):
                delta = np.zeros(E)
                assert O.orc().orc_bias_update(shape.n_ffn, shape.n_zero, shape.top_k,
                                               shape.k_expected, ptr(omu[l]), decay, ptr(ob[l]),
                                               ptr(routed[l]), ptr(seen[l]), ptr(delta)) == 0
                got_b = stack.layers[l].bias()
                assert (got_b.view(np.uint64) == ob[l].view(np.uint64)).all(), \
                    f"step {step} layer {l}: bias differs"
                assert (got_b[shape.n_ffn:] == 0).all()
    means = np.array(stack.trace.mean_ffn)  # [step, layer]
    # the controller pulls activated FFN experts from ~8 (= K N / E) towards K_e = 6
    assert (means[-1] < means[0] - 0.5).all(), means
