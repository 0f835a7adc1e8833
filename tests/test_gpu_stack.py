"""BASELINE config 5 / SURVEY.md 8(d) E5 at its configured parameters: a
4-layer ScMoE stack (LongCat layer shape: d = 6144, 512 FFN experts of inter
2048 + 256 zero experts, top-12) over 100 router steps of 1024 tokens, PID
bias control with K_e = 6, mu = 0.2, mu_decay = 0.999, bias_update every step.

Teacher-forced against the reference at every step and layer: the reference
(oracle/_ref, or the C restatement) takes the GPU's actual fp32 layer input,
applies rmsnorm (graph.hpp:322-335) and routes it with ITS OWN controller
state (router.hpp:133-141), accumulates (router.hpp:144-150) and ticks
(router.hpp:155-176; Model::accumulate_routing / update_biases,
model.hpp:235-244).  Indices, ffn counts, the per-expert counters and the bias
vectors must match bit for bit at every step and layer, and the activated-FFN
mean must track K_e: tail-20 mean within 2 % of 6 on every layer, i.e. the
zero-expert fraction 1 - mean/K within 0.01 of 1 - K_e/K = 0.5
(simulate_bias_control, router.hpp:349-369; tests/acceptance_main.cpp:103-134
checks the same tracking at 1 %).
"""
import os
import time

import numpy as np
import pytest

import _oracle as O
from _oracle import ptr

pytestmark = pytest.mark.gpu

N_LAYERS, T, STEPS, KE, MU0, DECAY = 4, 1024, 100, 6, 0.2, 0.999


class _RefController:
    """One layer's router + controller on the host (the reference itself
    where _ref is built)."""

    def __init__(self, w, s):
        self.w, self.s = w, s
        self.b = np.zeros(s.E)
        self.mu = np.array([MU0])
        self.routed = np.zeros(s.E, np.uint64)
        self.seen = np.zeros(1, np.uint64)
        self.ref = O.ref() if O.ref_available() else None

    def route(self, a1):
        s, (Tn, d) = self.s, a1.shape
        h = np.empty_like(a1)
        idx = np.empty(Tn * s.top_k, np.uint32)
        g = np.empty(Tn * s.top_k)
        c = np.empty(Tn, np.uint32)
        ones = np.ones(d, np.float32)
        if self.ref is not None:
            assert self.ref.ref_rmsnorm_f32(ptr(a1), ptr(ones), Tn, d, ptr(h)) == 0
            rc = self.ref.ref_route_topk_f32(ptr(h), Tn, d, ptr(self.w), s.n_ffn, s.n_zero,
                                             s.top_k, s.k_expected, float(self.mu[0]),
                                             ptr(self.b), ptr(idx), ptr(g), ptr(c), None,
                                             os.cpu_count() or 4)
        else:
            O.orc().orc_rmsnorm_f32(ptr(a1), ptr(ones), Tn, d, np.float32(1e-6), ptr(h))
            rc = O.orc().orc_route_topk_f32(ptr(h), Tn, d, ptr(self.w), s.n_ffn, s.n_zero,
                                            s.top_k, s.k_expected, float(self.mu[0]),
                                            ptr(self.b), ptr(idx), ptr(g), ptr(c), None)
        assert rc == 0
        return idx, c

    def accumulate(self, idx, Tn):
        s = self.s
        if self.ref is not None:
            assert self.ref.ref_accumulate_counters(ptr(idx), Tn, s.n_ffn, s.n_zero, s.top_k,
                                                    ptr(self.routed), ptr(self.seen)) == 0
        else:
            O.orc().orc_accumulate_counters(ptr(idx), Tn, s.top_k, ptr(self.routed),
                                            ptr(self.seen))

    def bias_update(self):
        s = self.s
        delta = np.zeros(s.E)
        fn = self.ref.ref_bias_update if self.ref is not None else O.orc().orc_bias_update
        assert fn(s.n_ffn, s.n_zero, s.top_k, s.k_expected, ptr(self.mu), DECAY, ptr(self.b),
                  ptr(self.routed), ptr(self.seen), ptr(delta)) == 0


def test_pid_stack_e5_teacher_forced_bitwise(scmoe):
    import torch
    from paper_2509_01322_b200.layer import LayerShape
    from paper_2509_01322_b200.stack import ScMoEStack
    P = scmoe
    shape = LayerShape(d=6144, n_ffn=512, n_zero=256, top_k=12, k_expected=KE, inter=2048,
                       precision=P.PREC_BF16)
    t0 = time.time()
    stream = torch.cuda.Stream()
    ctx = P.Context(0)
    ctx.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        stack = ScMoEStack(ctx, shape, N_LAYERS, seed=11, mu=MU0, mu_decay=DECAY)
        refs = [_RefController(l.router_weights(), shape) for l in stack.layers]
        for step in range(STEPS):
            x = torch.from_numpy(P.fill_normal(P.stream_seed(99, step), T * shape.d,
                                               threads=os.cpu_count() or 8)).cuda()
            idxs, inputs, _ = stack.step(x.view(T, shape.d), T, keep_inputs=True)
            for l in range(N_LAYERS):
                want_idx, want_c = refs[l].route(inputs[l].cpu().numpy().reshape(T, shape.d))
                got_idx = idxs[l].cpu().numpy().view(np.uint32)
                assert (got_idx == want_idx).all(), f"step {step} layer {l}: routing differs"
                assert stack.trace.mean_ffn[-1][l] == float(want_c.mean())
                refs[l].accumulate(want_idx, T)
            for l in range(N_LAYERS):
                refs[l].bias_update()
                got_b = stack.layers[l].bias()
                assert (got_b.view(np.uint64) == refs[l].b.view(np.uint64)).all(), \
                    f"step {step} layer {l}: bias differs"
                assert (got_b[shape.n_ffn:] == 0).all()  # zero experts never biased
                routed, seen = stack.layers[l].counters()
                assert seen == 0 and (routed == 0).all() and (refs[l].routed == 0).all()
    means = np.array(stack.trace.mean_ffn)  # [step, layer]
    tail = means[-20:].mean(0)
    zero_frac = 1.0 - tail / shape.top_k
    print(f"E5: {STEPS} steps x {N_LAYERS} layers in {time.time() - t0:.1f}s; first-step mean "
          f"{means[0].round(3)}, tail-20 mean {tail.round(4)}, zero-expert fraction "
          f"{zero_frac.round(4)}")
    assert (means[0] > KE + 1.0).all(), means[0]  # starts near K N / E = 8
    assert (np.abs(tail - KE) <= 0.02 * KE).all(), tail
    assert (np.abs(zero_frac - (1 - KE / shape.top_k)) <= 0.01).all(), zero_frac
