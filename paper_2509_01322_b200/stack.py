"""A stack of ScMoE MoE branches with PID-controlled expert bias
(BASELINE config 5).

Each step feeds x through L layers -- layer l computes
out = x + moe(rmsnorm(x)) with its own router, controller state and expert
bank (model.hpp:394-400 with the dense branch the identity) -- accumulates
every layer's slot counters (Model::accumulate_routing, model.hpp:235-238)
and ticks every layer's controller (Model::update_biases, model.hpp:241-244:
only layers with tokens_seen > 0).  Everything runs on the device; the host
only sequences calls and records statistics.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import torch

from . import Context
from .layer import DeviceLayer, LayerShape


@dataclass
class StackTrace:
    mean_ffn: List[List[float]] = field(default_factory=list)  # [step][layer]
    std_ffn: List[List[float]] = field(default_factory=list)


class ScMoEStack:
    def __init__(self, ctx: Context, shape: LayerShape, n_layers: int, seed: int, mu: float,
                 mu_decay: float):
        self.ctx, self.shape = ctx, shape
        self.layers = [DeviceLayer(ctx, shape, seed=seed + 1000 * l, mu=mu, mu_decay=mu_decay)
                       for l in range(n_layers)]
        self.trace = StackTrace()

    def step(self, x: torch.Tensor, T: int, keep_inputs: bool = False, record: bool = True):
        """One training-style step: forward through every layer, count, tick.
        Returns the per-layer routing indices (device) and, if requested, the
        per-layer inputs (for teacher-forced checking).  record=True appends
        the per-layer mean/std activated FFN experts to the trace (one host
        read of the ffn counts per step)."""
        s = self.shape
        inputs, idxs, cnts = [], [], []
        for layer in self.layers:
            if keep_inputs:
                inputs.append(x.clone())
            idx = torch.empty(T * s.top_k, dtype=torch.int32, device=x.device)
            gates = torch.empty(T * s.top_k, dtype=torch.float64, device=x.device)
            cnt = torch.empty(T, dtype=torch.int32, device=x.device)
            out = torch.empty_like(x)
            layer.forward(x.data_ptr(), x.data_ptr(), None, T, idx.data_ptr(), gates.data_ptr(),
                          cnt.data_ptr(), out.data_ptr())
            layer.accumulate(idx.data_ptr(), T)  # Model::accumulate_routing
            idxs.append(idx)
            cnts.append(cnt)
            x = out
        # Model::update_biases: only layers that saw tokens (every layer here
        # when T > 0); bias_update synchronises for its StateError check
        for layer in self.layers:
            if T > 0:
                layer.bias_update(want_delta=False)
        if record:
            c = torch.stack(cnts).to(torch.float64).cpu().numpy()  # [layer, T]
            self.trace.mean_ffn.append([float(v) for v in c.mean(1)])
            self.trace.std_ffn.append([float(v) for v in c.std(1)])
        return idxs, inputs, x
