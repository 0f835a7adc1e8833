"""Theoretical time-per-output-token from per-module latencies.

Restates the reference's calculator, analytics.hpp:211-253 (`CostModel`,
`TpotResult`, `tpot_theoretical`), so measured B200 module latencies (the
expert GEMMs of `scmoe_moe_rows`, the EP dispatch / return all-to-alls) can
be fed into the same SBO / TBO formulas as the reference's cost-model rows
(`data/costmodels/*.json`; its three rows are restated in
tests/test_costmodel.py, pinned on the reference's analytics tests).  bench.py
emits a ``tpot`` block that feeds this calculator with B200-measured expert
GEMM, dispatch and return latencies.

    SBO: per-layer time = attention + dispatch + moe + combine (every module
         exposed serially -- the reference's single-batch overlap row);
    TBO: per-layer time = max(attention + moe, dispatch + combine).
    tpot_ms = n_layer * tpl_us / (1000 * accept_factor)
    price   = device-hours per 1M tokens * price_per_device_hour.
"""
from __future__ import annotations

import json
from dataclasses import asdict, dataclass, replace

from . import ConfigError


@dataclass
class CostModel:
    """analytics.hpp:213-223"""
    attention_us: float = 0.0
    dispatch_us: float = 0.0
    moe_us: float = 0.0
    combine_us: float = 0.0
    n_layer: int = 0
    accept_factor: float = 1.0   # tokens emitted per decode step
    strategy: str = "sbo"
    batch_per_device: float = 96.0
    price_per_device_hour: float = 2.0


@dataclass
class TpotResult:
    """analytics.hpp:225-230"""
    tpl_us: float = 0.0
    tpot_ms: float = 0.0
    price_per_mtok: float = 0.0
    tbo_model_approximate: bool = False


def tpot_theoretical(cm: CostModel) -> TpotResult:
    """analytics.hpp:234-253, same checks (ConfigError) in the same order."""
    if cm.attention_us < 0 or cm.dispatch_us < 0 or cm.moe_us < 0 or cm.combine_us < 0:
        raise ConfigError("tpot: latencies must be >= 0")
    if cm.n_layer == 0:
        raise ConfigError("tpot: n_layer must be >= 1")
    if cm.accept_factor < 1.0:
        raise ConfigError("tpot: accept factor must be >= 1")
    if cm.batch_per_device <= 0.0 or cm.price_per_device_hour < 0.0:
        raise ConfigError("tpot: bad device assumptions")
    r = TpotResult()
    if cm.strategy == "sbo":
        r.tpl_us = cm.attention_us + cm.dispatch_us + cm.moe_us + cm.combine_us
    elif cm.strategy == "tbo":
        r.tpl_us = max(cm.attention_us + cm.moe_us, cm.dispatch_us + cm.combine_us)
        r.tbo_model_approximate = True
    else:
        raise ConfigError("tpot: unknown overlap strategy " + cm.strategy)
    r.tpot_ms = float(cm.n_layer) * r.tpl_us / (1000.0 * cm.accept_factor)
    # IEEE like the reference's C++: all latencies 0 -> inf tokens/s -> price 0
    tokens_per_device_second = (cm.batch_per_device * 1000.0 / r.tpot_ms if r.tpot_ms != 0.0
                                else float("inf"))
    device_hours_per_mtok = 1.0e6 / (tokens_per_device_second * 3600.0)
    r.price_per_mtok = device_hours_per_mtok * cm.price_per_device_hour
    return r


def load(path: str) -> CostModel:
    """A cost-model row in the reference's JSON format (data/costmodels/*.json)."""
    with open(path) as f:
        d = json.load(f)
    known = set(asdict(CostModel()))
    extra = set(d) - known
    if extra:
        raise ConfigError(f"cost model: unknown keys {sorted(extra)}")
    return CostModel(**d)


def with_measured(cm: CostModel, **measured_us) -> CostModel:
    """The row with some module latencies replaced by measured ones (e.g. the
    B200 expert-GEMM time of a decode batch as moe_us, the NVLink all-to-all
    times as dispatch_us / combine_us)."""
    bad = set(measured_us) - {"attention_us", "dispatch_us", "moe_us", "combine_us"}
    if bad:
        raise ConfigError(f"cost model: not a module latency: {sorted(bad)}")
    return replace(cm, **measured_us)
