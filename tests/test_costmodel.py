"""the TPOT calculator restated from analytics.hpp:211-253,
pinned on the reference's own cost-model tests (tests/test_analytics.cpp:189-240,
tests/acceptance_main.cpp:160-176) and its three data rows."""
import json

import pytest

import paper_2509_01322_b200 as P
from paper_2509_01322_b200.costmodel import CostModel, load, tpot_theoretical, with_measured

# the three rows of the reference's data/costmodels/*.json (values restated)
ROWS = {
    "sbo_28l": dict(attention_us=264, dispatch_us=236, moe_us=60, combine_us=472, n_layer=28,
                    accept_factor=1.8, strategy="sbo", batch_per_device=96,
                    price_per_device_hour=2.0),
    "tbo_61l": dict(attention_us=471, dispatch_us=275, moe_us=77, combine_us=551, n_layer=61,
                    accept_factor=1.8, strategy="tbo", batch_per_device=96,
                    price_per_device_hour=2.0),
    "tbo_94l": dict(attention_us=314, dispatch_us=157, moe_us=29, combine_us=315, n_layer=94,
                    accept_factor=1.8, strategy="tbo", batch_per_device=96,
                    price_per_device_hour=2.0),
}


def test_sbo_row_reproduces_16ms_and_price():
    # tests/test_analytics.cpp:205-211
    r = tpot_theoretical(CostModel(264, 236, 60, 472, 28, 1.8, "sbo"))
    assert abs(r.tpl_us - 1032.0) <= 1e-9
    assert abs(r.tpot_ms - 16.0) <= 0.5
    assert abs(r.price_per_mtok - 0.09) <= 0.01
    assert not r.tbo_model_approximate


def test_tbo_rows_within_15_percent():
    # tests/test_analytics.cpp:213-240
    ra = tpot_theoretical(CostModel(471, 275, 77, 551, 61, 1.8, "tbo"))
    assert ra.tbo_model_approximate
    assert abs(ra.tpot_ms - 30.0) / 30.0 < 0.15 and abs(ra.price_per_mtok - 0.17) <= 0.03
    rq = tpot_theoretical(CostModel(314, 157, 29, 315, 94, 1.8, "tbo"))
    assert abs(rq.tpot_ms - 26.2) / 26.2 < 0.15 and abs(rq.price_per_mtok - 0.15) <= 0.03


def test_data_rows_load_and_match_acceptance(tmp_path):
    # tests/acceptance_main.cpp:160-176 on the data/costmodels/*.json rows, read
    # back through the JSON loader
    t = {}
    for name, row in ROWS.items():
        f = tmp_path / f"{name}.json"
        f.write_text(json.dumps(row))
        t[name] = tpot_theoretical(load(str(f))).tpot_ms
    assert abs(t["sbo_28l"] - 16.0) <= 0.5
    assert abs(t["tbo_61l"] - 30.0) / 30.0 < 0.15
    assert abs(t["tbo_94l"] - 26.2) / 26.2 < 0.15


def test_errors_and_measured_substitution():
    with pytest.raises(P.ConfigError):
        tpot_theoretical(CostModel(-1, 0, 0, 0, 1))
    with pytest.raises(P.ConfigError):
        tpot_theoretical(CostModel(1, 1, 1, 1, 0))
    with pytest.raises(P.ConfigError):
        tpot_theoretical(CostModel(1, 1, 1, 1, 1, 0.5))
    with pytest.raises(P.ConfigError):
        tpot_theoretical(CostModel(1, 1, 1, 1, 1, 1.0, "xbo"))
    with pytest.raises(P.ConfigError):
        tpot_theoretical(CostModel(1, 1, 1, 1, 1, 1.0, "sbo", 0.0))
    base = CostModel(264, 236, 60, 472, 28, 1.8, "sbo")
    faster = with_measured(base, moe_us=30.0, dispatch_us=100.0)
    assert tpot_theoretical(faster).tpl_us == 264 + 100 + 30 + 472
    with pytest.raises(P.ConfigError):
        with_measured(base, n_layer=3)


def test_zero_latencies_give_zero_price_like_the_reference():
    # analytics.hpp:250-252 in IEEE double: tpot 0 -> tokens/s inf -> price 0
    r = tpot_theoretical(CostModel(0, 0, 0, 0, 28, 1.8, "sbo"))
    assert r.tpot_ms == 0.0 and r.price_per_mtok == 0.0
