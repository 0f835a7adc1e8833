"""CPU tests: pin the MLA restatement (oracle/scmoe_oracle.c, orc_mla_*) to
the reference's mla_block / mla_infer_step (blocks.hpp:73-181) compiled from
its headers (oracle/_ref), bitwise, plus the reference's own MLA test cases
(tests/test_blocks.cpp:139-209, tests/test_core.cpp:102-124)."""
import numpy as np
import pytest

import _oracle as O

SHAPES = [
    (32, 8, 4, 4, 8, 4, 4),     # test_blocks.cpp:158-169 (seq 4)
    (16, 8, 4, 1, 8, 4, 6),     # test_blocks.cpp:171-185 (seq 6)
    (16, 8, 4, 2, 6, 4, 5),     # test_blocks.cpp:187-200
    (64, 32, 16, 4, 16, 8, 16),
    (48, 24, 16, 3, 10, 6, 7),  # ragged widths
]


@pytest.mark.parametrize("shape", SHAPES)
def test_mla_forward_oracle_equals_reference(orc, ref, shape):
    *dims, seq = shape
    w = O.mla_weights(*dims, seed=11)
    h = O.normal_f32(O.stream_seed(5, 1), 3 * seq * dims[0]).reshape(3 * seq, dims[0])
    rc_o, out_o = O.mla_forward(orc, dims, w, h, seq)
    rc_r, out_r = O.mla_forward(ref, dims, w, h, seq)
    assert rc_o == rc_r == 0
    assert out_o.tobytes() == out_r.tobytes()
    assert np.abs(out_o).max() > 0


@pytest.mark.parametrize("va", [1, 0])
def test_mla_infer_oracle_equals_reference(orc, ref, va):
    dims = (16, 8, 4, 2, 6, 4)
    w = O.mla_weights(*dims, seed=3)
    h = O.normal_f32(O.stream_seed(1, 0), 5 * 16).reshape(5, 16)
    rc_o, out_o, ckv_o, kr_o = O.mla_infer(orc, dims, w, h, va=va)
    rc_r, out_r, ckv_r, kr_r = O.mla_infer(ref, dims, w, h, va=va)
    assert rc_o == rc_r == 0
    assert out_o.tobytes() == out_r.tobytes()
    assert ckv_o.tobytes() == ckv_r.tobytes() and kr_o.tobytes() == kr_r.tobytes()


def test_mla_decode_equals_prefill_rows(orc):
    # cached incremental decode == the packed forward, row by row
    # (tests/test_blocks.cpp:187-200 checks both against a straight-line
    # reference; in fp32 the two paths share every operation order)
    dims = (64, 32, 16, 4, 16, 8)
    w = O.mla_weights(*dims, seed=7)
    h = O.normal_f32(O.stream_seed(2, 0), 12 * 64).reshape(12, 64)
    _, pre = O.mla_forward(orc, dims, w, h, 12)
    _, dec, _, _ = O.mla_infer(orc, dims, w, h)
    assert pre.tobytes() == dec.tobytes()


def test_mla_zero_weights_and_errors(orc, ref):
    # test_blocks.cpp:158-169: zero weights -> zero output, shape preserved
    dims = (32, 8, 4, 4, 8, 4)
    w = [np.zeros(s, np.float32) for s in O.mla_shapes(*dims)]
    h = O.normal_f32(9, 4 * 32).reshape(4, 32)
    rc, out = O.mla_forward(orc, dims, w, h, 4)
    assert rc == 0 and not out.any()
    # rows must pack whole sequences (graph.hpp:404) -> DimensionError
    w = O.mla_weights(*dims)
    assert O.mla_forward(orc, dims, w, h, 3)[0] == 2 == O.mla_forward(ref, dims, w, h, 3)[0]
    # odd rotary width (tensor.hpp:204) -> DimensionError
    odd = (32, 8, 4, 4, 8, 3)
    w = O.mla_weights(*odd)
    assert O.mla_forward(orc, odd, w, h, 4)[0] == 2 == O.mla_forward(ref, odd, w, h, 4)[0]
    # cache/position mismatch (test_blocks.cpp:202-209) -> StateError
    assert ref.ref_mla_infer_position_check(1, 0) == 3
    assert ref.ref_mla_infer_position_check(1, 5) == 3
    assert ref.ref_mla_infer_position_check(1, 1) == 0
