"""GPU parity: MLA forward value and cached decode (csrc/mla.cu) against the
oracle restatement (oracle/scmoe_oracle.c orc_mla_*, pinned bitwise on the
reference in tests/test_oracle_mla.py).  Bar: bit-exact (fp32, same order)."""
import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [
    # (d, dq, dkv, H, dhc, dhr, seq_len, n_seq)
    (32, 8, 4, 4, 8, 4, 4, 1),       # test_blocks.cpp:158-169
    (16, 8, 4, 1, 8, 4, 6, 2),       # test_blocks.cpp:171-185
    (16, 8, 4, 2, 6, 4, 5, 3),       # test_blocks.cpp:187-200
    (48, 24, 16, 3, 10, 6, 7, 2),    # ragged widths
    (256, 64, 32, 4, 32, 16, 96, 3),   # 64-query tiles, diagonal chunks
    (128, 64, 32, 2, 72, 40, 200, 1),  # 128-tile kernels, partial column / k chunks
    (192, 64, 32, 3, 128, 64, 260, 2),  # 128-tile kernels, LongCat head widths, 3 query tiles
]


def _params(P, dims, w, va=True, base=1.0e4):
    from paper_2509_01322_b200.mla import MlaParams
    return MlaParams(*dims, weights=w, rope_base=base, variance_alignment=va)


@pytest.mark.parametrize("shape", SHAPES)
def test_mla_forward_bitwise(scmoe, orc, shape):
    from paper_2509_01322_b200.mla import mla_block
    *dims, seq, nseq = shape
    dims = tuple(dims)
    w = O.mla_weights(*dims, seed=11)
    rows = seq * nseq
    h = O.normal_f32(O.stream_seed(5, 1), rows * dims[0]).reshape(rows, dims[0])
    rc, want = O.mla_forward(orc, dims, w, h, seq)
    assert rc == 0
    got = mla_block(h, _params(scmoe, dims, w), seq)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("va", [True, False])
def test_mla_decode_bitwise(scmoe, orc, va):
    from paper_2509_01322_b200.mla import MlaCache, mla_block, mla_infer_step
    dims = (64, 32, 16, 4, 16, 8)
    T = 40
    w = O.mla_weights(*dims, seed=7)
    h = O.normal_f32(O.stream_seed(2, 0), T * 64).reshape(T, 64)
    rc, want, ckv, kr = O.mla_infer(orc, dims, w, h, va=int(va))
    assert rc == 0
    p = _params(scmoe, dims, w, va=va)
    cache = MlaCache(p, capacity_hint=4)  # grows 4 -> 64 on the way
    got = np.concatenate([mla_infer_step(p, cache, h[t:t + 1], t) for t in range(T)])
    assert got.tobytes() == want.tobytes()
    assert cache.length() == T
    c2, k2 = cache.read()
    assert c2.tobytes() == ckv.tobytes() and k2.tobytes() == kr.tobytes()
    # decode == prefill rows (one sequence of T)
    assert mla_block(h, p, T).tobytes() == want.tobytes()


def test_mla_errors(scmoe):
    from paper_2509_01322_b200.mla import MlaCache, MlaParams, mla_block, mla_infer_step
    dims = (32, 8, 4, 4, 8, 4)
    w = O.mla_weights(*dims)
    p = _params(scmoe, dims, w)
    h = O.normal_f32(9, 4 * 32).reshape(4, 32)
    with pytest.raises(scmoe.DimensionError):
        mla_block(h, p, 3)  # rows must pack whole sequences (graph.hpp:404)
    odd = (32, 8, 4, 4, 8, 3)
    with pytest.raises(scmoe.DimensionError):
        mla_block(h, MlaParams(*odd, weights=O.mla_weights(*odd)), 4)
    with pytest.raises(scmoe.ParameterError):
        MlaParams(32, 0, 4, 4, 8, 4, weights=[np.zeros((1, 1))] * 8).device(
            scmoe.default_context())
    cache = MlaCache(p)
    mla_infer_step(p, cache, h[:1], 0)
    with pytest.raises(scmoe.StateError):
        mla_infer_step(p, cache, h[:1], 0)  # test_blocks.cpp:202-209
    with pytest.raises(scmoe.StateError):
        mla_infer_step(p, cache, h[:1], 5)
    # zero weights -> zero output (test_blocks.cpp:158-169)
    z = [np.zeros(s, np.float32) for s in O.mla_shapes(*dims)]
    assert not mla_block(h, _params(scmoe, dims, z), 4).any()


def test_mla_device_api_and_longcat_widths(scmoe, orc):
    """LongCat MLA widths (d 6144, d_q 1536, d_kv 512, 64 heads x (128 + 64),
    PAPER.md / model.hpp config) on one 48-token sequence, through the
    device-pointer API with torch CUDA tensors: bitwise equal to the oracle."""
    import torch
    from paper_2509_01322_b200.mla import mla_block
    dims = (6144, 1536, 512, 64, 128, 64)
    seq = 48
    w = O.mla_weights(*dims, seed=2)
    h = O.normal_f32(O.stream_seed(8, 0), seq * dims[0]).reshape(seq, dims[0])
    rc, want = O.mla_forward(orc, dims, w, h, seq, base=1.0e6)
    assert rc == 0
    p = _params(scmoe, dims, [torch.from_numpy(x).cuda() for x in w], base=1.0e6)
    got = mla_block(torch.from_numpy(h).cuda(), p, seq)
    scmoe.default_context().synchronize()
    assert got.cpu().numpy().tobytes() == want.tobytes()
