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


@pytest.mark.parametrize("renorm", [False, True])
def test_full_scmoe_layer(scmoe, orc, renorm):
    """The whole ScMoE layer of Model::build_layer (model.hpp:355-409):
    a1 = x + MLA1(rmsnorm x); dd = a1 + FFN(rmsnorm a1); a3 = dd + MLA2(rmsnorm dd);
    out = a3 + moe(rmsnorm a1).  a1 and the routing are bit-exact (exact MLA,
    rmsnorm, router); a3 / out within the bf16 tolerance of the oracle run on
    the same bf16-rounded dense / expert weights.  The overlapped schedule
    (MoE branch on its own stream) is bitwise the serial one."""
    import torch
    P = scmoe
    from paper_2509_01322_b200.layer import DenseFFN
    from paper_2509_01322_b200.mla import ScMoELayer
    d, dq, dkv, H, dhc, dhr, seq, nseq = 256, 64, 32, 4, 32, 16, 64, 2
    N, Z, K, KE, I, DI = 8, 4, 3, 2, 256, 512
    T = seq * nseq
    dims = (d, dq, dkv, H, dhc, dhr)
    ctx = P.Context(0)
    w1 = O.mla_weights(*dims, seed=21)
    w2 = O.mla_weights(*dims, seed=22)
    dw_in = O.bf16_round(O.uniform_f32(O.stream_seed(23, 0), d * DI, 1.0 / d)).reshape(d, DI)
    dw_out = O.bf16_round(O.uniform_f32(O.stream_seed(23, 1), DI * d, 1.0 / d)).reshape(DI, d)
    wr = O.uniform_f32(O.stream_seed(24, 0), d * (N + Z), 1.0 / d).reshape(d, N + Z)
    ew_in = [O.bf16_round(O.uniform_f32(O.stream_seed(25, 2 * e), d * I, 1.0 / d)).reshape(d, I)
             for e in range(N)]
    ew_out = [O.bf16_round(O.uniform_f32(O.stream_seed(25, 2 * e + 1), I * d, 1.0 / d)).reshape(I, d)
              for e in range(N)]
    norms = [(1.0 + 0.1 * O.normal_f32(26 + i, d)).astype(np.float32) for i in range(4)]
    x = O.normal_f32(O.stream_seed(27, 0), T * d).reshape(T, d)

    from paper_2509_01322_b200.mla import MlaParams
    layer = ScMoELayer(MlaParams(*dims, weights=w1, rope_base=1.0e4),
                       MlaParams(*dims, weights=w2, rope_base=1.0e4),
                       DenseFFN(ctx, d, DI, w_in=dw_in, w_out=dw_out),
                       P.RouterState(wr, N, Z, K, KE, 0.0, 1.0),
                       P.ExpertBank(ew_in, ew_out, precision=P.PREC_BF16), *norms, ctx=ctx)
    out, idx, gates, cnt, a1, a3 = layer.forward(x, seq, renormalize=renorm, overlap=True,
                                                 want_intermediates=True)
    out0, idx0, gates0, cnt0 = layer.forward(x, seq, renormalize=renorm, overlap=False)
    assert out.tobytes() == out0.tobytes() and idx.tobytes() == idx0.tobytes()

    # oracle composition
    def rms(v, g):
        o = np.empty_like(v)
        orc.orc_rmsnorm_f32(O.ptr(v), O.ptr(g), v.shape[0], d, np.float32(1e-6), O.ptr(o))
        return o
    _, m1 = O.mla_forward(orc, dims, w1, rms(x, norms[0]), seq)
    a1_w = x + m1
    assert a1.tobytes() == a1_w.tobytes()
    dd_w = np.empty_like(x)
    assert orc.orc_dense_branch_f32(O.ptr(a1_w), O.ptr(norms[1]), T, d, O.ptr(dw_in),
                                    O.ptr(dw_out), DI, O.ptr(dd_w)) == 0
    _, m2 = O.mla_forward(orc, dims, w2, rms(dd_w, norms[2]), seq)
    a3_w = dd_w + m2
    assert O.rel_l2(a3 - a1_w, a3_w - a1_w) <= 5e-3
    idx_w = np.empty(T * K, np.uint32)
    g_w = np.empty(T * K)
    c_w = np.empty(T, np.uint32)
    out_w = np.empty_like(x)
    assert orc.orc_scmoe_layer_f32(O.ptr(a1_w), O.ptr(a3_w), O.ptr(norms[3]), T, d, O.ptr(wr), N,
                                   Z, K, KE, 0.0, O.ptr(np.zeros(N + Z)), O.ptr_array(ew_in),
                                   O.ptr_array(ew_out), I, 1.0, 1.0, int(renorm), O.ptr(idx_w),
                                   O.ptr(g_w), O.ptr(c_w), O.ptr(out_w)) == 0
    assert idx.tobytes() == idx_w.tobytes() and gates.tobytes() == g_w.tobytes()
    assert cnt.tobytes() == c_w.tobytes()
    assert O.rel_l2(out - a3, out_w - a3_w) <= 5e-3
    assert O.rel_l2(out, out_w) <= 5e-3


def test_full_scmoe_layer_tensor_core_mla(scmoe, orc):
    """The full layer with the tensor-core MLA (fused tcgen05 attention, two
    query tiles per CTA at seq 260): a1 and a3 within the MLA's bf16 tolerance
    of the exact oracle; the MoE branch teacher-forced on the GPU's own a1 /
    a3 is bit-exact in routing and within 5e-3 in output; overlapped ==
    serial bitwise."""
    P = scmoe
    from paper_2509_01322_b200.layer import DenseFFN
    from paper_2509_01322_b200.mla import MlaParams, ScMoELayer
    d, dq, dkv, H, dhc, dhr, seq, nseq = 256, 64, 64, 4, 32, 16, 260, 2
    N, Z, K, KE, I, DI = 8, 4, 3, 2, 256, 512
    T = seq * nseq
    dims = (d, dq, dkv, H, dhc, dhr)
    ctx = P.Context(0)
    w1 = O.mla_weights(*dims, seed=31)
    w2 = O.mla_weights(*dims, seed=32)
    dw_in = O.bf16_round(O.uniform_f32(O.stream_seed(33, 0), d * DI, 1.0 / d)).reshape(d, DI)
    dw_out = O.bf16_round(O.uniform_f32(O.stream_seed(33, 1), DI * d, 1.0 / d)).reshape(DI, d)
    wr = O.uniform_f32(O.stream_seed(34, 0), d * (N + Z), 1.0 / d).reshape(d, N + Z)
    ew_in = [O.bf16_round(O.uniform_f32(O.stream_seed(35, 2 * e), d * I, 1.0 / d)).reshape(d, I)
             for e in range(N)]
    ew_out = [O.bf16_round(O.uniform_f32(O.stream_seed(35, 2 * e + 1), I * d, 1.0 / d)).reshape(I, d)
              for e in range(N)]
    norms = [(1.0 + 0.1 * O.normal_f32(36 + i, d)).astype(np.float32) for i in range(4)]
    x = O.normal_f32(O.stream_seed(37, 0), T * d).reshape(T, d)
    layer = ScMoELayer(MlaParams(*dims, weights=w1, rope_base=1.0e4, precision=P.PREC_BF16),
                       MlaParams(*dims, weights=w2, rope_base=1.0e4, precision=P.PREC_BF16),
                       DenseFFN(ctx, d, DI, w_in=dw_in, w_out=dw_out),
                       P.RouterState(wr, N, Z, K, KE, 0.0, 1.0),
                       P.ExpertBank(ew_in, ew_out, precision=P.PREC_BF16), *norms, ctx=ctx)
    out, idx, gates, cnt, a1, a3 = layer.forward(x, seq, overlap=True, want_intermediates=True)
    out0, idx0, _, _ = layer.forward(x, seq, overlap=False)
    assert out.tobytes() == out0.tobytes() and idx.tobytes() == idx0.tobytes()

    def rms(v, g):
        o = np.empty_like(v)
        orc.orc_rmsnorm_f32(O.ptr(v), O.ptr(g), v.shape[0], d, np.float32(1e-6), O.ptr(o))
        return o
    _, m1 = O.mla_forward(orc, dims, w1, rms(x, norms[0]), seq)
    a1_w = x + m1
    assert O.rel_l2(a1 - x, a1_w - x) <= TC_TOL
    # dense branch + MLA2 on the GPU's own a1 (teacher-forced)
    dd_w = np.empty_like(x)
    assert orc.orc_dense_branch_f32(O.ptr(a1), O.ptr(norms[1]), T, d, O.ptr(dw_in),
                                    O.ptr(dw_out), DI, O.ptr(dd_w)) == 0
    _, m2 = O.mla_forward(orc, dims, w2, rms(dd_w, norms[2]), seq)
    assert O.rel_l2(a3 - a1, dd_w + m2 - a1) <= TC_TOL
    # the MoE branch on the GPU's a1 / a3: routing bit-exact
    idx_w = np.empty(T * K, np.uint32)
    g_w = np.empty(T * K)
    c_w = np.empty(T, np.uint32)
    out_w = np.empty_like(x)
    assert orc.orc_scmoe_layer_f32(O.ptr(a1), O.ptr(a3), O.ptr(norms[3]), T, d, O.ptr(wr), N,
                                   Z, K, KE, 0.0, O.ptr(np.zeros(N + Z)), O.ptr_array(ew_in),
                                   O.ptr_array(ew_out), I, 1.0, 1.0, 0, O.ptr(idx_w),
                                   O.ptr(g_w), O.ptr(c_w), O.ptr(out_w)) == 0
    assert idx.tobytes() == idx_w.tobytes() and gates.tobytes() == g_w.tobytes()
    assert cnt.tobytes() == c_w.tobytes()
    assert O.rel_l2(out - a3, out_w - a3) <= 5e-3


TC_SHAPES = [
    # (d, dq, dkv, H, dhc, dhr, seq_len, n_seq): d, dq, dkv, H*dhc multiples of 64
    (256, 64, 64, 4, 32, 16, 96, 3),      # one 256-key block, partial
    (192, 64, 64, 3, 128, 64, 260, 2),    # LongCat head widths, two key blocks
    (1024, 256, 128, 8, 128, 64, 512, 2),  # wider projections, 2 full key blocks
]
TC_TOL = 2e-2  # bf16 operands, fp32 accumulation (BASELINE north_star bound)


@pytest.mark.parametrize("shape", TC_SHAPES)
def test_mla_forward_tensor_cores(scmoe, orc, shape):
    """The tensor-core MLA (csrc/mla_tc.cu: projections, scores and P.V on the
    tcgen05 grouped GEMM, bf16 operands) within rel-L2 2e-2 of the exact
    oracle (blocks.hpp:73-102)."""
    from paper_2509_01322_b200.mla import MlaParams, mla_block
    *dims, seq, nseq = shape
    dims = tuple(dims)
    w = O.mla_weights(*dims, seed=13)
    rows = seq * nseq
    h = O.normal_f32(O.stream_seed(6, 1), rows * dims[0]).reshape(rows, dims[0])
    rc, want = O.mla_forward(orc, dims, w, h, seq, threads=8)
    assert rc == 0
    got = mla_block(h, MlaParams(*dims, weights=w, rope_base=1.0e4, precision=scmoe.PREC_BF16),
                    seq)
    err = O.rel_l2(got, want)
    print(f"MLA tensor cores {shape}: rel-L2 {err:.2e}")
    assert np.isfinite(got).all() and err <= TC_TOL, err


def test_mla_tensor_cores_long_sequence(scmoe):
    """Long causal sequences (4096 keys: 32 query tiles, 16 two-tile CTAs per
    head, lazy rescaling over 32 key tiles) at LongCat head widths: the
    tensor-core forward within 2e-2 of the exact device MLA (itself bitwise
    equal to the oracle, test_mla_forward_bitwise)."""
    import torch
    from paper_2509_01322_b200.mla import MlaParams, mla_block
    dims = (512, 128, 128, 4, 128, 64)
    seq, nseq = 4096, 2
    w = O.mla_weights(*dims, seed=41)
    h = torch.from_numpy(O.normal_f32(O.stream_seed(42, 0), seq * nseq * dims[0])
                         .reshape(seq * nseq, dims[0])).cuda()
    exact = mla_block(h, MlaParams(*dims, weights=w, rope_base=1.0e6), seq)
    tc = mla_block(h, MlaParams(*dims, weights=w, rope_base=1.0e6, precision=scmoe.PREC_BF16), seq)
    scmoe.default_context().synchronize()
    exact, tc = exact.cpu().numpy(), tc.cpu().numpy()
    err = O.rel_l2(tc, exact)
    print(f"MLA tensor cores, 2 x 4096 causal: rel-L2 {err:.2e}")
    assert np.isfinite(tc).all() and err <= TC_TOL, err


def test_mla_tensor_core_dims_checked(scmoe):
    from paper_2509_01322_b200.mla import MlaParams, mla_block
    dims = (48, 24, 16, 3, 10, 6)  # not multiples of 64
    w = O.mla_weights(*dims, seed=1)
    h = O.normal_f32(3, 7 * 48).reshape(7, 48)
    with pytest.raises(scmoe.ConfigError):
        mla_block(h, MlaParams(*dims, weights=w, precision=scmoe.PREC_BF16), 7)
