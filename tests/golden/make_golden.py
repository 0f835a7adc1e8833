"""Regenerate tests/golden/*.npz from the REFERENCE itself (oracle/_ref,
compiled from /root/reference/proj/include).  Run in the dev container:

    python tests/golden/make_golden.py

config_a.npz: BASELINE config A (tiny ScMoE layer fp32: T=512, d=256, 8 FFN +
4 zero experts, top-2, K_e=1, inter=128) -- route_topk + moe_forward outputs.
router_longcat.npz: LongCat router (d=6144, 512+256 experts, top-12) on 64
tokens with non-zero FFN biases -- indices / gates / ffn_count.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle as O  # noqa: E402
from _oracle import ptr, ptr_array  # noqa: E402


def ref_route(ref, x, w, n, z, k, ke, b):
    T, d = x.shape
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k)
    c = np.empty(T, np.uint32)
    assert ref.ref_route_topk_f32(ptr(x), T, d, ptr(w), n, z, k, ke, 0.0, ptr(b), ptr(idx), ptr(g),
                                  ptr(c), None, 8) == 0
    return idx, g, c


def main():
    ref = O.ref()
    T, d, n, z, k, ke, I = 512, 256, 8, 4, 2, 1, 128
    sx, sw, sb = 99, 5, 21
    x = O.normal_f32(O.stream_seed(sx, 0), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(sw, 0), d * (n + z), 1.0 / d).reshape(d, n + z)
    idx, g, c = ref_route(ref, x, w, n, z, k, ke, np.zeros(n + z))
    w_in = [O.uniform_f32(O.stream_seed(sb, 2 * e), d * I, 1.0 / d).reshape(d, I) for e in range(n)]
    w_out = [O.uniform_f32(O.stream_seed(sb, 2 * e + 1), I * d, 1.0 / d).reshape(I, d)
             for e in range(n)]
    out = np.empty((T, d), np.float32)
    assert ref.ref_moe_forward_f32(ptr(x), T, d, ptr(idx), ptr(g), k, n, z, ptr_array(w_in),
                                   ptr_array(w_out), I, 1, 0, ptr(out), 8) == 0
    np.savez_compressed(os.path.join(HERE, "config_a.npz"), T=T, d=d, n=n, z=z, k=k, ke=ke, I=I,
                        seed_x=sx, seed_w=sw, seed_bank=sb, indices=idx, gates=g, ffn_count=c,
                        out=out)

    T, d, n, z, k, ke = 64, 6144, 512, 256, 12, 8
    x = O.normal_f32(O.stream_seed(sx, 1), T * d).reshape(T, d)
    w = O.uniform_f32(O.stream_seed(sw, 1), d * (n + z), 1.0 / d).reshape(d, n + z)
    b = np.zeros(n + z)
    b[:n] = O.normal_f64(17, n) * 1e-3
    idx, g, c = ref_route(ref, x, w, n, z, k, ke, b)
    np.savez_compressed(os.path.join(HERE, "router_longcat.npz"), T=T, d=d, n=n, z=z, k=k, ke=ke,
                        seed_x=sx, seed_w=sw, bias=b, indices=idx, gates=g, ffn_count=c)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
