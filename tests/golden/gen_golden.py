"""Generate tests/golden/golden.npz from the UNMODIFIED reference (oracle/_ref/libhfpref.so,
built from /root/reference/proj by oracle/Makefile). Run here, where /root/reference exists;
the .npz is committed so the tests can pin the oracle and the product without the reference.

    python tests/golden/gen_golden.py
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Ref, build  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def diag_of(fr):
    d = np.zeros(fr["n"])
    ro, ci, v = fr["row_offsets"], fr["col_indices"], fr["values"]
    for i in range(fr["n"]):
        for p in range(ro[i], ro[i + 1]):
            if ci[p] == i:
                d[i] = v[p]
    return d


def main():
    build()
    r = Ref()
    g = {}
    # test_core.cpp:333-335 Morton known answers
    g["morton"] = np.array([r.lib.ref_morton_encode(x, y) for x, y in ((0, 0), (1, 1), (3, 5))],
                           np.uint32)
    # acceptance.cpp:57-68 packed widths
    g["packed_widths"] = np.array([r.packed_width(n, 128, 32) for n in (1024, 2048, 8192, 16384)],
                                  np.uint64)
    g["partition_2048_128"] = r.partition(2048, 128)
    g["rng_bits_2024_0_4"], g["rng_normals_2024_0_4"] = r.rng(2024, 0, 4, 64)
    # frames: full arrays for a small one, digests for larger ones
    fr = r.make_frame(256, 9, 1)
    for k in ("cell_order", "rho", "row_offsets", "col_indices", "values", "b"):
        g[f"frame256_{k}"] = fr[k]
    digests = []
    for n, seed, fi in ((1024, 2024, 0), (8192, 2024, 0), (65536, 2024, 0), (2048, 42, 0)):
        f = r.make_frame(n, seed, fi)
        digests.append([f"{n}/{seed}/{fi}"] + [sha(f[k]) for k in
                                               ("cell_order", "rho", "row_offsets", "col_indices",
                                                "values", "b")])
    g["frame_digests"] = np.array(digests)
    # init_factors digests (factor_tensor.cpp:30-39)
    fi_d = []
    for n, sigma, seed, frm in ((1024, 1e-2, 7, 3), (8192, 1e-2, 2024, 0), (512, 1.0, 8, 512)):
        fi_d.append([f"{n}/{sigma}/{seed}/{frm}", sha(r.init_factors(n, 128, 32, sigma, seed, frm))])
    g["init_digests"] = np.array(fi_d)
    # apply<float> / apply<double> on a sigma=1 tensor at N=512 (crit. 3 style)
    rng = np.random.default_rng(512)
    f512 = r.init_factors(512, 128, 32, 1.0, 8, 512)
    d512 = 1.0 + np.abs(rng.standard_normal(512))
    r512 = rng.standard_normal(512)
    g["apply512_diag"], g["apply512_r"] = d512, r512
    g["apply512_y_f32"] = r.apply_f32(512, 128, 32, f512, d512, r512)
    g["apply512_y_f64"] = r.apply_f64_of_f32(512, 128, 32, f512, d512, r512)
    # PCG on make_frame(1024, 7, 3) (test_pcg.cpp:169-179 setup)
    f = r.make_frame(1024, 7, 3)
    csr = (f["row_offsets"], f["col_indices"], f["values"])
    t = r.init_factors(1024, 128, 32, 1e-2, 7, 3)
    for kind, name in ((0, "identity"), (1, "jacobi"), (2, "factor")):
        rep, x, hist = r.pcg_solve(csr, f["b"], kind, 128, 32, t)
        g[f"pcg1024_{name}_iters"] = np.array([rep["iterations"]])
        g[f"pcg1024_{name}_hist"] = hist
        g[f"pcg1024_{name}_x"] = x
    np.savez_compressed(OUT, **g)
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
