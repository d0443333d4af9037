"""Reference iteration counts for the large parity cases (slow: minutes of single-core CPU).
Runs the UNMODIFIED reference pcg_solve (oracle/_ref) on the product's inputs (2D frames are
bit-identical to make_frame; the 3D frame is the product's new generator, fed to the
reference's generic pcg_solve/apply) and writes tests/golden/ref_iterations.json.

    python tests/golden/gen_iters.py [case ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2605_13343_b200 as H  # noqa: E402  (host generators only; no GPU used)
from oracle.oracle import Ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_iterations.json")

# name -> (frame, sigma of the seeded jacobi_seed tensor, max_iters)
CASES = {
    "2d_8192": (lambda: H.make_frame(8192, 2024, 0), 1e-2, 20000),
    "2d_65536": (lambda: H.make_frame(65536, 2024, 0), 1e-2, 20000),
    "3d_1m_s1e-3": (lambda: H.make_frame_3d(128, 128, 64, 2024, 0), 1e-3, 20000),
    "2d_262144_t0_s1e-3": (lambda: H.make_frame(262144, 2024, H.test_frame_id(262144, 0)), 1e-3,
                           20000),
    "2d_262144_t0_s1e-2": (lambda: H.make_frame(262144, 2024, H.test_frame_id(262144, 0)), 1e-2,
                           20000),
    "3d_1m_s1e-2": (lambda: H.make_frame_3d(128, 128, 64, 2024, 0), 1e-2, 20000),
}


def main(names):
    r = Ref()
    for name in names:
        make, sigma, max_iters = CASES[name]
        fr = make()
        csr = (fr.A.row_offsets, fr.A.col_indices, fr.A.values)
        t = r.init_factors(fr.n, 128, 32, sigma, 2024, fr.frame_index)
        out = {"n": fr.n, "nnz": int(fr.A.nnz()), "frame_index": fr.frame_index, "sigma": sigma}
        for kind, tag in ((1, "jacobi"), (2, "factor")):
            t0 = time.time()
            rep, x, hist = r.pcg_solve(csr, fr.b, kind, 128, 32, t, max_iters=max_iters)
            out[tag] = {"iterations": rep["iterations"], "status": rep["status"],
                        "final_rel": float(hist[-1]), "hist_head": hist[:8].tolist(),
                        "wall_s": time.time() - t0}
            print(name, tag, out[tag]["iterations"], round(time.time() - t0, 1), flush=True)
        res = json.load(open(OUT)) if os.path.exists(OUT) else {}  # merge with concurrent runs
        res[name] = out
        json.dump(res, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
