"""Dot-product summation-order sensitivity of the PCG iteration count (test infrastructure).

The reference sums every f64 dot product sequentially (pcg.cpp), a parallel solver cannot. This
runs the CPU oracle — whose apply is bit-identical to the reference's — with the reference's
sequential dots and with two other valid orders (ORC_DOT_MODE 1: 128-element blocks combined
pairwise, like a GPU reduction; 2: compensated, ~exact), and records the iteration counts as
`dot_order_band` next to the reference count in ref_iterations.json. On long, chaotic solves
(N >= 262,144 here) the order alone moves the count by several iterations; the parity tests use
the band, widened by +-2, where it is recorded.

    python tests/golden/gen_dot_band.py CASE [CASE ...]
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "ref_iterations.json")

CHILD = r"""
import json, os, sys
sys.path.insert(0, %r)
import paper_2605_13343_b200 as H
from oracle.oracle import Oracle
case = json.load(open(%r))[sys.argv[1]]
n = case["n"]
fr = H.make_frame(n, 2024, case["frame_index"])
f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, case["sigma"],
                   H.RngStream(2024, fr.frame_index, H.RngPurpose.factor_init))
rep, x, h = Oracle().pcg_solve((fr.A.row_offsets, fr.A.col_indices, fr.A.values), fr.b, 2, 128, 32, f.data)
print(rep["iterations"])
""" % (ROOT, OUT)


def main(cases):
    for name in cases:
        procs = {m: subprocess.Popen([sys.executable, "-c", CHILD, name], stdout=subprocess.PIPE, text=True,
                                     env=dict(os.environ, ORC_DOT_MODE=str(m))) for m in (0, 1, 2)}
        its = {m: int(p.communicate()[0].strip()) for m, p in procs.items()}
        d = json.load(open(OUT))
        d[name]["dot_order_band"] = {"oracle_sequential": its[0], "oracle_blocked": its[1],
                                     "oracle_compensated": its[2]}
        json.dump(d, open(OUT, "w"), indent=1)
        print(name, its, "reference", d[name]["factor"]["iterations"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
