"""crmath.cuh (the GPU frame generator's correctly rounded log/cos) on the host.

* tools/crmath_check.cpp: double-double log/cos equal the __float128 values rounded once on the
  generator's own inputs, built with the library's host flags (-ffp-contract=fast).
* HFPG_FRAME_CRMATH=1 host frames differ from the default (glibc, reference-identical) frames
  only in floating values, by at most 2 ulp, on well under 1% of entries."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_crmath_matches_quad(tmp_path):
    exe = tmp_path / "crcheck"
    src = os.path.join(ROOT, "tools", "crmath_check.cpp")
    r = subprocess.run(["g++", "-O3", "-march=x86-64-v3", "-ffp-contract=fast", "-fopenmp", src,
                        "-lquadmath", "-o", str(exe)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("libquadmath unavailable: " + r.stderr[-200:])
    for key in ["", "12345"]:
        out = subprocess.run([str(exe), "20"] + ([key] if key else []), capture_output=True, text=True)
        rep = json.loads(out.stdout)
        assert out.returncode == 0 and rep["quad_mismatch"] == 0 and rep["quad_checked"] > 60000
        # glibc 2.39 is not correctly rounded on a small fraction of draws
        assert rep["normal_mismatch"] < 0.005 * rep["samples"]


@pytest.mark.parametrize("spec", [65536, (24, 16, 12)], ids=str)
def test_host_crmath_switch(H, spec):
    def gen(cr):
        os.environ["HFPG_FRAME_CRMATH"] = "1" if cr else "0"
        try:
            return H.make_frame_3d(*spec, 5, 9) if isinstance(spec, tuple) else H.make_frame(spec, 5, 9)
        finally:
            del os.environ["HFPG_FRAME_CRMATH"]
    a, b = gen(False), gen(True)
    assert (a.cell_order == b.cell_order).all()
    assert (a.A.row_offsets == b.A.row_offsets).all() and (a.A.col_indices == b.A.col_indices).all()
    for x, y in [(a.rho, b.rho), (a.A.values, b.A.values), (a.b, b.b)]:
        assert (x != y).mean() < 0.01
        assert (np.abs(x - y) <= 4.5e-16 * np.maximum(np.abs(y), 1.0)).all()
