"""The fast path's A/B kernel variants agree with the defaults (each variant is selected by an
environment switch read once per process, so every arm runs in its own subprocess):

  HFPG_PROLONG_WARP=1  k_prolong_fast instead of k_prolong_tma   (same arithmetic lane for lane)
  HFPG_COARSE_SPLIT=1  k_sums_tree + k_tiles_all instead of k_coarse_coop (same pairwise trees)
  HFPG_PDL=1           programmatic dependent launch of the solve kernels

The preconditioner apply must be bit-identical across the arms (z depends only on the per-row
arithmetic, which the variants share); a solve must take the same number of iterations and
agree to rounding (r.z is summed in a different order by the two prolongations)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ARMS = {"default": {}, "prolong_warp": {"HFPG_PROLONG_WARP": "1"}, "coarse_split": {"HFPG_COARSE_SPLIT": "1"},
        "pdl": {"HFPG_PDL": "1"}}

SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, ROOT)
import bench
import paper_2605_13343_b200 as H
from paper_2605_13343_b200 import _native as N
out = {}
for cfg_name in ("2d_8192", "2d_65536", "3d_1m"):
    fr, f = bench.make_inputs(bench.CONFIGS[cfg_name], 0)
    d = H.Device(0)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(fr.n)
    z = H.apply(f, fr.A.diagonal(), r, device=d)
    d.load_csr(fr.A)
    d.load_factors(f)
    d.set_precond(2)
    x = np.empty(fr.n)
    rep = d.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(max_iters=3000), None, N.HOST)
    out[cfg_name] = {"z": hashlib.sha256(z.tobytes()).hexdigest(), "iters": int(rep.iterations),
                     "x": x[::997].tolist()}
print("RESULT " + json.dumps(out))
"""


def run_arm(env_extra):
    env = dict(os.environ, **env_extra)
    for k in ("HFPG_PROLONG_WARP", "HFPG_COARSE_SPLIT", "HFPG_PDL"):
        if k not in env_extra:
            env.pop(k, None)
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], capture_output=True, text=True,
                       timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("RESULT ")][-1][7:])


def test_fast_path_variants_agree():
    res = {name: run_arm(e) for name, e in ARMS.items()}
    base = res["default"]
    for name, got in res.items():
        for cfg, v in got.items():
            b = base[cfg]
            assert v["z"] == b["z"], (name, cfg, "apply not bit-identical")
            assert v["iters"] == b["iters"], (name, cfg, v["iters"], b["iters"])
            np.testing.assert_allclose(v["x"], b["x"], rtol=1e-9, atol=1e-12 * max(1.0, np.abs(b["x"]).max()),
                                       err_msg=f"{name} {cfg}")
