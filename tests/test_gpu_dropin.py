"""The drop-in from the reference's side: the reference's own pcg_solve driving
hfp::gpu::factor_applier, and hfp::gpu::pcg_solve<hfp::SolveReport>, against the reference's
CPU factor_applier on the same inputs (oracle/dropin_test.cpp, linked with the unmodified
reference objects)."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.parametrize("n", [8192, 65536])
def test_cpp_dropin_against_reference(n):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    out = subprocess.run([BIN, str(n)], capture_output=True, text=True, timeout=600)
    rep = json.loads(out.stdout.strip().splitlines()[-1])
    assert rep["ok"], rep
    assert rep["apply_rel_l2_vs_ref_f32"] <= 1e-9, rep
