"""The multi-process row-partitioned solve (one process per rank, CUDA IPC-mapped mailboxes and
ghost slots, spin-wait exchange — the 8-GPU code path) on this box's GPU: two processes share
cuda:0 and must reproduce the in-process group solve bit for bit (same rank-ordered sums)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4])
def test_processes_match_group(G):
    port = 29500 + (os.getpid() % 400) + G
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "mp_partition_check.py"), "--same-gpu", "--size", "16384",
           "--max-iters", "25"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["G"] == G and res["ranks_agree"], res
    assert res["same_iterations"] and res["same_history"] and res["x_bit_identical"], res
