"""The N > 1 host paths on CPU: two processes over gloo (tools/dist_cpu_check.py) — bench's
rank plumbing and configs[3] sharding, the row partition's halo map and a distributed SpMV."""
import os
import socket
import subprocess
import sys

from conftest import ROOT


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


import pytest


@pytest.mark.parametrize("nproc", [2, 4])
def test_ranks_gloo(nproc):
    env = dict(os.environ, HFPG_BENCH_GLOO="1", CUDA_VISIBLE_DEVICES="")
    for attempt in range(3):  # a rendezvous port can be taken between free_port() and the bind
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
               os.path.join(ROOT, "tools", "dist_cpu_check.py")]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
        if r.returncode == 0 or "ok rank" in r.stdout:
            break
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert all(f"ok rank {q}" in r.stdout for q in range(nproc))
