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


def test_bench_gpus_flag_self_launches():
    """`python bench.py --gpus 2` (no torchrun) re-execs itself under torch.distributed.run with
    two ranks; --check-launch runs the rank plumbing only (gloo on CPU)."""
    env = dict(os.environ, HFPG_BENCH_GLOO="1", CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    import json
    for attempt in range(3):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--check-launch"],
                           capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
        if r.returncode == 0:
            break
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gpus_requested"] == 2
    assert line["max_over_ranks"] == 2.0 and line["frames_covered"]
