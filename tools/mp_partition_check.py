"""Multi-process row-partitioned solve (one process per rank, CUDA IPC peers, spin-wait
exchange) checked against the in-process group solve of the same system.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/mp_partition_check.py \
        [--size 16384] [--max-iters 40] [--same-gpu]

Every rank maps its peers' mailboxes and z vectors through CUDA IPC handles all-gathered with
torch.distributed (gloo). With --same-gpu all ranks share cuda:0 (time-sliced contexts), which
is how the IPC path is exercised on a single-GPU box. Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--max-iters", type=int, default=40)
    ap.add_argument("--same-gpu", action="store_true")
    a = ap.parse_args()
    import torch.distributed as dist
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    dev = 0 if a.same_gpu else int(os.environ.get("LOCAL_RANK", rank))
    import paper_2605_13343_b200 as H

    def allgather(blob):
        out = [None] * G
        dist.all_gather_object(out, blob)
        return out

    fr = H.make_frame(a.size, 2024, 0)
    rs = H.RankSolver(fr.A, G, rank, allgather, sigma=1e-2, seed=2024, frame=0, device=dev)
    cfg = H.SolveConfig(max_iters=a.max_iters)
    b_loc = fr.b[rs.row_begin: rs.row_begin + rs.n_local]
    rep, x_loc = rs.solve(b_loc, cfg)
    xs = [None] * G
    dist.all_gather_object(xs, (rep.iterations, rep.status.value, rep.residual_history, x_loc))
    if rank == 0:
        x = np.concatenate([t[3] for t in xs])
        grp = H.PartitionGroup(fr.A, G, sigma=1e-2, seed=2024, frame=0, device=dev)
        rg, xg = grp.solve(fr.b, cfg)
        same_its = all(t[0] == rg.iterations for t in xs)
        same_hist = all(t[2] == rg.residual_history for t in xs)
        h0 = np.array(xs[0][2])
        hg = np.array(rg.residual_history)
        m = min(len(h0), len(hg))
        hd = np.abs(h0[:m] - hg[:m]) / np.abs(hg[:m])
        first = int(np.argmax(hd > 0)) if (hd > 0).any() else -1
        print(json.dumps({"G": G, "n": a.size, "iterations": [t[0] for t in xs], "group_iterations": rg.iterations,
                          "same_iterations": same_its, "same_history": same_hist,
                          "x_bit_identical": bool((x == xg).all()),
                          "x_rel": float(np.linalg.norm(x - xg) / np.linalg.norm(xg)),
                          "hist_max_rel": float(hd.max()), "hist_first_diff": first,
                          "ranks_agree": all(t[2] == xs[0][2] for t in xs),
                          "wall_ms": rep.wall_ms}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
