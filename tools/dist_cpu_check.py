"""CPU multi-process check of the N > 1 host paths (gloo), launched as
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P \\
        tools/dist_cpu_check.py
* bench.py's rank plumbing: max over ranks, barrier, configs[3]'s frame sharding (disjoint, complete);
* the row partition (configs[4]): every rank builds its plan on the host; the halo each rank pushes
  to each peer lands exactly in the ghost slots that peer expects (global ids), and a distributed
  SpMV — owned rows + halo received over gloo — reproduces the global A x bit for bit.
Prints "ok rank R" on success.
"""
import os
import sys

os.environ.setdefault("HFPG_BENCH_GLOO", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import partition as P  # noqa: E402

world, rank, local = bench.dist_init()
assert world >= 2 and dist.get_backend() == "gloo"
# bench plumbing
assert bench.max_over_ranks(1.5 + rank, world, local) == 0.5 + world
bench.barrier(world)
got = [None] * world
dist.all_gather_object(got, bench.frames_of(rank, world, 64))
flat = sorted(f for g in got for f in g)
assert flat == list(range(64)), flat
# row partition of a 2D frame over `world` ranks
fr = H.make_frame(8192, 2024, 0)
A = fr.A
pl = P.plan(A, world, rank)
plans = [None] * world
dist.all_gather_object(plans, pl)
for r, pr in enumerate(plans):  # every (sender r -> receiver q) halo matches q's ghost list
    for q, pq in enumerate(plans):
        if q == r:
            continue
        a, b = int(pr.send_off[q]), int(pr.send_off[q + 1])
        rows = pr.send_rows[a:b].astype(np.int64) + pr.row_begin
        assert np.array_equal(pq.ghost_cols[pr.send_slot[a:b]].astype(np.int64), rows), (r, q)
# distributed SpMV: owned x + ghosts received from the peers over gloo
x = np.random.default_rng(5).standard_normal(A.n_rows)
nl, r0 = pl.n_local, pl.row_begin
mine = x[r0:r0 + nl].copy()
owned = [None] * world
dist.all_gather_object(owned, mine)
ghost = np.empty(len(pl.ghost_cols))
for i, gcol in enumerate(pl.ghost_cols):  # ghost gcol lives on rank gcol // nl
    q = int(gcol) // nl
    ghost[i] = owned[q][int(gcol) - q * nl]
xl = np.concatenate([mine, ghost])
ro = np.asarray(A.row_offsets[r0:r0 + nl + 1], np.int64) - int(A.row_offsets[r0])
vals = np.asarray(A.values)[int(A.row_offsets[r0]):int(A.row_offsets[r0 + nl])]
y = np.zeros(nl)
for i in range(nl):
    acc = 0.0
    for p in range(ro[i], ro[i + 1]):
        acc += vals[p] * xl[pl.local_cols[p]]
    y[i] = acc
ys = [None] * world
dist.all_gather_object(ys, y)
yg = np.concatenate(ys)
ro_g = np.asarray(A.row_offsets, np.int64)
want = np.zeros(A.n_rows)
for i in range(A.n_rows):
    acc = 0.0
    for p in range(ro_g[i], ro_g[i + 1]):
        acc += A.values[p] * x[A.col_indices[p]]
    want[i] = acc
assert np.array_equal(yg, want)
print("ok rank", rank, flush=True)
dist.destroy_process_group()
