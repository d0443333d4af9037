"""On-disk formats: GPU crc32 throughput vs zlib, HFTC checkpoint load
(file -> device tensor) and MPPF frame load (file -> device system), each against the host
path (read + zlib crc32 + upload). Files live in /tmp of the box. Prints one JSON line.

    python tools/bench_io.py [--n 1048576]
"""
import argparse
import json
import os
import sys
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_13343_b200 as H  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
a = ap.parse_args()
out = {"n": a.n}
dev = H.Device(0)
# crc32 of the factor-tensor-sized buffer (4P bytes)
f = H.init_factors(H.build_partition(a.n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                   H.RngStream(2024, 0, H.RngPurpose.factor_init))
buf = torch.from_numpy(f.data.view(np.uint8)).cuda()
dev.crc32((buf.data_ptr(), buf.numel()))
torch.cuda.synchronize()
t = time.perf_counter()
reps = 5
for _ in range(reps):
    c_gpu = dev.crc32((buf.data_ptr(), buf.numel()))
gpu_s = (time.perf_counter() - t) / reps
t = time.perf_counter()
c_host = zlib.crc32(f.data.view(np.uint8))
host_s = time.perf_counter() - t
assert c_gpu == c_host
out["crc32"] = {"bytes": int(buf.numel()), "gpu_ms": gpu_s * 1e3, "gpu_GBps": buf.numel() / gpu_s / 1e9,
                "zlib_ms": host_s * 1e3, "zlib_GBps": buf.numel() / host_s / 1e9}
# HFTC: write, then load both ways (page cache warm for both: the second read of each)
path = "/tmp/hfpg_bench.hftc"
H.write_checkpoint(f, path)
fr = H.make_frame(a.n, 2024, 0)
dev.load_csr(fr.A)
for _ in range(2):
    t = time.perf_counter()
    dev.load_checkpoint(path)
    t_dev = time.perf_counter() - t
    t = time.perf_counter()
    dev.load_factors(H.read_checkpoint(path).factors)
    t_host = time.perf_counter() - t
out["hftc_load"] = {"bytes": os.path.getsize(path), "device_path_ms": t_dev * 1e3, "host_path_ms": t_host * 1e3}
# MPPF
mp = "/tmp/hfpg_bench.mppf"
H.write_mppf(fr, mp)
for _ in range(2):
    t = time.perf_counter()
    dev.load_mppf(mp)
    t_dev = time.perf_counter() - t
    t = time.perf_counter()
    g = H.read_mppf(mp)
    dev.load_csr(g.A)
    t_host = time.perf_counter() - t
out["mppf_load"] = {"bytes": os.path.getsize(mp), "device_path_ms": t_dev * 1e3, "host_path_ms": t_host * 1e3}
print(json.dumps(out))
