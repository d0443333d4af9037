"""`python -m paper_2605_13343_b200 solve ...`: the reference CLI's `hfp solve` (hfp_cli.cpp:399-437)
on the GPU path, with the `hfactor-gpu` method tag next to the reference's method names
(SURVEY 8(b)). Frames come from an MPPF file (`--frame`) or are generated (`--n` / `--dims`).

    python -m paper_2605_13343_b200 solve --frame f.mppf --method hfactor-gpu --checkpoint m.hftc
    python -m paper_2605_13343_b200 solve --n 65536 --method jacobi --report rep.json
Methods: hfactor-gpu (alias hfactor), jacobi, identity (alias none), ic0. `--exact`: the bit-exact
loop (hfpg_pcg_solve_exact). Exit status 0 when converged, 3 otherwise (kExitNumerical)."""
import argparse
import json
import sys

import numpy as np

K_EXIT_NUMERICAL = 3  # hfp_cli.cpp:30


def _frame(H, a):
    if a.frame:
        return H.read_mppf(a.frame), a.frame
    if a.dims:
        nx, ny, nz = a.dims
        return H.make_frame_3d(nx, ny, nz, a.seed, a.frame_index), f"3d_{nx}x{ny}x{nz}"
    return H.make_frame(a.n, a.seed, a.frame_index), f"2d_{a.n}"


def _applier(H, a, fr):
    m = a.method
    if m in ("identity", "none"):
        return H.identity_applier()
    if m == "jacobi":
        return H.jacobi_applier(fr.A)
    if m == "ic0":
        return H.ic0_applier(H.ic0_factorize(fr.A))
    if m in ("hfactor-gpu", "hfactor"):
        if a.checkpoint:
            f = H.read_checkpoint(a.checkpoint).factors
        else:  # no model: the jacobi_seed initialisation (factor_tensor.cpp:30-39)
            f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, a.sigma,
                               H.RngStream(a.seed, fr.frame_index, H.RngPurpose.factor_init))
        return H.factor_applier(f, fr.A)
    raise SystemExit(f"solve: unknown method {m!r}")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2605_13343_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="PCG solve of one frame (hfp solve)")
    g = s.add_mutually_exclusive_group()
    g.add_argument("--frame", help="MPPF v1 file")
    g.add_argument("--n", type=int, default=65536, help="generated 2D frame size")
    g.add_argument("--dims", type=int, nargs=3, metavar=("NX", "NY", "NZ"), help="generated 3D frame")
    s.add_argument("--seed", type=int, default=2024)
    s.add_argument("--frame-index", type=int, default=0)
    s.add_argument("--method", default="hfactor-gpu")
    s.add_argument("--checkpoint", default="", help="HFTC checkpoint (factor methods)")
    s.add_argument("--sigma", type=float, default=1e-2, help="jacobi_seed sigma when no checkpoint")
    s.add_argument("--rtol", type=float, default=1e-8)
    s.add_argument("--max-iters", type=int, default=20000)
    s.add_argument("--exact", action="store_true", help="bit-exact loop (hfpg_pcg_solve_exact)")
    s.add_argument("--report", default="", help="write SolveReport JSON here")
    s.add_argument("--residuals", default="", help="write per-iteration residual vectors (JSON lines)")
    a = ap.parse_args(argv)

    import paper_2605_13343_b200 as H
    fr, frame_id = _frame(H, a)
    M = _applier(H, a, fr)
    rv = [] if a.residuals else None
    rep = H.pcg_solve(fr.A, fr.b, M, H.SolveConfig(rtol=a.rtol, max_iters=a.max_iters), exact=a.exact,
                      residual_vectors=rv)
    rep.method = a.method
    rep.frame_id = a.frame or frame_id
    print(f"{rep.method}: {'converged' if rep.converged else 'failed'} in {rep.iterations} iterations, "
          f"{rep.wall_ms:g} ms")
    if a.report:
        with open(a.report, "w") as fh:
            fh.write(rep.to_json() + "\n")
    if rv is not None:
        with open(a.residuals, "w") as fh:
            for k, r in enumerate(rv):
                fh.write(json.dumps({"iteration": k + 1, "rel_residual": rep.residual_history[k],
                                     "residual": np.asarray(r).tolist()}) + "\n")
    return 0 if rep.converged else K_EXIT_NUMERICAL


if __name__ == "__main__":
    sys.exit(main())
