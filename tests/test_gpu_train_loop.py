"""train_factors (train.cpp:29-217) on the GPU against the reference's own train_factors run on the
same frames, seed and config (oracle/_ref). The device loss sums its three global dot products in
a parallel order (<= 1e-12 relative per step, test_gpu_train.py), so the trajectories agree to
rounding drift rather than bit for bit (measured: losses to 1e-15 relative over 40 steps); the
held-out PCG counts come from the exact solver, so they differ only where a last-ulp difference
of the float snapshot moves a count (within the north star's +-2)."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def frames(H, n, idx):
    return [H.make_frame(n, 2024, i) for i in idx]


def test_training_history_matches_reference(H, ref):
    n = 1024
    cfg = H.TrainConfig(max_steps=40, log_every=10, lr=2e-3, contexts_per_step=2)
    fr = frames(H, n, [0, 1])
    ev = H.make_frame(n, 2024, 2)
    res = H.train_factors(fr, cfg, seed=7, eval_frame=ev)
    want_f, want, summ = ref.train_factors(n, 2024, [0, 1], 2, cfg.to_c(), 7)
    assert res.history.total_steps == summ["total_steps"] == 40
    assert len(res.history.entries) == len(want) == 4
    for got, w in zip(res.history.entries, want):
        assert got.step == w["step"] and got.lr == w["lr"]
        assert abs(got.train_loss - w["train_loss"]) <= 1e-9 * abs(w["train_loss"]), (got, w)
        assert abs(got.sai_heldout - w["sai_heldout"]) <= 1e-9 * abs(w["sai_heldout"]), (got, w)
        assert abs(got.pcg_iters_heldout - w["pcg_iters_heldout"]) <= 2, (got, w)
    assert rel_l2(res.factors.data.astype(np.float64), want_f.astype(np.float64)) <= 1e-6
    assert '"pcg_iters_heldout":' in res.history.to_jsonl()


def test_plateau_schedule_and_autostop_match_reference(H, ref):
    # a learning rate far too large: the plateau schedule halves it down to the floor and the
    # min-lr auto-stop ends the run, at the same step as the reference's
    n = 256
    cfg = H.TrainConfig(max_steps=400, log_every=2, lr=5.0, contexts_per_step=1, eval_every_logs=0,
                        plateau=H.PlateauConfig(factor=0.1, patience=1, rel_threshold=5e-3), autostop_window=3)
    res = H.train_factors(frames(H, n, [3]), cfg, seed=11)
    _, want, summ = ref.train_factors(n, 2024, [3], 3, cfg.to_c(), 11)
    assert res.history.total_steps == summ["total_steps"]
    assert res.history.auto_stopped == bool(summ["auto_stopped"])
    assert [e.lr for e in res.history.entries] == [w["lr"] for w in want]


def test_trained_checkpoint_beats_jacobi_like_reference(H):
    """tests/golden/trained_8192.hftc (GPU train_factors on the reference's acceptance recipe,
    tools/train_tensor.py --acceptance --n 8192) on BASELINE configs[0]'s system: the reference's
    own pcg_solve with this checkpoint takes 221 iterations against Jacobi's 513
    (tests/golden/ref_iterations.json); the graph solve is within +-2 and the exact solve equal."""
    import json
    import os
    from conftest import ROOT
    want = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_iterations.json")))["2d_8192_trained"]
    fr = H.make_frame(8192, 2024, 0)
    dev = H.Device(0)
    dev.load_csr(fr.A)
    dev.load_checkpoint(os.path.join(ROOT, "tests", "golden", "trained_8192.hftc"))
    dev.set_precond(2)
    x = np.empty(fr.n)
    rep = dev.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(), None, 0)
    assert rep.converged and abs(int(rep.iterations) - want["factor"]["iterations"]) <= 2
    rex = dev.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(), None, 0, exact=True)
    assert int(rex.iterations) == want["factor"]["iterations"]
    assert want["factor"]["iterations"] < want["jacobi"]["iterations"] / 2
