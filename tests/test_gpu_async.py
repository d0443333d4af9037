"""hfpg_pcg_solve_async / _wait: independent systems on separate handles solved concurrently on
one GPU give exactly the results of one-at-a-time solves (same kernels, same order per handle)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_concurrent_solves_match_sequential(H):
    import torch
    from paper_2605_13343_b200 import _native as N
    devs, bs, xs, want = [], [], [], []
    for i in range(4):
        n = [4096, 16384, 65536, 131072][i]
        fr = H.make_frame(n, 2024, i)
        f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                           H.RngStream(2024, i, H.RngPurpose.factor_init))
        d = H.Device(0)
        d.load_csr(fr.A)
        d.load_factors(f)
        d.set_precond(2)
        x = np.empty(n)
        rep = d.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(), None, N.HOST)
        want.append((int(rep.iterations), x))
        devs.append(d)
        bs.append(torch.from_numpy(fr.b).cuda())
        xs.append(torch.empty_like(bs[-1]))
    for d, b, x in zip(devs, bs, xs):
        d.solve_async(b.data_ptr(), x.data_ptr(), H.SolveConfig(), N.DEVICE)
    for d, x, (its, xw) in zip(devs, xs, want):
        rep = d.wait()
        assert int(rep.iterations) == its
        assert (x.cpu().numpy() == xw).all()
    with pytest.raises(ValueError):
        devs[0].wait()  # nothing in flight


def test_second_solve_while_one_is_in_flight_is_refused(H):
    # the handle's pinned report buffer also stages the config: a second enqueue before the
    # wait would upload the first solve's scalars as its config
    from paper_2605_13343_b200 import _native as N
    fr = H.make_frame(4096, 2024, 0)
    d = H.Device(0)
    d.load_csr(fr.A)
    d.set_precond(1)
    x = np.empty(fr.n)
    d.solve_async(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(), N.HOST)
    with pytest.raises(ValueError):
        d.solve_async(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(rtol=1e-3), N.HOST)
    with pytest.raises(ValueError):
        d.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(), None, N.HOST)
    rep = d.wait()
    ref = H.pcg_solve(fr.A, fr.b, H.jacobi_applier(fr.A))
    assert int(rep.iterations) == ref.iterations
