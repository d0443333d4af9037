"""GPU training pieces against the reference (adjoint.cpp, train.cpp):
the double-precision batched apply and its adjoint are bit-identical to factor_apply_batch /
factor_apply_batch_adjoint (same operation order, FMA-contracted like the reference build); the
probe losses and their gradients match loss_gradient to f64 rounding (the global dot products
are reduced in a different order); the AdamW step matches train.cpp's update."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def csr_of(A):
    return (np.ascontiguousarray(A.row_offsets, np.uint64), np.ascontiguousarray(A.col_indices, np.uint32),
            np.ascontiguousarray(A.values, np.float64))


def params64(H, n, sigma=0.05, seed=3):
    f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, sigma,
                       H.RngStream(seed, 0, H.RngPurpose.factor_init))
    return f.data.astype(np.float64)


@pytest.mark.parametrize("n,kz", [(1024, 64), (4096, 16), (2048, 5)])
def test_batch_apply_and_adjoint_bit_exact(H, ref, n, kz):
    fr = H.make_frame(n, 2024, 1)
    dev = H.Device(0)
    dev.load_csr(fr.A)
    P = params64(H, n)
    rng = np.random.default_rng(n + kz)
    X = rng.standard_normal(n * kz)
    BY = rng.standard_normal(n * kz)
    y = H.factor_apply_batch(P, X, kz, dev)
    g = H.factor_apply_batch_adjoint(P, BY, dev)
    yr, gr = ref.apply_batch_adjoint(n, P, fr.A.diagonal(), X, kz, BY)
    assert np.array_equal(y.view(np.uint64), yr.view(np.uint64))
    assert np.array_equal(g.view(np.uint64), gr.view(np.uint64)), np.max(np.abs(g - gr))


@pytest.mark.parametrize("kind", [0, 1])
def test_loss_gradient(H, ref, kind):
    n, kz = 2048, 32
    fr = H.make_frame(n, 2024, 2)
    dev = H.Device(0)
    dev.load_csr(fr.A)
    P = params64(H, n, sigma=0.02)
    Z = np.random.default_rng(9).standard_normal(n * kz)
    norm_a = 7.5
    r = H.loss_gradient(P, Z, kz, H.LossKind(kind), dev, norm_a=norm_a)
    loss, deg, grad = ref.loss_gradient(csr_of(fr.A), P, Z, kz, kind, norm_a)
    assert not r.degenerate and not deg
    assert abs(r.loss - loss) <= 1e-12 * max(1.0, abs(loss))
    rel = np.linalg.norm(r.grad - grad) / np.linalg.norm(grad)
    assert rel <= 1e-12, rel


def test_loss_degenerate(H):
    n, kz = 1024, 8
    fr = H.make_frame(n, 2024, 3)
    dev = H.Device(0)
    dev.load_csr(fr.A)
    r = H.loss_gradient(np.zeros(len(params64(H, n))), np.ones(n * kz), kz, H.LossKind.cosine, dev)
    assert r.degenerate and not np.any(r.grad)


def test_adamw_step(H):
    dev = H.Device(0)
    rng = np.random.default_rng(4)
    cnt = 10000
    p, g, m1, m2 = (rng.standard_normal(cnt) for _ in range(4))
    m2 = np.abs(m2)
    tp, tg, tm1, tm2 = (torch.from_numpy(a.copy()).cuda() for a in (p, g, m1, m2))
    lr, b1, b2, eps, wd, clip, step = 1e-3, 0.9, 0.999, 1e-8, 0.01, 1.0, 3
    gn = H.adamw_step(dev, tp.data_ptr(), tg.data_ptr(), tm1.data_ptr(), tm2.data_ptr(), cnt, step, lr, b1, b2,
                      eps, wd, clip)
    # train.cpp:136-160 in numpy
    norm = np.sqrt(np.sum(g * g))
    assert abs(gn - norm) <= 1e-12 * norm
    gg = g * (clip / norm) if norm > clip else g
    m1n = b1 * m1 + (1 - b1) * gg
    m2n = b2 * m2 + (1 - b2) * gg * gg
    pn = p - lr * ((m1n / (1 - b1 ** step)) / (np.sqrt(m2n / (1 - b2 ** step)) + eps) + wd * p)
    np.testing.assert_allclose(tp.cpu().numpy(), pn, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(tm1.cpu().numpy(), m1n, rtol=1e-13, atol=1e-16)
