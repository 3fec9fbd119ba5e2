"""GPU unit test of the tcgen05 operand path: one M=128 x N=32 x K=16 FP16 MMA through the same
shared-memory descriptors and instruction descriptor the rasterizer uses, read back with
tcgen05.ld, against a float64 reference of the same op.  Also checks the exactness premise of the
monomial formulation: pixel monomials relative to a tile centre are exact in FP16, and the hi/lo
split reproduces an FP32 coefficient vector to ~2^-22."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mma(a16, b16):
    from tools.debug.build import load  # the microbenchmark library (not the product ABI)
    lib = load()
    d = np.zeros((128, 32), np.float32)
    a = np.ascontiguousarray(a16.view(np.uint16))
    b = np.ascontiguousarray(b16.view(np.uint16))
    rc = lib.tgs_debug_mma(a.ctypes.data, b.ctypes.data, d.ctypes.data)
    assert rc == 0
    return d


def test_mma_random():
    rng = np.random.default_rng(1)
    a = rng.uniform(-2, 2, (128, 16)).astype(np.float16)
    b = rng.uniform(-2, 2, (32, 16)).astype(np.float16)
    d = _mma(a, b)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert np.max(np.abs(d - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_mma_layout_one_hot():
    # each output must select exactly one (row, col, k) product: catches LBO/SBO/N/M mix-ups
    a = np.zeros((128, 16), np.float16)
    b = np.zeros((32, 16), np.float16)
    for r in range(128):
        a[r, r % 16] = 1.0 + r / 128.0
    for c in range(32):
        b[c, (c * 3) % 16] = 1.0 + c / 32.0
    d = _mma(a, b)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert np.array_equal(d, ref.astype(np.float32))


def test_monomial_contraction_precision():
    """w.phi through the tensor core vs an fp64 evaluation of the quadratic form."""
    rng = np.random.default_rng(2)
    ux = (np.arange(128) % 16) - 7.5
    uy = (np.arange(128) // 16) - 7.5
    phi = np.stack([ux * ux, ux * uy, uy * uy, ux, uy, np.ones(128)], 1)
    assert np.array_equal(phi.astype(np.float16).astype(np.float64), phi)  # exact in FP16
    a = np.zeros((128, 16), np.float16)
    a[:, 0:6] = phi
    a[:, 6:12] = phi
    b = np.zeros((32, 16), np.float16)
    wref = np.zeros((32, 6))
    for j in range(32):
        s = rng.uniform(0.6, 12.0, 2)
        th = rng.uniform(0, np.pi)
        R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        cov = R @ np.diag(s * s) @ R.T + 0.3 * np.eye(2)
        q = np.linalg.inv(cov)
        qa, qb, qc = q[0, 0], q[0, 1], q[1, 1]
        m = rng.uniform(-12, 12, 2)
        l2e = 1.4426950408889634
        w = l2e * np.array([-qa / 2, -qb, -qc / 2, qa * m[0] + qb * m[1], qb * m[0] + qc * m[1],
                            -(qa * m[0] ** 2 / 2 + qb * m[0] * m[1] + qc * m[1] ** 2 / 2)])
        w32 = w.astype(np.float32)
        hi = w32.astype(np.float16)
        lo = (w32 - hi.astype(np.float32)).astype(np.float16)
        b[j, 0:6] = hi
        b[j, 6:12] = lo
        wref[j] = w
    d = _mma(a, b)
    ref = phi @ wref.T
    live = ref > -12.0  # the region that can reach alpha >= 1/255
    err = np.abs(d.astype(np.float64) - ref)[live]
    assert err.max() < 2e-4, err.max()
