"""The per-thread 9x9 PSD projection of the CUDA element kernel (csrc/eig9.cuh), compiled for
the host with g++, against numpy's eigh clamp (reading R2: P+(H) = V max(Lambda,0) V^T).

Not oracle code: the oracle's own PSD step is oracle/fem.psd_project; this test checks the
arithmetic of the GPU algorithm (tridiagonalisation, QL, inverse iteration) on hard spectra."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2508_13386_b200", "csrc")
IU = np.triu_indices(9)


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("eig9") / "eig9_driver")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, os.path.join(ROOT, "tests", "native", "eig9_driver.cpp"),
                    "-o", exe], check=True)
    return exe


def run(exe, mats):
    packed = np.stack([m[IU] for m in mats]).astype(np.float64)
    out = subprocess.run([exe], input=packed.tobytes(), capture_output=True, check=True).stdout
    res = np.frombuffer(out, dtype=np.float64).reshape(len(mats), 46)
    P = np.zeros((len(mats), 9, 9))
    for k in range(len(mats)):
        P[k][IU] = res[k, 1:]
        P[k] = P[k] + np.triu(P[k], 1).T
    return res[:, 0].astype(int), P


def clamp(m):
    w, V = np.linalg.eigh(m)
    return (V * np.maximum(w, 0)) @ V.T


def spectra(rng, n):
    mats = []
    for k in range(n):
        Q, _ = np.linalg.qr(rng.standard_normal((9, 9)))
        kind = k % 6
        if kind == 0:
            lam = rng.standard_normal(9)
        elif kind == 1:   # clustered negative eigenvalues
            lam = np.concatenate([np.full(3, -1.0) + 1e-13 * rng.standard_normal(3), rng.uniform(0.1, 5, 6)])
        elif kind == 2:   # zero and tiny eigenvalues of both signs
            lam = np.concatenate([[0.0, 1e-15, -1e-15, -1e-9], rng.uniform(-1, 5, 5)])
        elif kind == 3:   # large dynamic range
            lam = np.concatenate([[-1e-6, -1e-3], 10.0 ** rng.uniform(-3, 6, 7)])
        elif kind == 4:   # all negative / all positive
            lam = -rng.uniform(0.1, 2, 9) if k % 12 == 4 else rng.uniform(0.1, 2, 9)
        else:             # repeated positive + one negative
            lam = np.concatenate([np.full(8, 2.0), [-0.5]])
        mats.append((Q * lam) @ Q.T)
    return mats


def test_psd_projection_random_spectra(driver):
    rng = np.random.default_rng(11)
    mats = spectra(rng, 600)
    st, P = run(driver, mats)
    assert (st >= 0).all()
    for m, p in zip(mats, P):
        ref = clamp(m)
        scale = np.abs(m).max()
        assert np.abs(p - ref).max() <= 1e-12 * scale, np.abs(p - ref).max() / scale


def test_psd_projection_structured_inputs(driver):
    # diagonal, already tridiagonal, block-diagonal (exact zeros in the reduction), PSD input
    rng = np.random.default_rng(5)
    mats = [np.diag(rng.standard_normal(9)), np.diag([1, -2, 3, 0, 0, -1, 5, 0, 2.0])]
    T = np.diag(rng.standard_normal(9)) + np.diag(rng.standard_normal(8), 1)
    mats.append(T + np.triu(T, 1).T)
    B = np.zeros((9, 9))
    B[:4, :4] = spectra(rng, 1)[0][:4, :4]
    B[4:, 4:] = spectra(rng, 1)[0][4:, 4:]
    mats.append(B)
    A = rng.standard_normal((9, 9))
    mats.append(A @ A.T)
    st, P = run(driver, mats)
    assert (st >= 0).all()
    for m, p in zip(mats, P):
        assert np.abs(p - clamp(m)).max() <= 1e-12 * np.abs(m).max()
    assert st[-1] == 0   # PSD input: nothing clamped, Q T Q^T returned (= M to rounding)
    assert np.abs(P[-1] - mats[-1]).max() <= 1e-14 * np.abs(mats[-1]).max()


def test_psd_projection_element_hessians(driver):
    """Reduced element Hessians Q^T H_e Q of the stable Neo-Hookean energy (oracle/fem) under
    compression, stretch, shear and near-inversion."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle import fem
    rng = np.random.default_rng(3)
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]) * 0.1
    Dm = np.stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]], axis=1)
    Bm = np.linalg.inv(Dm)
    V = np.linalg.det(Dm) / 6
    Q4 = 0.5 * np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1.0]])
    Q = np.kron(Q4, np.eye(3))
    mats = []
    for k in range(300):
        amp = [1e-4, 1e-2, 0.2, 0.5][k % 4]
        F = np.eye(3) + amp * rng.standard_normal((3, 3))
        if np.linalg.det(F) <= 0.05:
            continue
        x = X @ F.T
        mu, lam = 3e5, 2.7e6
        H = fem.element_hessian(x, np.arange(4)[None], Bm[None], np.array([V]), np.array([mu]),
                                np.array([lam]))[0]
        mats.append(Q.T @ H @ Q)
    st, P = run(driver, mats)
    assert (st >= 0).all()
    assert max(st) <= 6
    for m, p in zip(mats, P):
        assert np.abs(p - clamp(m)).max() <= 1e-12 * np.abs(m).max()
