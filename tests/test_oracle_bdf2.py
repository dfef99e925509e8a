"""Pins of the oracle's BDF2 integrator (NEXT-4; §3.1, reading C2 in DESIGN.md).

* steady state (SPEC S:107, S:116 worked cases): x^t = x^{t-1}, v = 0, no gravity -> xhat = x^t,
  and a state at rest stays at rest with v = v*;
* BDF2 integrates a constant acceleration exactly when its history is exact (a textbook
  property of the method: it is exact on quadratics): free fall of C1 without its Dirichlet
  vertices, started from the exact parabola at t = -h and t = 0, stays on x0 + g t^2 / 2 to
  rounding -- this pins the predictor and the velocity update, including the corrected
  9/(4h^2) factor of the acceleration (the printed 4h^2/9 breaks it);
* momentum balance at convergence: 9/(4h^2)(x^{t+1} - xtilde) = M^-1 f(x^{t+1}) + g at the free
  vertices (to the Newton tolerance), which pins the alpha = 4/9 scaling of the potentials.
"""
import dataclasses

import numpy as np

from oracle import fem, ip, solver
from precompute.basis import build_basis
from precompute.mesh import make_scene


def test_bdf2_predictor_steady_state():
    s = make_scene(1)
    m = ip.make_model(s)
    m.gravity = np.zeros(3)
    x = m.X + 0.01
    v = np.zeros_like(x)
    assert np.array_equal(ip.predictor_bdf2(m, x, v, x, v), x * 0 + (4.0 * x - x) / 3.0)
    assert np.abs(ip.predictor_bdf2(m, x, v, x, v) - x).max() < 1e-15


def test_bdf2_exact_on_free_fall():
    s = make_scene(1)
    s = dataclasses.replace(s, dbc=np.zeros(0, np.int32))   # free body: a rigid translation, Psi = 0
    b = build_basis(s, workers=1)
    sim = solver.OracleSim(s, b, integrator="bdf2")
    g, h = np.asarray(s.gravity), s.h
    x0 = s.X.copy()
    # exact history: x(t) = x0 + g t^2 / 2, v(t) = g t at t = -h (previous) and t = 0 (current)
    sim.x_prev, sim.v_prev = x0 + 0.5 * g * h ** 2, -g * h + 0 * x0
    sim.x, sim.v = x0.copy(), np.zeros_like(x0)
    for n in range(1, 5):
        sim.timestep()
        exact = x0 + 0.5 * g * (n * h) ** 2
        assert np.abs(sim.x - exact).max() <= 1e-12, (n, np.abs(sim.x - exact).max())
        assert np.abs(sim.v - g * n * h).max() <= 1e-10


def test_bdf2_momentum_balance_at_convergence():
    s = make_scene(1)
    s = dataclasses.replace(s, eps=1e-10)
    b = build_basis(s, workers=1)
    sim = solver.OracleSim(s, b, integrator="bdf2")
    for _ in range(3):                      # IE first step, then BDF2
        sim.timestep()
    assert sim.model.alpha == 4.0 / 9.0
    m, h = sim.model, s.h
    xtilde = sim.xhat - (4.0 / 9.0) * h ** 2 * m.gravity[None, :]
    a = 9.0 / (4.0 * h ** 2) * (sim.x - xtilde)
    ge = fem.element_gradient(sim.x, m.tets, m.Bm, m.V, m.mu, m.lam)
    f = np.zeros_like(sim.x)
    for k in range(4):
        np.add.at(f, m.tets[:, k], -ge[:, 3 * k:3 * k + 3])
    acc = f / m.mass[:, None] + m.gravity[None, :]
    free = m.free
    err = np.abs(a[free] - acc[free]).max() / np.abs(acc[free]).max()
    assert err < 1e-6, err
    # with alpha = 1 (implicit Euler's scaling) the balance would be off by 9/4
    assert np.abs(a[free] - (4.0 / 9.0) * acc[free]).max() > 0.1 * np.abs(acc[free]).max()
