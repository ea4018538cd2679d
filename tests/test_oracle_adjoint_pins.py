"""Pins for the oracle's adjoint recurrence (vto_adjoint_ex_*: the backward
leg of adjoint-state FWI) against the pinned forward scheme and plain linear algebra.

* One adjoint step equals psi^{m-1} = g (2 psi^m - g psi^{m+1} + dt^2 A^T psi^m) with A^T the
  numpy TRANSPOSE of the dense 2N x 2N operator assembled point by point from Eqs. 1-2, 4-5
  (the same builder that pins the forward step, tests/test_oracle_pins.py), fp64, 1e-12.
* <A x, y> = <x, A^T y> through the steppers themselves (W = 0, u^{n-1} = 2u^n isolates dt^2 A).
* The discrete dot-product identity of the whole damped K-step propagation,
  <M^K X, Y> = <X, (M^T)^K Y>, with X = (u^0, u^{-1}) stepped by the pinned forward oracle and
  Y = (psi^K / g, -g psi^{K+1}) stepped back by the adjoint oracle.
* Injection in the adjoint: the step-1 closed form g (dt^2 trace) from the zero state.
"""
import numpy as np

import oracle
from test_oracle_pins import _brute_setup, _dense_operator


def _g(c):
    d = lambda i, n: oracle.lib().vto_damping(i, n, c["damp_width"], c["damp_alpha"])
    nx, ny, nz = c["nx"], c["ny"], c["nz"]
    gx = np.array([d(i, nx) for i in range(nx)])
    gy = np.array([d(j, ny) for j in range(ny)])
    gz = np.array([d(k, nz) for k in range(nz)])
    return (gx[None, None, :] * gy[None, :, None]) * gz[:, None, None]


def test_adjoint_step_is_the_dense_transpose():
    c, wxy, wz, vx2, vn2, vz2 = _brute_setup()
    dt = 4e-4
    P = oracle.params(c, dt, src=None)
    shape = vx2.shape
    rng = np.random.default_rng(3)
    st = [rng.normal(size=shape) for _ in range(4)]
    m64 = [a.astype(np.float64) for a in (vx2, vn2, vz2)]
    got = oracle.adjoint_ex(P, wxy, wz, *m64, st, m0=5, nsteps=1, dtype=np.float64)[:2]
    AT = _dense_operator(c, wxy, wz, *m64).T
    g = np.concatenate([_g(c).reshape(-1)] * 2)
    psi_m = np.concatenate([st[0].reshape(-1), st[1].reshape(-1)])
    psi_m1 = np.concatenate([st[2].reshape(-1), st[3].reshape(-1)])
    dt2 = P.dt * P.dt
    want = g * (2 * psi_m - g * psi_m1 + dt2 * (AT @ psi_m))
    N = psi_m.size // 2
    for f in range(2):
        w = want[f * N:(f + 1) * N].reshape(shape)
        assert np.linalg.norm(got[f] - w) <= 1e-12 * np.linalg.norm(w)


def test_dot_product_through_the_steppers():
    """W = 0, dt = 1: a forward step from (x, 2x) is A x, an adjoint step from (y, 2y) is A^T y."""
    c, wxy, wz, vx2, vn2, vz2 = _brute_setup()
    c = dict(c, damp_width=0)
    P = oracle.params(c, 1.0, src=None)
    m64 = [a.astype(np.float64) for a in (vx2, vn2, vz2)]
    rng = np.random.default_rng(5)
    x = [rng.normal(size=vx2.shape) for _ in range(2)]
    y = [rng.normal(size=vx2.shape) for _ in range(2)]
    Ax = oracle.run(P, wxy, wz, *m64, (x[0], x[1], 2 * x[0], 2 * x[1]), nsteps=1, dtype=np.float64)[:2]
    ATy = oracle.adjoint_ex(P, wxy, wz, *m64, (y[0], y[1], 2 * y[0], 2 * y[1]), nsteps=1, dtype=np.float64)[:2]
    lhs = sum(np.vdot(a, b) for a, b in zip(Ax, y))
    rhs = sum(np.vdot(a, b) for a, b in zip(x, ATy))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)
    assert abs(lhs) > 1.0


def test_damped_k_step_dot_product_identity():
    c, wxy, wz, vx2, vn2, vz2 = _brute_setup()
    dt, K = 4e-4, 12
    P = oracle.params(c, dt, src=None)
    m64 = [a.astype(np.float64) for a in (vx2, vn2, vz2)]
    g = _g(c)
    assert g.min() < 1.0   # the band really damps
    rng = np.random.default_rng(9)
    X0 = [rng.normal(size=vx2.shape) for _ in range(4)]            # u^0 (p, q), u^-1 (p, q)
    XK = oracle.run(P, wxy, wz, *m64, X0, nsteps=K, dtype=np.float64)[:4]
    psiK = [rng.normal(size=vx2.shape) for _ in range(4)]          # psi^K (p, q), psi^{K+1} (p, q)
    psi0 = oracle.adjoint_ex(P, wxy, wz, *m64, psiK, m0=K, nsteps=K, dtype=np.float64)[:4]
    dot = lambda u, v: sum(np.vdot(a, b) for a, b in zip(u, v))
    lhs = dot(XK[:2], [a / g for a in psiK[:2]]) - dot(XK[2:], [g * a for a in psiK[2:]])
    rhs = dot(X0[:2], [a / g for a in psi0[:2]]) - dot(X0[2:], [g * a for a in psi0[2:]])
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), abs(rhs))
    # the forward oracle's own transpose would not be its time reversal: a wrong-sided
    # damping (g (2 + dt^2 A^T) instead of (2 + dt^2 A^T) g) breaks the identity
    assert abs(lhs) > 1.0


def test_adjoint_injection_closed_form():
    c, wxy, wz, vx2, vn2, vz2 = _brute_setup()
    P = oracle.params(c, 4e-4, src=None)
    z = [np.zeros(vx2.shape) for _ in range(4)]
    pts = [(0, 0, 0), (4, 3, 3), (8, 7, 6)]
    tr = np.array([[1.5, -2.0, 0.25]] * 3)
    p, q = oracle.adjoint_ex(P, wxy, wz, vx2, vn2, vz2, z, m0=7, nsteps=1, inj=(pts, 3, 5, tr),
                             dtype=np.float64)[:2]
    g = _g(c)
    want = np.zeros(vx2.shape)
    for (i, j, k), v in zip(pts, tr[2]):   # time index 7 = row 7 - 5
        want[k, j, i] = g[k, j, i] * (P.dt * P.dt * v)
    assert np.array_equal(p, want) and np.array_equal(q, want)
