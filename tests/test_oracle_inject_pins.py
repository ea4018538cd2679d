"""Pins for the oracle's N4 extensions (vto_run_ex_*: time direction, multi-point trace
injection, receivers) against things other than themselves -- SURVEY.md 8(f) N4, the RTM/FWI
use of the propagator.

* Injection reduces to the pinned point source: a trace equal to the Ricker samples
  s(t^n) (rounded once) injected at one point is bitwise the Eq. 1 source run.
* Superposition (the scheme is linear in its forcing, Eqs. 1-3): n-point injection equals the
  sum of n single-point runs, fp64, within 1e-12 relative.
* Step-1 closed form from the zero state: u^1(x_r) = g_r * (dt^2 * trace[0][r]), 0 elsewhere.
* Receivers record exactly the fields the plain stepper leaves at those points, step by step.
* Time reversal (SPEC.md "Time-reversal symmetry", no damping): K forward steps with
  injection, then K-1 steps of the reversed recurrence from the swapped levels, return u^0.
"""
import numpy as np
import pytest

import oracle
from synth import weights as W

SHAPE = (13, 15, 17)   # (nz, ny, nx)


def _setup(dtype, damp=3, r=(4, 4), seed=1):
    nz, ny, nx = SHAPE
    rng = np.random.default_rng(seed)
    cfg = dict(nx=nx, ny=ny, nz=nz, r_xy=r[0], r_z=r[1], h=10.0, damp_width=damp, damp_alpha=0.015,
               src=None, f=15.0, t0=0.03, amp=1.0, mask=1)
    dt = 1.0e-3
    wxy = W.xy_weights(r[0]).astype(dtype)
    wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(nz, r[1], 6.0, 12.0), r[1]).astype(dtype))
    vz2 = rng.uniform(2e6, 9e6, SHAPE).astype(dtype)
    vx2 = (vz2 * rng.uniform(1.0, 1.5, SHAPE)).astype(dtype)
    vn2 = (vz2 * rng.uniform(1.0, 1.2, SHAPE)).astype(dtype)
    return cfg, dt, wxy, wz, (vx2, vn2, vz2)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("mask", [1, 2, 3])
def test_ricker_trace_injection_equals_point_source(dtype, mask):
    cfg, dt, wxy, wz, model = _setup(dtype)
    src, nsteps = (8, 7, 6), 30
    P_src = oracle.params(dict(cfg, mask=mask), dt, src=src)
    ref = oracle.run(P_src, wxy, wz, *model, None, nsteps=nsteps, dtype=dtype)[:4]
    P0 = oracle.params(cfg, dt, src=None)
    tr = np.array([[dtype(cfg["amp"] * oracle.ricker(n * P0.dt, cfg["f"], cfg["t0"]))] for n in range(nsteps)])
    got = oracle.run_ex(P0, wxy, wz, *model, None, nsteps=nsteps, inj=([src], mask, 0, tr), dtype=dtype)[:4]
    for a, b in zip(got, ref):
        assert np.abs(b).max() > 0
        assert np.array_equal(a, b)


def test_superposition_fp64():
    dtype = np.float64
    cfg, dt, wxy, wz, model = _setup(dtype)
    P = oracle.params(cfg, dt, src=None)
    pts = [(3, 4, 5), (12, 9, 2), (8, 7, 10)]
    rng = np.random.default_rng(4)
    nsteps, t_first = 25, 2
    tr = rng.normal(size=(20, 3))
    full = oracle.run_ex(P, wxy, wz, *model, None, nsteps=nsteps, inj=(pts, 3, t_first, tr), dtype=dtype)[:4]
    parts = [oracle.run_ex(P, wxy, wz, *model, None, nsteps=nsteps,
                           inj=([pts[r]], 3, t_first, tr[:, r:r + 1]), dtype=dtype)[:4] for r in range(3)]
    for f in range(4):
        s = parts[0][f] + parts[1][f] + parts[2][f]
        assert np.linalg.norm(full[f] - s) <= 1e-12 * np.linalg.norm(full[f])
        assert np.abs(full[f]).max() > 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_step1_closed_form(dtype):
    cfg, dt, wxy, wz, model = _setup(dtype, damp=3)
    P = oracle.params(cfg, dt, src=None)
    pts = [(0, 0, 0), (16, 14, 12), (8, 7, 6), (1, 13, 2)]   # corners (damped) and the centre
    tr = np.array([[1.5, -2.25, 0.75, 3.0]], dtype)
    p, q = oracle.run_ex(P, wxy, wz, *model, None, nsteps=1, inj=(pts, 3, 0, tr), dtype=dtype)[:2]
    g = [oracle.damping_profile(n, cfg["damp_width"], cfg["damp_alpha"]).astype(dtype) if dtype == np.float32
         else np.array([oracle.lib().vto_damping(i, n, cfg["damp_width"], cfg["damp_alpha"]) for i in range(n)])
         for n in (SHAPE[2], SHAPE[1], SHAPE[0])]
    dt2 = dtype(P.dt * P.dt)
    expect = np.zeros(SHAPE, dtype)
    for (i, j, k), v in zip(pts, tr[0]):
        gg = (g[0][i] * g[1][j]) * g[2][k]
        expect[k, j, i] = gg * (dt2 * v)
    assert np.array_equal(p, expect) and np.array_equal(q, expect)


def test_receivers_record_the_stepped_fields():
    dtype = np.float32
    cfg, dt, wxy, wz, model = _setup(dtype)
    P = oracle.params(dict(cfg, mask=1), dt, src=(8, 7, 6))
    rec = [(8, 7, 6), (0, 0, 0), (16, 14, 12), (9, 7, 6), (8, 7, 9)]
    nsteps = 12
    _, _, _, _, traces, _ = oracle.run_ex(P, wxy, wz, *model, None, nsteps=nsteps, rec=(rec, 3), dtype=dtype)
    st = None
    for n in range(nsteps):
        st = oracle.run(P, wxy, wz, *model, st, n0=n, nsteps=1, dtype=dtype)[:4]
        for r, (i, j, k) in enumerate(rec):
            assert traces[n, r, 0] == st[0][k, j, i] and traces[n, r, 1] == st[1][k, j, i]
    assert np.abs(traces).max() > 0


def test_time_reversal_with_injection_returns_initial_state():
    dtype = np.float64
    cfg, dt, wxy, wz, model = _setup(dtype, damp=0)
    P = oracle.params(cfg, dt, src=None)
    rng = np.random.default_rng(8)
    st0 = [rng.normal(size=SHAPE) for _ in range(4)]
    K = 16
    pts = [(4, 4, 4), (10, 11, 7)]
    tr = 1e3 * rng.normal(size=(K, 2))   # dt^2 * 1e3 ~ 1e-3: well above the fp64 reversal error
    p, q, pm, qm = oracle.run_ex(P, wxy, wz, *model, st0, nsteps=K, inj=(pts, 1, 0, tr), dtype=dtype)[:4]
    # reversed recurrence from (u^{K-1}, u^K): K-1 steps back to u^0 (the stored level is u^1)
    b = oracle.run_ex(P, wxy, wz, *model, (pm, qm, p, q), n0=K - 1, nsteps=K - 1, direction=-1,
                      inj=(pts, 1, 0, tr), dtype=dtype)[:4]
    for got, want in ((b[0], st0[0]), (b[1], st0[1])):
        assert np.linalg.norm(got - want) <= 1e-9 * np.linalg.norm(want)
    # and the reversal really used the time-indexed samples: dropping them breaks it
    c = oracle.run_ex(P, wxy, wz, *model, (pm, qm, p, q), n0=K - 1, nsteps=K - 1, direction=-1, dtype=dtype)[:4]
    assert np.linalg.norm(c[0] - st0[0]) > 1e-5 * np.linalg.norm(st0[0])


def test_run_ex_rejects_bad_points():
    cfg, dt, wxy, wz, model = _setup(np.float32)
    P = oracle.params(cfg, dt, src=None)
    tr = np.ones((2, 2), np.float32)
    with pytest.raises(ValueError):
        oracle.run_ex(P, wxy, wz, *model, None, inj=([(1, 1, 1), (1, 1, 1)], 1, 0, tr))   # duplicate
    with pytest.raises(ValueError):
        oracle.run_ex(P, wxy, wz, *model, None, inj=([(1, 1, 1), (17, 1, 1)], 1, 0, tr))  # outside
    with pytest.raises(ValueError):
        oracle.run_ex(P, wxy, wz, *model, None, rec=([(1, 1, 13)], 1))
