"""Pins for the oracle's single-point evaluator (vto_point_*) and its plane-window stepper
(vto_step_planes_*) against the pinned full-grid stepper vto_run_* (tests/test_oracle_pins.py
ties that one to polynomial exactness, closed forms, symmetry and a dense-operator brute force).

Both are the checkers of GPU tests on grids too large for vto_run (C4: 2048^2 x 1024), so a
wrong damping axis, source bit, s(t^n) time index, w^z row or zero-exterior edge in their own
preambles must fail here, without any CUDA path involved. Every point of a ragged grid (all six
faces, the damping band, the eight corners, the source point) is compared bitwise, in fp32 and
fp64, at the default and the paper's radii (R_xy = 12, R_z = 8), from a
random state at a time index n0 > 0 (so s(t^{n0}) != s(0)).
"""
import numpy as np
import pytest

import oracle
from synth import weights as W

SHAPE = (23, 29, 37)   # (nz, ny, nx): ragged in every axis


def _setup(r, dtype, seed=5):
    nz, ny, nx = SHAPE
    rng = np.random.default_rng(seed)
    cfg = dict(nx=nx, ny=ny, nz=nz, r_xy=r[0], r_z=r[1], h=10.0, damp_width=5, damp_alpha=0.015,
               src=(17, 11, 9), f=15.0, t0=0.02, amp=1.0, mask=3)
    P = oracle.params(cfg, dt=1.1e-3)
    wxy = W.xy_weights(r[0]).astype(dtype)
    wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(nz, r[1], 5.0, 15.0), r[1]).astype(dtype))
    state = [rng.uniform(-1, 1, SHAPE).astype(dtype) for _ in range(4)]
    vz2 = rng.uniform(2e6, 9e6, SHAPE).astype(dtype)
    vx2 = (vz2 * rng.uniform(1.0, 1.5, SHAPE)).astype(dtype)
    vn2 = (vz2 * rng.uniform(1.0, 1.2, SHAPE)).astype(dtype)
    return P, wxy, wz, state, (vx2, vn2, vz2)


CASES = [((4, 4), np.float32), ((4, 4), np.float64), ((12, 8), np.float32), ((12, 8), np.float64)]


@pytest.mark.parametrize("r,dtype", CASES)
def test_point_equals_run_at_every_point(r, dtype):
    n0 = 7
    P, wxy, wz, state, model = _setup(r, dtype)
    pn, qn = oracle.run(P, wxy, wz, *model, state, n0=n0, nsteps=1, dtype=dtype)[:2]
    R, Rz = r
    nz, ny, nx = SHAPE
    p, q, pm, qm = state
    pp = np.pad(p, ((0, 0), (R, R), (R, R)))      # zero exterior in x, y
    qp = np.pad(q, ((Rz, Rz), (0, 0), (0, 0)))    # zero exterior in z
    bad = 0
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                a, b = j + R, i + R
                pc = np.concatenate([[pp[k, a, b]], pp[k, a, b + 1:b + R + 1],
                                     pp[k, a, b - R:b][::-1], pp[k, a + 1:a + R + 1, b],
                                     pp[k, a - R:a, b][::-1]])
                qc = qp[k:k + 2 * Rz + 1, j, i]
                po, qo = oracle.point(P, wxy, wz[k], i, j, k, n0, pc, qc, pm[k, j, i], qm[k, j, i],
                                      model[0][k, j, i], model[1][k, j, i], model[2][k, j, i], dtype=dtype)
                bad += (po != pn[k, j, i]) + (qo != qn[k, j, i])
    assert bad == 0, f"{bad} mismatches of vto_point vs vto_run"
    # the source point really injected something (mask 3 adds s(t^{n0}) to both F_p and F_q)
    s = dtype(oracle.ricker(n0 * P.dt, P.src_f, P.src_t0))
    assert s != 0


@pytest.mark.parametrize("r,dtype", CASES)
def test_step_planes_equals_run(r, dtype):
    n0 = 4
    P, wxy, wz, state, model = _setup(r, dtype, seed=9)
    pn, qn = oracle.run(P, wxy, wz, *model, state, n0=n0, nsteps=1, dtype=dtype)[:2]
    R, Rz = r
    nz = SHAPE[0]
    p, q, pm, qm = state
    qpad = np.pad(q, ((Rz, Rz), (0, 0), (0, 0)), constant_values=np.nan)   # never read
    windows = [(0, 1), (0, nz), (1, 3), (Rz, 2), (9, 1), (nz - Rz - 1, Rz + 1), (nz - 1, 1), (5, 0)]
    for k0, nk in windows:
        sl = slice(k0, k0 + nk)
        got = oracle.step_planes(P, wxy, wz, k0, p[sl], qpad[k0:k0 + nk + 2 * Rz], pm[sl], qm[sl],
                                 model[0][sl], model[1][sl], model[2][sl], n=n0, dtype=dtype)
        assert np.array_equal(got[0], pn[sl]), (k0, nk)
        assert np.array_equal(got[1], qn[sl]), (k0, nk)


def test_step_planes_rejects_bad_window():
    P, wxy, wz, state, model = _setup((4, 4), np.float32)
    nz = SHAPE[0]
    z = np.zeros((2,) + SHAPE[1:], np.float32)
    with pytest.raises(ValueError):
        oracle.step_planes(P, wxy, wz, nz - 1, z, np.zeros((10,) + SHAPE[1:], np.float32), z, z, z, z, z)
