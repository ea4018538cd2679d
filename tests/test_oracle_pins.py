"""Pins for the CPU oracle (oracle/vti_oracle.c) against things other than itself.

Each test ties one part of the oracle to the paper or to mathematics:
  * operators (Eq. 4, Eq. 5): exact derivatives of polynomials, through the
    oracle's own step function, in fp64;
  * couplings (Eqs. 1-2): early-step closed forms from a point source
    (F_q uses L(p) and vn2; F_p uses vx2; the z term uses vz2 and w^z[k][m]
    with the paper's orientation l = m - Rz);
  * isotropic limit (P:41-43 with eps = delta = 0): p == q bitwise with dual
    injection, and p equals an independent numpy acoustic solver;
  * symmetry: x -> -x, y -> -y, x <-> y bitwise for a centred source;
  * brute force: a dense 2N x 2N operator assembled from the definitions on an
    8^3 grid, stepped in numpy;
  * Ricker and Cerjan (reading c9) closed forms;
  * determinism across thread counts; fp32 vs fp64 drift bound.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from synth import weights as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def cfg_small(n=(12, 12, 12), r=(2, 2), damp=0, src=None, mask=1, t0=0.0, h=10.0):
    return dict(nx=n[0], ny=n[1], nz=n[2], r_xy=r[0], r_z=r[1], h=h, damp_width=damp,
                damp_alpha=0.015, src=src, f=15.0, t0=t0, amp=1.0, mask=mask)


def const_model(shape, vx2, vn2, vz2, dtype=np.float64):
    return tuple(np.full(shape, v, dtype=dtype) for v in (vx2, vn2, vz2))


# ----------------------------------------------------------------------------- operators

@pytest.mark.parametrize("r", [1, 2, 4])
def test_xy_laplacian_of_polynomials_through_step(r):
    """One step with dt=1, g=1, p^{n-1}=2p^n, q=0: p^{n+1} = vx2 L(p), q^{n+1} = vn2 L(p)."""
    n = 4 * r + 6
    c = cfg_small((n, n, 3), (r, 1))
    P = oracle.params(c, dt=1.0, src=None)
    h = c["h"]
    wxy = W.xy_weights(r)  # fp64 weights
    wz = np.zeros((3, 3))
    shape = (3, n, n)
    vx2, vn2, vz2 = const_model(shape, 2.0, 3.0, 0.0)
    x = (np.arange(n) - n / 2 + 0.25) * h
    X, Y = np.meshgrid(x, x, indexing="xy")  # [y][x]
    for dx, dy in [(0, 0), (1, 0), (2, 0), (0, 2), (2, 2), (2 * r, 0), (r, r)]:
        if dx + dy > 2 * r:
            continue
        p2d = X ** dx * Y ** dy
        lap = (dx * (dx - 1) * X ** max(dx - 2, 0) * Y ** dy if dx >= 2 else 0) + \
              (dy * (dy - 1) * Y ** max(dy - 2, 0) * X ** dx if dy >= 2 else 0)
        lap = np.broadcast_to(lap, (n, n))
        p = np.broadcast_to(p2d, shape).copy()
        zero = np.zeros(shape)
        pn, qn, _, _, _ = oracle.run(P, wxy, wz, vx2, vn2, vz2, (p, zero, 2 * p, zero),
                                     nsteps=1, dtype=np.float64)
        inner = (slice(None), slice(r, n - r), slice(r, n - r))
        scale = max(1.0, np.abs(p2d).max() / h ** 2)
        np.testing.assert_allclose(pn[inner], 2.0 * lap[None][(slice(None),) + inner[1:]] * np.ones(shape)[inner],
                                   rtol=1e-10, atol=1e-11 * scale)
        np.testing.assert_allclose(qn[inner], 3.0 * np.broadcast_to(lap, shape)[inner],
                                   rtol=1e-10, atol=1e-11 * scale)


@pytest.mark.parametrize("rz", [1, 2, 4])
def test_z_derivative_of_polynomials_through_step(rz):
    """vx2=vn2=0, vz2=1, u^{n-1}=2u^n: p^{n+1} = q^{n+1} = D(q) on nonuniform nodes."""
    nz = 4 * rz + 6
    c = cfg_small((4, 4, nz), (1, rz))
    P = oracle.params(c, dt=1.0, src=None)
    zc = W.z_coords_ramp(nz, rz, 5.0, 15.0)
    wz = W.z_weights(zc, rz)
    z = zc[rz:rz + nz] - zc[rz + nz // 2] + 0.5
    shape = (nz, 4, 4)
    vx2, vn2, vz2 = const_model(shape, 0.0, 0.0, 1.0)
    for m in range(0, 2 * rz + 1):
        q = np.broadcast_to((z ** m)[:, None, None], shape).copy()
        d2 = (m * (m - 1) * z ** (m - 2) if m >= 2 else 0 * z)
        p = np.zeros(shape)
        pn, qn, _, _, _ = oracle.run(P, W.xy_weights(1), wz, vx2, vn2, vz2, (p, q, p, 2 * q),
                                     nsteps=1, dtype=np.float64)
        ks = slice(rz, nz - rz)
        want = np.broadcast_to(d2[:, None, None], shape)[ks]
        scale = np.abs(q).max() / 25.0
        np.testing.assert_allclose(qn[ks], want, rtol=1e-9, atol=1e-11 * max(scale, 1))
        np.testing.assert_allclose(pn[ks], want, rtol=1e-9, atol=1e-11 * max(scale, 1))


def test_zero_exterior_at_edge_point():
    """At the first interior column, the x-neighbours beyond the edge count as 0."""
    c = cfg_small((8, 8, 3), (2, 1))
    P = oracle.params(c, dt=1.0, src=None)
    shape = (3, 8, 8)
    p = np.ones(shape)
    zero = np.zeros(shape)
    vx2, vn2, vz2 = const_model(shape, 1.0, 1.0, 0.0)
    wxy = np.array([-5.0, 4 / 3, -1 / 12])
    pn, _, _, _, _ = oracle.run(P, wxy, np.zeros((3, 3)), vx2, vn2, vz2, (p, zero, 2 * p, zero),
                                nsteps=1, dtype=np.float64)
    h2 = 100.0
    # corner (0,0): missing 2 neighbours on -x (l=1,2) and 2 on -y
    assert pn[1, 0, 0] == pytest.approx(-2 * (4 / 3 - 1 / 12) / h2, rel=1e-14)
    # interior: constant -> 0
    assert abs(pn[1, 4, 4]) < 1e-15


# ----------------------------------------------------------------------------- couplings

def _point_source_cfg(nonuniform=True):
    c = cfg_small((13, 13, 13), (3, 2), src=(6, 6, 6), mask=1, t0=0.02)
    zc = W.z_coords_ramp(13, 2, 5.0, 15.0) if nonuniform else np.arange(17) * 10.0
    return c, W.xy_weights(3), W.z_weights(zc, 2)


def test_early_steps_closed_forms():
    c, wxy, wz = _point_source_cfg()
    dt = 1e-3
    P = oracle.params(c, dt=dt)
    shape = (13, 13, 13)
    vx2, vn2, vz2 = 5.0e6, 4.0e6, 3.0e6
    model = const_model(shape, vx2, vn2, vz2)
    cxy = wxy / c["h"] ** 2
    f, t0 = 15.0, 0.02
    s = lambda n: (1 - 2 * (math.pi * f * (n * dt - t0)) ** 2) * math.exp(-(math.pi * f * (n * dt - t0)) ** 2)
    st = None
    out = []
    for n in range(3):
        st = oracle.run(P, wxy, wz, *model, st, n0=n, nsteps=1, dtype=np.float64)[:4]
        out.append([a.copy() for a in st])
    (p1, q1, _, _), (p2, q2, _, _), (p3, q3, _, _) = out
    i0 = j0 = k0 = 6
    # step 1: p^1 = dt^2 s_0 at the source only; q^1 == 0 (source enters F_p only, Eq. 1)
    assert p1[k0, j0, i0] == pytest.approx(dt * dt * s(0), rel=1e-14)
    assert np.count_nonzero(p1) == 1 and np.count_nonzero(q1) == 0
    a = p1[k0, j0, i0]
    for l in range(1, 4):
        for (dj, di) in [(0, l), (0, -l), (l, 0), (-l, 0)]:
            # step 2: F_q = vn2 L(p^1) -> q^2 = dt^2 vn2 cxy_l p^1(src)  (Eq. 2 uses L(p))
            assert q2[k0, j0 + dj, i0 + di] == pytest.approx(dt * dt * vn2 * cxy[l] * a, rel=1e-13)
            assert p2[k0, j0 + dj, i0 + di] == pytest.approx(dt * dt * vx2 * cxy[l] * a, rel=1e-13)
    assert p2[k0, j0, i0] == pytest.approx(2 * a + dt * dt * (vx2 * cxy[0] * a + s(1)), rel=1e-13)
    assert q2[k0, j0, i0] == pytest.approx(dt * dt * vn2 * cxy[0] * a, rel=1e-13)
    assert np.count_nonzero(p2[:k0]) == 0 and np.count_nonzero(q2[k0 + 1:]) == 0
    # step 3: off-plane points see only vz2 * w^z[k][m] q^2 (Eq. 5, l = m - Rz)
    for l in (1, 2, 3):
        for m in (-2, -1, 1, 2):
            k = k0 + m
            want = dt * dt * vz2 * wz[k, 2 - m] * q2[k0, j0, i0 + l]
            assert p3[k, j0, i0 + l] == pytest.approx(want, rel=1e-13)
            assert q3[k, j0, i0 + l] == pytest.approx(want, rel=1e-13)


def test_source_mask_q_only():
    c, wxy, wz = _point_source_cfg()
    c["mask"] = 2
    P = oracle.params(c, dt=1e-3)
    model = const_model((13, 13, 13), 5e6, 4e6, 3e6)
    p1, q1, _, _, _ = oracle.run(P, wxy, wz, *model, None, nsteps=1, dtype=np.float64)
    assert np.count_nonzero(p1) == 0 and np.count_nonzero(q1) == 1


# ----------------------------------------------------------------------------- isotropic

def _iso_setup(n=17, r=(2, 2), damp=4, mask=3):
    c = cfg_small((n, n, n), r, damp=damp, src=(n // 2, n // 2 - 1, n // 2 + 1), mask=mask, t0=0.05)
    zc = W.z_coords_ramp(n, r[1], 6.0, 14.0)
    wxy = W.xy_weights(r[0]).astype(np.float32)
    wz = W.z_weights(zc, r[1]).astype(np.float32)
    rng = np.random.default_rng(3)
    vz2 = rng.uniform(2e6, 9e6, size=(n, n, n)).astype(np.float32)
    return c, wxy, wz, vz2


def test_isotropic_dual_injection_p_equals_q_bitwise():
    c, wxy, wz, vz2 = _iso_setup(mask=3)
    P = oracle.params(c, dt=6e-4)
    p, q, pm, qm, _ = oracle.run(P, wxy, wz, vz2, vz2, vz2, None, nsteps=60)
    assert np.abs(p).max() > 0
    assert np.array_equal(p, q) and np.array_equal(pm, qm)


def test_isotropic_p_only_injection_differs_only_at_source():
    c, wxy, wz, vz2 = _iso_setup(mask=1)
    P = oracle.params(c, dt=6e-4)
    p, q, _, _, _ = oracle.run(P, wxy, wz, vz2, vz2, vz2, None, nsteps=60)
    diff = np.argwhere(p != q)
    assert len(diff) == 1 and tuple(diff[0]) == (c["src"][2], c["src"][1], c["src"][0])


def _acoustic_numpy(c, wxy, wz, v2, dt, nsteps):
    """Independent fp64 acoustic solver u_tt = v2 (u_xx + u_yy + u_zz) + s delta, slicing-based."""
    nx, ny, nz, R, Rz = c["nx"], c["ny"], c["nz"], c["r_xy"], c["r_z"]
    pad = lambda a: np.pad(a, ((Rz, Rz), (R, R), (R, R)))
    u = np.zeros((nz, ny, nx))
    um = np.zeros_like(u)
    g1 = lambda n: np.array([math.exp(-(c["damp_alpha"] * (c["damp_width"] - min(i, n - 1 - i))) ** 2)
                             if min(i, n - 1 - i) < c["damp_width"] else 1.0 for i in range(n)])
    g = g1(nz)[:, None, None] * g1(ny)[None, :, None] * g1(nx)[None, None, :]
    si, sj, sk = c["src"]
    for n in range(nsteps):
        U = pad(u)
        lap = wxy[0] * u
        for l in range(1, R + 1):
            lap = lap + wxy[l] * (U[Rz:Rz + nz, R:R + ny, R + l:R + l + nx] + U[Rz:Rz + nz, R:R + ny, R - l:R - l + nx]
                                  + U[Rz:Rz + nz, R + l:R + l + ny, R:R + nx] + U[Rz:Rz + nz, R - l:R - l + ny, R:R + nx])
        lap = lap / c["h"] ** 2
        dzz = np.zeros_like(u)
        for m in range(2 * Rz + 1):
            dzz = dzz + wz[:, m][:, None, None] * U[m:m + nz, R:R + ny, R:R + nx]
        F = v2 * (lap + dzz)
        tau = n * dt - c["t0"]
        F[sk, sj, si] += c["amp"] * (1 - 2 * (math.pi * c["f"] * tau) ** 2) * math.exp(-(math.pi * c["f"] * tau) ** 2)
        un = g * (2 * u - g * um + dt * dt * F)
        um, u = u, un
    return u


def test_isotropic_matches_independent_acoustic_solver():
    c, wxy, wz, vz2 = _iso_setup(mask=3)
    dt = float(np.float32(6e-4))
    P = oracle.params(c, dt=dt)
    v = vz2.astype(np.float64)
    p, q, _, _, _ = oracle.run(P, wxy.astype(np.float64), wz.astype(np.float64), v, v, v, None,
                               nsteps=40, dtype=np.float64)
    u = _acoustic_numpy(c, wxy.astype(np.float64), wz.astype(np.float64), v, dt, 40)
    assert np.abs(u).max() > 0
    np.testing.assert_allclose(p, u, rtol=0, atol=1e-11 * np.abs(u).max())


# ----------------------------------------------------------------------------- symmetry

def test_mirror_symmetry_centred_source():
    n = 21
    c = cfg_small((n, n, n), (4, 4), damp=5, src=(10, 10, 10), t0=0.04)
    wxy = W.xy_weights(4).astype(np.float32)
    wz = W.z_weights(np.arange(n + 8) * 10.0, 4).astype(np.float32)
    model = const_model((n, n, n), 1.26e7, 1.08e7, 9e6, np.float32)
    P = oracle.params(c, dt=1.2e-3)
    p, q, _, _, _ = oracle.run(P, wxy, wz, *model, None, nsteps=50)
    assert np.abs(p).max() > 0
    for f in (p, q):
        assert np.array_equal(f, f[:, :, ::-1])              # x -> -x
        assert np.array_equal(f, f[:, ::-1, :])              # y -> -y
        assert np.array_equal(f, f.transpose(0, 2, 1))       # x <-> y
        zf = f[::-1]
        assert np.linalg.norm(zf - f) <= 1e-5 * np.linalg.norm(f)  # z mirror: not bitwise


# ----------------------------------------------------------------------------- brute force

def _dense_operator(c, wxy, wz, vx2, vn2, vz2):
    """Dense 2N x 2N operator [[vx2 L, vz2 D], [vn2 L, vz2 D]] built point by point."""
    nx, ny, nz, R, Rz = c["nx"], c["ny"], c["nz"], c["r_xy"], c["r_z"]
    N = nx * ny * nz
    idx = lambda i, j, k: (k * ny + j) * nx + i
    Lm = np.zeros((N, N))
    Dm = np.zeros((N, N))
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                a = idx(i, j, k)
                Lm[a, a] += wxy[0] / c["h"] ** 2
                for l in range(1, R + 1):
                    for (ii, jj) in [(i + l, j), (i - l, j), (i, j + l), (i, j - l)]:
                        if 0 <= ii < nx and 0 <= jj < ny:
                            Lm[a, idx(ii, jj, k)] += wxy[l] / c["h"] ** 2
                for m in range(2 * Rz + 1):
                    kk = k - Rz + m
                    if 0 <= kk < nz:
                        Dm[a, idx(i, j, kk)] += wz[k, m]
    A = np.block([[vx2.reshape(-1)[:, None] * Lm, vz2.reshape(-1)[:, None] * Dm],
                  [vn2.reshape(-1)[:, None] * Lm, vz2.reshape(-1)[:, None] * Dm]])
    return A


def _brute_setup(shape=(7, 8, 9)):
    nz, ny, nx = shape
    c = cfg_small((nx, ny, nz), (2, 2), damp=2, src=(3, 4, 3), mask=1, t0=0.01)
    zc = W.z_coords_ramp(nz, 2, 6.0, 12.0)
    wxy = W.xy_weights(2).astype(np.float32).astype(np.float64)
    wz = W.z_weights(zc, 2).astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(11)
    vz2 = rng.uniform(2e6, 6e6, shape).astype(np.float32)
    eps = rng.uniform(0.05, 0.25, shape)
    dl = eps * rng.uniform(0, 1, shape)
    vx2 = (vz2 * (1 + 2 * eps)).astype(np.float32)
    vn2 = (vz2 * (1 + 2 * dl)).astype(np.float32)
    return c, wxy, wz, vx2, vn2, vz2


def test_brute_force_dense_operator_8cubed():
    """~8^3 grid (9 x 8 x 7, all extents distinct so axis mix-ups show)."""
    c, wxy, wz, vx2, vn2, vz2 = _brute_setup()
    nz, ny, nx = vz2.shape
    N = vz2.size
    A = _dense_operator(c, wxy, wz, vx2.astype(np.float64), vn2.astype(np.float64), vz2.astype(np.float64))
    rho = np.abs(np.linalg.eigvals(A)).max()
    dt = float(np.float32(0.8 * 2 / math.sqrt(rho)))
    g1 = lambda n: np.array([oracle.lib().vto_damping(i, n, 2, 0.015) for i in range(n)])
    g = (g1(nx)[None, None, :] * g1(ny)[None, :, None] * g1(nz)[:, None, None]).reshape(-1)
    G = np.concatenate([g, g])
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, 2 * N)
    um = rng.uniform(-1, 1, 2 * N)
    state = [a.reshape(nz, ny, nx) for a in (u[:N], u[N:], um[:N], um[N:])]
    st = [a.copy() for a in state]
    si = (c["src"][2] * ny + c["src"][1]) * nx + c["src"][0]
    for step in range(50):
        F = A @ u
        tau = step * dt - c["t0"]
        F[si] += (1 - 2 * (math.pi * 15 * tau) ** 2) * math.exp(-(math.pi * 15 * tau) ** 2)
        u, um = G * (2 * u - G * um + dt * dt * F), u
    P = oracle.params(c, dt=dt)
    p, q, pm, qm, _ = oracle.run(P, wxy, wz, vx2.astype(np.float64), vn2.astype(np.float64),
                                 vz2.astype(np.float64), st, nsteps=50, dtype=np.float64)
    ref = np.concatenate([u[:N], u[N:]])
    got = np.concatenate([p.reshape(-1), q.reshape(-1)])
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    np.testing.assert_allclose(np.concatenate([pm.reshape(-1), qm.reshape(-1)]), um, rtol=0,
                               atol=1e-12 * np.abs(um).max())
    # fp32 canonical mode on the same inputs stays within the parity gate
    p32, q32, _, _, _ = oracle.run(P, wxy.astype(np.float32), wz.astype(np.float32), vx2, vn2, vz2,
                                   [a.astype(np.float32) for a in st], nsteps=50)
    got32 = np.concatenate([p32.reshape(-1), q32.reshape(-1)]).astype(np.float64)
    assert np.linalg.norm(got32 - ref) <= 1e-5 * np.linalg.norm(ref)


def test_dense_operator_stability_and_eps_delta_sign():
    """eps >= delta: spectrum real and <= 0 (stable); eps < delta: a positive eigenvalue.
    This pins reading c5 (the paper's 'eps - delta <= 0 is necessary', is a sign slip)."""
    c, wxy, wz, vx2, vn2, vz2 = _brute_setup()
    c = dict(c, nx=6, ny=6, nz=6)
    wz6 = W.z_weights(W.z_coords_ramp(6, 2, 6.0, 12.0), 2)
    v = np.full((6, 6, 6), 9e6)
    ev = np.linalg.eigvals(_dense_operator(c, wxy, wz6, v * 1.4, v * 1.2, v))  # eps=.2, delta=.1
    assert ev.real.max() < 1e-6 * np.abs(ev).max()
    ev = np.linalg.eigvals(_dense_operator(c, wxy, wz6, v * 1.2, v * 1.4, v))  # eps=.1, delta=.2
    assert ev.real.max() > 1e-3 * np.abs(ev).max()
    # Gershgorin dt of the generator is stable for the dense operator of config-style inputs
    cc = synth.scaled(synth.CONFIGS["C1"](), 6, 6, 6)
    wxy4, wz4, _ = synth.weights_f32(dict(cc, r_xy=2, r_z=2))
    dt = synth.stable_dt(dict(cc, r_xy=2, r_z=2), wxy4, wz4)
    vm = np.full((6, 6, 6), 9e6, dtype=np.float64)
    A = _dense_operator(dict(cc, r_xy=2, r_z=2), wxy4.astype(np.float64), wz4.astype(np.float64),
                        vm * 1.4, vm * 1.2, vm)
    assert dt <= 2 / math.sqrt(np.abs(np.linalg.eigvals(A)).max())
    del vx2, vn2, vz2


# ----------------------------------------------------------------------------- closed forms

def test_ricker_closed_forms():
    f = GOLD["ricker"]["f"]
    assert oracle.ricker(0.3, f, 0.3) == 1.0
    tz = 1.0 / (math.sqrt(2) * math.pi * f)
    assert abs(oracle.ricker(tz, f, 0.0)) < 1e-15
    assert abs(oracle.ricker(-tz, f, 0.0)) < 1e-15
    t = 0.0123
    a = (math.pi * f * t) ** 2
    assert oracle.ricker(t, f, 0.0) == pytest.approx((1 - 2 * a) * math.exp(-a), rel=1e-15)
    assert oracle.ricker(t, f, 0.0) == oracle.ricker(-t, f, 0.0)


def test_damping_closed_forms():
    d = GOLD["damping"]
    g = oracle.damping_profile(100, d["edge"]["W"], d["edge"]["alpha"])
    assert g[0] == np.float32(d["edge"]["g"]) and g[-1] == np.float32(d["edge"]["g"])
    assert (g[20:80] == 1.0).all() and g[19] < 1.0
    assert (np.diff(g[:21]) >= 0).all() and (g > 0).all() and (g <= 1).all()
    for k in range(20):
        assert g[k] == np.float32(math.exp(-(0.015 * (20 - k)) ** 2))
    assert (oracle.damping_profile(50, 0, 0.015) == 1.0).all()


def test_damping_corner_product_through_step():
    """Corner of a damped grid: p^{n+1} = g^3-product * 2p^n when F=0 and u^{n-1}=0."""
    c = cfg_small((45, 45, 45), (1, 1), damp=20, src=None)
    P = oracle.params(c, dt=1e-3)
    shape = (45, 45, 45)
    p = np.ones(shape)
    zero = np.zeros(shape)
    model = const_model(shape, 0.0, 0.0, 0.0)
    pn, _, _, _, _ = oracle.run(P, W.xy_weights(1), np.zeros((45, 3)), *model, (p, zero, zero, zero),
                                nsteps=1, dtype=np.float64)
    ge = math.exp(-0.09)
    assert pn[0, 0, 0] == pytest.approx(2 * ge ** 3, rel=1e-15)
    assert pn[22, 0, 0] == pytest.approx(2 * ge ** 2, rel=1e-15)
    assert pn[22, 22, 0] == pytest.approx(2 * ge, rel=1e-15)
    assert pn[0, 22, 22] == pytest.approx(2 * ge, rel=1e-15)
    assert pn[22, 22, 22] == 2.0


def test_thomsen_relations_generator():
    t = GOLD["thomsen"]
    cfg = dict(nx=2, ny=2, nz=2, model=dict(kind="homogeneous", vz=3000.0, eps=t["eps"], delta=t["delta"]))
    vx2, vn2, vz2 = synth.fields.model_planes(cfg, 0, 2)
    assert float(vz2[0, 0, 0]) == t["vz2"]
    assert float(vx2[0, 0, 0]) == pytest.approx(t["vx2"], rel=1e-7)
    assert float(vn2[0, 0, 0]) == pytest.approx(t["vn2"], rel=1e-7)


# ----------------------------------------------------------------------------- determinism

def test_thread_count_independence_and_linearity():
    c, wxy, wz, vz2 = _iso_setup(n=15, mask=1)
    vx2 = (vz2 * 1.4).astype(np.float32)
    vn2 = (vz2 * 1.2).astype(np.float32)
    P = oracle.params(c, dt=5e-4)
    a = oracle.run(P, wxy, wz, vx2, vn2, vz2, None, nsteps=30, nthreads=1)
    b = oracle.run(P, wxy, wz, vx2, vn2, vz2, None, nsteps=30, nthreads=4)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)
    c2 = dict(c, amp=2.0)
    P2 = oracle.params(c2, dt=5e-4)
    d = oracle.run(P2, wxy, wz, vx2, vn2, vz2, None, nsteps=30)
    for x, y in zip(a[:2], d[:2]):
        assert np.linalg.norm(2 * x - y) <= 1e-6 * np.linalg.norm(y)


def test_split_run_equals_single_run():
    """Running n1 then n2 steps from the returned state equals n1+n2 steps (time index carried)."""
    c, wxy, wz, vz2 = _iso_setup(n=13, mask=1)
    P = oracle.params(c, dt=5e-4)
    full = oracle.run(P, wxy, wz, vz2, vz2, vz2, None, nsteps=20)
    half = oracle.run(P, wxy, wz, vz2, vz2, vz2, None, nsteps=12)
    rest = oracle.run(P, wxy, wz, vz2, vz2, vz2, half[:4], n0=12, nsteps=8)
    for x, y in zip(full[:4], rest[:4]):
        assert np.array_equal(x, y)


def test_fp32_tracks_fp64_on_c1():
    """C1 (64^3, 100 steps): canonical fp32 within 1e-5 rel-L2 of the fp64 oracle."""
    cfg = synth.CONFIGS["C1"]()
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    vx2, vn2, vz2 = (a.numpy() for a in synth.fields.model_planes(cfg, 0, cfg["nz"]))
    P = oracle.params(cfg, dt=dt)
    p32, q32, _, _, _ = oracle.run(P, wxy, wz, vx2, vn2, vz2, None, nsteps=cfg["steps"])
    p64, q64, _, _, _ = oracle.run(P, wxy.astype(np.float64), wz.astype(np.float64), vx2, vn2, vz2,
                                   None, nsteps=cfg["steps"], dtype=np.float64)
    for a, b in ((p32, p64), (q32, q64)):
        assert np.abs(b).max() > 0
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)
