"""vti_step_adjoint (the transpose recurrence) against the oracle's
vto_adjoint_ex (pinned in tests/test_oracle_adjoint_pins.py): bitwise for every compiled radius
pair in fp32 and in fp64, with damping, injected adjoint sources and receivers; plus the
dot-product identity <M^K X, Y> = <X, (M^T)^K Y> between the library's own forward and adjoint
steps."""
import numpy as np
import pytest

import oracle
import synth
from synth import fields as SF
from synth import weights as W

pytestmark = pytest.mark.gpu


def setup(r, rz, prec=32, shape=(70, 45, 33)):
    nx, ny, nz = shape
    cfg = synth.scaled(synth.CONFIGS["C2"](), nx, ny, max(nz, 2 * rz + 9), r_xy=r, r_z=rz, damp_width=5,
                       dz=(6.0, 12.0), t0=0.02)
    if prec == 32:
        wxy, wz, _ = synth.weights_f32(cfg)
    else:
        wxy = W.xy_weights(r)
        wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(cfg["nz"], rz, 6.0, 12.0), rz))
    dt = synth.stable_dt(cfg)
    dtype = np.float32 if prec == 32 else np.float64
    model = [a.numpy().astype(dtype) for a in SF.model_planes(cfg, 0, cfg["nz"])]
    st = [SF.random_planes(cfg["nx"], cfg["ny"], 0, cfg["nz"], 12, s, 1e-3).numpy().astype(dtype) for s in range(4)]
    return cfg, wxy, wz, dt, model, st, dtype


def handle(cfg, dt, wxy, wz, prec=32, **kw):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0, precision=prec, **kw)


@pytest.mark.parametrize("r,rz,prec", [(4, 4, 32), (8, 4, 32), (6, 6, 32), (12, 8, 32), (4, 4, 64), (12, 8, 64)])
def test_adjoint_matches_oracle(r, rz, prec):
    cfg, wxy, wz, dt, model, st, dtype = setup(r, rz, prec)
    rng = np.random.default_rng(r * 10 + rz)
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    pts = np.array(sorted({(int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))) for _ in range(40)}
                          | {(0, 0, 0), (nx - 1, ny - 1, nz - 1), (64, 20, 3)}), np.int32)
    tr = (rng.normal(size=(12, len(pts))) * 1e2).astype(dtype)
    m0, K = 30, 12
    with handle(cfg, dt, wxy, wz, prec) as v:
        v.set_model(*model)
        v.set_fields(*st, time_index=m0)
        v.set_injection(pts, tr, fields=3, t_first=m0 - 10)   # rows for m = 20..31: part of the run
        v.set_receivers(pts[:15], fields=3, capacity_steps=K)
        v.step_adjoint(K)
        assert v.time_index == m0 - K
        g = v.get_fields(0) + v.get_fields(1)
        _, traces = v.get_traces()
    o = oracle.adjoint_ex(oracle.params(cfg, dt, src=None), wxy, wz, *model, st, m0=m0, nsteps=K,
                          inj=(pts, 3, m0 - 10, tr), rec=(pts[:15], 3), dtype=dtype)
    for a, b in zip(g, o[:4]):
        assert np.abs(b).max() > 0
        assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"
    assert np.array_equal(traces, o[4])


@pytest.mark.parametrize("r,rz,prec", [(4, 4, 32), (8, 4, 32), (6, 6, 32), (12, 8, 32),
                                        (4, 4, 64), (8, 4, 64), (6, 6, 64), (12, 8, 64)])
def test_adjoint_no_points_matches_oracle(r, rz, prec):
    """The kernel without point sets, on a grid of 3 x tiles (ragged), ragged tile rows and
    several z-chunks, from a damped random state: bitwise."""
    cfg, wxy, wz, dt, model, st, dtype = setup(r, rz, prec, shape=(150, 37, 2 * rz + 60))
    m0, K = 9, 5
    with handle(cfg, dt, wxy, wz, prec) as v:
        v.set_model(*model)
        v.set_fields(*st, time_index=m0)
        v.step_adjoint(K)
        g = v.get_fields(0) + v.get_fields(1)
    o = oracle.adjoint_ex(oracle.params(cfg, dt, src=None), wxy, wz, *model, st, m0=m0, nsteps=K, dtype=dtype)
    for f, (a, b) in enumerate(zip(g, o[:4])):
        assert np.abs(b).max() > 0
        assert np.array_equal(a, b), f"field {f}: max |diff| {np.abs(a - b).max():.3e}"


@pytest.mark.parametrize("r,rz,prec", [(4, 4, 32), (12, 8, 32), (4, 4, 64)])
def test_adjoint_split_calls_equal_one_call(r, rz, prec):
    """Calls of 1 + 3 + 4 adjoint steps equal one call of 8 (the chained form restarts its
    first pass per call), with receivers spanning the calls and check_every on."""
    cfg, wxy, wz, dt, model, st, dtype = setup(r, rz, prec, shape=(100, 40, 2 * rz + 30))
    pts = np.array([(3, 4, 5), (50, 20, 10), (99, 39, 2 * rz + 29)], np.int32)
    out = []
    for split in ((8,), (1, 3, 4)):
        with handle(cfg, dt, wxy, wz, prec, check_every=2) as v:
            v.set_model(*model)
            v.set_fields(*st, time_index=20)
            v.set_receivers(pts, fields=3, capacity_steps=8)
            for k in split:
                v.step_adjoint(k)
            out.append((v.get_fields(0) + v.get_fields(1), v.get_traces()[1], v.time_index))
    assert out[0][2] == out[1][2] == 12
    for a, b in zip(out[0][0], out[1][0]):
        assert np.array_equal(a, b)
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("r,rz,prec", [(4, 4, 32), (12, 8, 32), (4, 4, 64)])
def test_adjoint_long_calls_match_oracle(r, rz, prec):
    """Long calls (37 then 20 steps: programmatic dependent launches back to back, the chained
    s1 buffers alternating from both buffer parities), bitwise against the oracle."""
    cfg, wxy, wz, dt, model, st, dtype = setup(r, rz, prec, shape=(70, 40, 2 * rz + 20))
    with handle(cfg, dt, wxy, wz, prec) as v:
        v.set_model(*model)
        v.set_fields(*st, time_index=80)
        v.step_adjoint(37)
        v.step_adjoint(20)
        assert v.time_index == 23
        g = v.get_fields(0) + v.get_fields(1)
    o = oracle.adjoint_ex(oracle.params(cfg, dt, src=None), wxy, wz, *model, st, m0=80, nsteps=57, dtype=dtype)
    for f, (a, b) in enumerate(zip(g, o[:4])):
        assert np.abs(b).max() > 0
        assert np.array_equal(a, b), f"field {f}: max |diff| {np.abs(a - b).max():.3e}"


def test_library_dot_product_identity():
    """fp64, damped: the library's K forward steps and K adjoint steps satisfy
    <u^K, psi^K / g> - <u^{K-1}, g psi^{K+1}> = <u^0, psi^0 / g> - <u^{-1}, g psi^1>."""
    cfg, wxy, wz, dt, model, st, dtype = setup(4, 4, 64, shape=(40, 36, 30))
    rng = np.random.default_rng(17)
    shape = model[0].shape
    X0 = [rng.normal(size=shape) for _ in range(4)]
    psiK = [rng.normal(size=shape) for _ in range(4)]
    K = 16
    with handle(cfg, dt, wxy, wz, 64) as v:
        v.set_model(*model)
        v.set_fields(*X0)
        v.step(K)
        XK = list(v.get_fields(0) + v.get_fields(1))
        v.set_fields(*psiK, time_index=K)
        v.step_adjoint(K)
        psi0 = list(v.get_fields(0) + v.get_fields(1))
    d = lambda i, n: oracle.lib().vto_damping(i, n, cfg["damp_width"], cfg["damp_alpha"])
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    g = (np.array([d(i, nx) for i in range(nx)])[None, None, :] * np.array([d(j, ny) for j in range(ny)])[None, :, None]) \
        * np.array([d(k, nz) for k in range(nz)])[:, None, None]
    dot = lambda u, w: sum(np.vdot(a, b) for a, b in zip(u, w))
    lhs = dot(XK[:2], [a / g for a in psiK[:2]]) - dot(XK[2:], [g * a for a in psiK[2:]])
    rhs = dot(X0[:2], [a / g for a in psi0[:2]]) - dot(X0[2:], [g * a for a in psi0[2:]])
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs)) and abs(lhs) > 1.0


def test_adjoint_errors():
    from paper_1410_1387_b200 import VTIError
    cfg, wxy, wz, dt, model, st, dtype = setup(4, 4)
    with handle(cfg, dt, wxy, wz) as v:
        with pytest.raises(VTIError) as e:
            v.step_adjoint(1)
        assert e.value.name == "VTI_E_STATE"
    with handle(cfg, dt, wxy, wz, rank=0, nranks=2) as v:
        v.set_model(*[np.ascontiguousarray(a[:, :v.ny_local]) for a in model])
        with pytest.raises(VTIError) as e:
            v.step_adjoint(1)
        assert e.value.name == "VTI_E_STATE"


@pytest.mark.parametrize("r,rz,prec,nranks", [(4, 4, 32, 2), (8, 4, 32, 3), (12, 8, 32, 2), (6, 6, 64, 3)])
def test_group_adjoint_matches_single_slab_and_oracle(r, rz, prec, nranks):
    """vti_group_step_adjoint over y-slabs (s1 halo rows copied from the neighbours): bitwise
    equal to the oracle's adjoint, with injection (points on slab boundaries) and receivers."""
    from paper_1410_1387_b200 import group_step
    cfg, wxy, wz, dt, model, st, dtype = setup(r, rz, prec, shape=(70, 24 * nranks + 5, 2 * rz + 9))
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    from paper_1410_1387_b200 import slab
    bounds = [slab(ny, q, nranks) for q in range(nranks)]
    pts = [(5, 0, 0), (69, ny - 1, nz - 1), (30, ny // 2, nz // 2)]
    for y0, nyl in bounds[1:]:
        pts += [(31, y0 - 1, 3), (32, y0, 4), (33, y0 + 1, 5)]
    pts = np.array(sorted(set(pts)), np.int32)
    tr = np.random.default_rng(7).normal(size=(8, len(pts))).astype(dtype) * 10
    m0, K = 20, 8
    hs = [handle(cfg, dt, wxy, wz, prec, rank=q, nranks=nranks) for q in range(nranks)]
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st], time_index=m0)
        h.set_injection(pts, tr, fields=3, t_first=m0 - 6)
        h.set_receivers(pts, fields=1, capacity_steps=K)
    group_step(hs, K, transport="adjoint")
    got = [np.concatenate([h.get_fields(0)[f] for h in hs], axis=1) for f in range(2)]
    traces = np.zeros((K, len(pts), 1), dtype)
    for h in hs:
        ids, t = h.get_traces()
        traces[:, ids] = t
        h.close()
    o = oracle.adjoint_ex(oracle.params(cfg, dt, src=None), wxy, wz, *model, st, m0=m0, nsteps=K,
                          inj=(pts, 3, m0 - 6, tr), rec=(pts, 1), dtype=dtype)
    for f in range(2):
        assert np.array_equal(got[f], o[f]), f"field {f}"
    assert np.array_equal(traces, o[4])


def test_group_forward_after_adjoint_republishes_halos():
    """Forward steps after adjoint steps in a local group read fresh halo rows: equal to the
    same sequence on one slab."""
    from paper_1410_1387_b200 import group_step
    cfg, wxy, wz, dt, model, st, dtype = setup(4, 4, 32, shape=(70, 53, 17))
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.set_fields(*st, time_index=10)
        v.step(3)
        v.step_adjoint(4)
        v.step(5)
        ref = v.get_fields(0) + v.get_fields(1)
    hs = [handle(cfg, dt, wxy, wz, rank=q, nranks=2) for q in range(2)]
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st], time_index=10)
    group_step(hs, 3)
    group_step(hs, 4, transport="adjoint")
    group_step(hs, 5)
    got = [np.concatenate([(h.get_fields(0) + h.get_fields(1))[f] for h in hs], axis=1) for f in range(4)]
    for h in hs:
        h.close()
    for f in range(4):
        assert np.array_equal(got[f], ref[f]), f"field {f}"
