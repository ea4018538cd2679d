"""fp64 path: the double-precision kernel vs the oracle's fp64 mode.

Same canonical operation order as fp32 with __fma_rn / fma, every derived
scalar (cxy = w/h^2, dt^2, damping, s_n) evaluated in double on both sides and
never rounded, so the expected difference is zero; the gate is 1e-12 rel-L2.
"""
import numpy as np
import pytest

import oracle
import synth
from synth import fields as SF
from synth import weights as W

pytestmark = pytest.mark.gpu


def cfg_of(nx, ny, nz, r, rz, damp=5, src=None, t0=0.02):
    c = synth.scaled(synth.CONFIGS["C2"](), nx, ny, nz, r_xy=r, r_z=rz, damp_width=damp, dz=(6.0, 14.0), t0=t0)
    if src is not None:
        c["src"] = src
    return c


def weights64(cfg):
    wxy = W.xy_weights(cfg["r_xy"])
    zc = W.z_coords_ramp(cfg["nz"], cfg["r_z"], cfg["dz"][0], cfg["dz"][1])
    return wxy, np.ascontiguousarray(W.z_weights(zc, cfg["r_z"]))


def make64(cfg, dt, wxy, wz, **kw):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], precision=64, **kw)


def inputs(cfg, seed=4):
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    model = [a.numpy().astype(np.float64) for a in SF.model_planes(cfg, 0, nz)]
    st = [SF.random_planes(nx, ny, 0, nz, seed, s, 1e-3).numpy().astype(np.float64) for s in range(4)]
    return model, st


def run64(cfg, nsteps, state, model, variant=None):
    wxy, wz = weights64(cfg)
    dt = synth.stable_dt(cfg)
    with make64(cfg, dt, wxy, wz) as v:
        if variant:
            v.set_variant(*variant)
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        if state is not None:
            v.set_fields(*state, time_index=3)
        v.step(nsteps)
        g = v.get_fields(0) + v.get_fields(1)
    n0 = 3 if state is not None else 0
    o = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, state, n0=n0, nsteps=nsteps, dtype=np.float64)[:4]
    return g, o


def check(g, o):
    for a, b in zip(g, o):
        assert a.dtype == np.float64
        assert np.linalg.norm(a - b) <= 1e-12 * max(np.linalg.norm(b), 1e-300)
        assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"


@pytest.mark.parametrize("r,rz", [(4, 4), (8, 4), (6, 6), (12, 8)])
@pytest.mark.parametrize("ty,wp,px", [(16, 1, 4), (16, 0, 4), (14, 1, 4), (15, 1, 2), (16, 0, 2), (16, 1, 2)])
def test_fp64_random_state_ragged(r, rz, ty, wp, px):
    from paper_1410_1387_b200 import VTIError
    cfg = cfg_of(77, 45, 41, r, rz, src=(30, 22, 20))
    model, st = inputs(cfg)
    try:
        g, o = run64(cfg, 4, st, model, variant=(ty, wp, 1, px))
    except VTIError as e:
        assert e.name == "VTI_E_UNSUPPORTED"
        pytest.skip(f"variant ({ty}, {wp}, px {px}) not compiled for ({r}, {rz})")
    check(g, o)


def test_fp64_c1_from_zero_state():
    cfg = synth.CONFIGS["C1"]()
    cfg = dict(cfg, dz=(10.0, 10.0))
    model = [a.numpy().astype(np.float64) for a in SF.model_planes(cfg, 0, cfg["nz"])]
    g, o = run64(cfg, 60, None, model)
    assert np.abs(o[0]).max() > 0
    check(g, o)


def test_fp64_precision_mismatch_is_param_error():
    from paper_1410_1387_b200 import VTIError, lib
    import ctypes as C
    cfg = cfg_of(40, 20, 30, 4, 4, damp=0)
    wxy, wz = weights64(cfg)
    with make64(cfg, 1e-4, wxy, wz) as v:
        a = np.ones((30, 20, 40), np.float32)
        st = lib.vti_set_model(v.h, a.ctypes.data, a.ctypes.data, a.ctypes.data)
        assert st == 1 and b"fp64" in lib.vti_last_error(v.h)
        with pytest.raises(TypeError):
            v.get_fields(0, p=np.empty((30, 20, 40), np.float32))


def test_fp64_local_group_equals_single():
    from paper_1410_1387_b200 import group_step
    cfg = cfg_of(70, 66, 36, 4, 4, damp=6, src=(30, 33, 18))
    model, st = inputs(cfg)
    g, o = run64(cfg, 5, st, model)
    check(g, o)
    wxy, wz = weights64(cfg)
    dt = synth.stable_dt(cfg)
    hs = [make64(cfg, dt, wxy, wz, rank=r, nranks=2) for r in range(2)]
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st], time_index=3)
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
    group_step(hs, 5)
    parts = [h.get_fields(0) + h.get_fields(1) for h in hs]
    for f in range(4):
        assert np.array_equal(np.concatenate([p[f] for p in parts], axis=1), g[f])
    for h in hs:
        h.close()


@pytest.mark.parametrize("r,rz", [(4, 4), (12, 8)])
def test_fp64_thin_grid_minimum_depth(r, rz):
    cfg = cfg_of(5, 3, 2 * rz + 1, r, rz, damp=0, src=(2, 1, rz))
    model, st = inputs(cfg)
    g, o = run64(cfg, 4, st, model)
    check(g, o)
