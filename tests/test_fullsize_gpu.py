"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(default schedule of a fresh handle).

* C2 512^3 (R 4/4) and C3 1024x1024x512 (R 8/4), C5 1024^3 (R 6/6), N1 512^3
  (R 12/8, the float2 x 2-row default): the whole grid against the full-grid
  oracle, from seeded random states (every point non-trivial) and, for C2, from
  the bench's own start (zero state + source); C2 also in fp64 (double2 default).
* C4 2048x2048x1024 (R 4/4, 4.3 G points, 120 GB on the GPU): too large for the
  host oracle's full-grid run, so one step from a seeded random state is compared
  over 8 whole planes (z faces, middle, bottom band) against the oracle's
  plane-window stepper, from inputs regenerated on the host by the same
  counter-based generator.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import fields as SF

pytestmark = pytest.mark.gpu


def handle(cfg, dt, wxy, wz):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0)


def upload(v, cfg, seed=None, amp=1e-3, chunk=32):
    """Model (and optionally a random state) generated on the GPU plane-chunk by plane-chunk."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    for k0 in range(0, nz, chunk):
        nk = min(chunk, nz - k0)
        v.set_model_planes(k0, *[a.contiguous() for a in SF.model_planes(cfg, k0, nk, device="cuda")])
        if seed is not None:
            st = [SF.random_planes(nx, ny, k0, nk, seed, s, amp, device="cuda") for s in range(4)]
            v.set_fields_planes(k0, *st)
        torch.cuda.synchronize()


def host_inputs(cfg, seed=None, amp=1e-3):
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    model = [a.cpu().numpy() for a in SF.model_planes(cfg, 0, nz, device="cuda")]
    st = None
    if seed is not None:
        st = [SF.random_planes(nx, ny, 0, nz, seed, s, amp, device="cuda").cpu().numpy() for s in range(4)]
    torch.cuda.empty_cache()
    return model, st


def compare(a, b):
    assert np.isfinite(a).all()
    rel = np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30)
    assert rel <= 1e-5
    assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"


@pytest.mark.parametrize("name,nsteps", [("C2", 3), ("C3", 2), ("C5", 1), ("N1", 2)])
def test_full_grid_random_state(name, nsteps):
    cfg = synth.CONFIGS[name]()
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    with handle(cfg, dt, wxy, wz) as v:
        upload(v, cfg, seed=21)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.step(nsteps)
        g = v.get_fields(0) + v.get_fields(1)
    model, st = host_inputs(cfg, seed=21)
    o = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=nsteps)[:4]
    for a, b in zip(g, o):
        compare(a, b)


def test_c2_bench_start_50_steps():
    """bench.py's workload: C2 from the zero state with the Ricker source, 50 steps, whole grid."""
    cfg = synth.CONFIGS["C2"]()
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    with handle(cfg, dt, wxy, wz) as v:
        upload(v, cfg)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        v.step(50)
        p, q = v.get_fields(0)
    model, _ = host_inputs(cfg)
    po, qo, _, _, _ = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, None, nsteps=50)
    assert np.abs(po).max() > 0 and np.abs(qo).max() > 0
    compare(p, po)
    compare(q, qo)


def _host_planes(cfg, k0, nk, seed, stream, amp):
    """Planes k0..k0+nk-1 of a seeded random field on the host; planes outside the grid are 0."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    out = np.zeros((nk, ny, nx), np.float32)
    lo, hi = max(k0, 0), min(k0 + nk, nz)
    if hi > lo:
        out[lo - k0:hi - k0] = SF.random_planes(nx, ny, lo, hi - lo, seed, stream, amp).numpy()
    return out


# plane windows (k0, nk): the z faces, plane R_z (first with a full q column), the middle,
# and the band near the bottom face -- whole 2048 x 2048 planes, every x and y edge included
C4_WINDOWS = [(0, 2), (4, 1), (511, 2), (1019, 1), (1022, 2)]


def test_c4_whole_planes_one_step():
    """C4 (4.3 G points, 120 GB on the GPU) is too large for the host oracle's full-grid run:
    one step from a seeded random state is compared over whole planes (8 planes x 4.2 M points)
    against the oracle's plane-window stepper vto_step_planes (pinned against vto_run in
    tests/test_oracle_point_pins.py), with the windows' inputs regenerated on the host by the
    same counter-based generator."""
    cfg = synth.CONFIGS["C4"]()
    free, _ = torch.cuda.mem_get_info()
    if free < 130e9:
        pytest.skip(f"C4 needs ~125 GB of device memory, {free / 1e9:.0f} GB free")
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    seed, amp, Rz = 33, 1e-3, cfg["r_z"]
    got = {}
    with handle(cfg, dt, wxy, wz) as v:
        upload(v, cfg, seed=seed, amp=amp, chunk=16)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.step(1)
        for k0, nk in C4_WINDOWS:
            got[k0] = v.get_fields(0, planes=(k0, nk))
    torch.cuda.empty_cache()
    P = oracle.params(cfg, dt)
    for k0, nk in C4_WINDOWS:
        p = _host_planes(cfg, k0, nk, seed, 0, amp)
        q = _host_planes(cfg, k0 - Rz, nk + 2 * Rz, seed, 1, amp)
        pm = _host_planes(cfg, k0, nk, seed, 2, amp)
        qm = _host_planes(cfg, k0, nk, seed, 3, amp)
        model = [a.numpy() for a in SF.model_planes(cfg, k0, nk)]
        po, qo = oracle.step_planes(P, wxy, wz, k0, p, q, pm, qm, *model, n=0)
        gp, gq = got[k0]
        assert np.abs(po).max() > 0
        assert np.array_equal(gp, po), f"planes {k0}..{k0 + nk - 1}: p differs at {np.count_nonzero(gp != po)} points"
        assert np.array_equal(gq, qo), f"planes {k0}..{k0 + nk - 1}: q differs at {np.count_nonzero(gq != qo)} points"


def test_c2_fp64_full_grid():
    """The fp64 path (N3) at the C2 size, whole grid, against the oracle's fp64 mode."""
    from synth import weights as W
    from paper_1410_1387_b200 import VTI
    cfg = synth.CONFIGS["C2"]()
    wxy = W.xy_weights(cfg["r_xy"])
    zc = W.z_coords_ramp(cfg["nz"], cfg["r_z"], cfg["dz"][0], cfg["dz"][1])
    wz = np.ascontiguousarray(W.z_weights(zc, cfg["r_z"]))
    dt = synth.stable_dt(cfg)
    model, st = host_inputs(cfg, seed=23)
    model = [a.astype(np.float64) for a in model]
    st = [a.astype(np.float64) for a in st]
    with VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
             damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0, precision=64) as v:
        assert v.info()["points_per_thread"] == 2
        v.set_model(*model)
        v.set_fields(*st)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.step(2)
        g = v.get_fields(0) + v.get_fields(1)
    o = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=2, dtype=np.float64)[:4]
    for a, b in zip(g, o):
        assert a.dtype == np.float64 and np.isfinite(a).all()
        assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"
