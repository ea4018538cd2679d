"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(default schedule of a fresh handle).

* C2 512^3 (R 4/4) and C3 1024x1024x512 (R 8/4), C5 1024^3 (R 6/6), N1 512^3
  (R 12/8, the float2 x 2-row default): the whole grid against the full-grid
  oracle, from seeded random states (every point non-trivial) and, for C2, from
  the bench's own start (zero state + source); C2 also in fp64 (double2 default).
* C4 2048x2048x1024 (R 4/4, 4.3 G points, 120 GB on the GPU): too large for the
  host oracle, so one step from a seeded random state is compared at ~3000
  sampled points (tile, chunk, slab and domain edges included), each evaluated
  by the oracle's single-point function from neighbourhoods regenerated on the
  host by the same counter-based generator.
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


def _samples(cfg, n_random=2500, seed=3):
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    rng = np.random.default_rng(seed)
    pts = set()
    edges_x = [0, 1, 3, 4, 63, 64, 65, nx // 2, nx - 5, nx - 4, nx - 1]
    edges_y = [0, 1, 4, 15, 16, 17, ny // 2, ny - 17, ny - 16, ny - 1]
    edges_z = [0, 1, 3, 4, 63, 64, 65, nz // 2, nz - 5, nz - 1]
    for _ in range(400):
        pts.add((int(rng.choice(edges_x)), int(rng.choice(edges_y)), int(rng.choice(edges_z))))
    for _ in range(n_random):
        pts.add((int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))))
    pts.add(tuple(cfg["src"]))
    return sorted(pts, key=lambda t: (t[2], t[1], t[0]))


def _gather(cfg, pts, seed, amp):
    """Oracle-side neighbourhoods regenerated on the host (same counter-based generator)."""
    nx, ny, nz, R, Rz = cfg["nx"], cfg["ny"], cfg["nz"], cfg["r_xy"], cfg["r_z"]
    I = np.array([p[0] for p in pts])
    J = np.array([p[1] for p in pts])
    K = np.array([p[2] for p in pts])
    offs = [(0, 0)] + [(l, 0) for l in range(1, R + 1)] + [(-l, 0) for l in range(1, R + 1)] + \
           [(0, l) for l in range(1, R + 1)] + [(0, -l) for l in range(1, R + 1)]
    pc = np.zeros((len(pts), 4 * R + 1), np.float32)
    for c, (di, dj) in enumerate(offs):
        ii, jj = I + di, J + dj
        ok = (ii >= 0) & (ii < nx) & (jj >= 0) & (jj < ny)
        val = SF.random_at(torch.from_numpy(np.clip(ii, 0, nx - 1)), torch.from_numpy(np.clip(jj, 0, ny - 1)),
                           torch.from_numpy(K), nx, ny, seed, 0, amp).numpy()
        pc[:, c] = np.where(ok, val, 0.0)
    qc = np.zeros((len(pts), 2 * Rz + 1), np.float32)
    for m in range(2 * Rz + 1):
        kk = K - Rz + m
        ok = (kk >= 0) & (kk < nz)
        val = SF.random_at(torch.from_numpy(I), torch.from_numpy(J), torch.from_numpy(np.clip(kk, 0, nz - 1)),
                           nx, ny, seed, 1, amp).numpy()
        qc[:, m] = np.where(ok, val, 0.0)
    ti, tj, tk = (torch.from_numpy(a) for a in (I, J, K))
    pm = SF.random_at(ti, tj, tk, nx, ny, seed, 2, amp).numpy()
    qm = SF.random_at(ti, tj, tk, nx, ny, seed, 3, amp).numpy()
    vx2, vn2, vz2 = (a.numpy() for a in SF.layered_model_at(ti, tj, tk, nx, ny, nz, cfg["model"]))
    return pc, qc, pm, qm, vx2, vn2, vz2


def test_c4_sampled_points_one_step():
    cfg = synth.CONFIGS["C4"]()
    free, _ = torch.cuda.mem_get_info()
    if free < 130e9:
        pytest.skip(f"C4 needs ~125 GB of device memory, {free / 1e9:.0f} GB free")
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    seed, amp = 33, 1e-3
    pts = _samples(cfg)
    planes = sorted({p[2] for p in pts})
    got = {}
    with handle(cfg, dt, wxy, wz) as v:
        upload(v, cfg, seed=seed, amp=amp, chunk=16)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.step(1)
        for k in planes:
            p, q = v.get_fields(0, planes=(k, 1))
            for (i, j, kk) in pts:
                if kk == k:
                    got[(i, j, k)] = (p[0, j, i], q[0, j, i])
    pc, qc, pm, qm, vx2, vn2, vz2 = _gather(cfg, pts, seed, amp)
    P = oracle.params(cfg, dt)
    bad = 0
    for n, (i, j, k) in enumerate(pts):
        po, qo = oracle.point(P, wxy, wz[k], i, j, k, 0, pc[n], qc[n], pm[n], qm[n], vx2[n], vn2[n], vz2[n])
        gp, gq = got[(i, j, k)]
        bad += (gp != po) + (gq != qo)
    assert bad == 0, f"{bad} mismatching values over {len(pts)} points"


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
