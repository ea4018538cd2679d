"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Gate (BASELINE.json north_star): max relative L2 <= 1e-5 in fp32. Both sides
implement the same canonical fp32 operation order (reading c12),
so the expected difference is exactly zero; the bitwise assertions below
document that, the 1e-5 gate is the contract.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import fields as SF
from synth import weights as W

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel_l2(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30))


def make(cfg, dt, wxy, wz, **kw):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0, **kw)


def random_state(cfg, seed=7, amp=1e-3):
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    return [SF.random_planes(nx, ny, 0, nz, seed, s, amp).numpy() for s in range(4)]


def random_model(cfg, seed=3):
    """Pointwise random VTI model, eps >= delta (stable)."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    u = [SF.random_planes(nx, ny, 0, nz, seed, 10 + s, 1.0).numpy().astype(np.float64) * 0.5 + 0.5
         for s in range(3)]
    vz2 = (2.0e6 + 7.0e6 * u[0]).astype(np.float32)
    eps = 0.25 * u[1]
    dl = eps * u[2]
    vx2 = (vz2.astype(np.float64) * (1 + 2 * eps)).astype(np.float32)
    vn2 = (vz2.astype(np.float64) * (1 + 2 * dl)).astype(np.float32)
    return vx2, vn2, vz2


def small_cfg(nx, ny, nz, r, rz, damp=4, src=None, mask=1, t0=0.02, dz=(6.0, 14.0)):
    c = synth.scaled(synth.CONFIGS["C2"](), nx, ny, nz, r_xy=r, r_z=rz, damp_width=damp, dz=dz, t0=t0,
                     mask=mask)
    if src is not None:
        c["src"] = src
    return c


def run_both(cfg, nsteps, state=None, model=None, with_source=True, n0=0):
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    if model is None:
        model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        if with_source:
            v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        if state is not None:
            v.set_fields(*state, time_index=n0)
        v.step(nsteps)
        assert v.time_index == n0 + nsteps
        g = v.get_fields(0) + v.get_fields(1)
    P = oracle.params(cfg, dt, src=cfg["src"] if with_source else None)
    o = oracle.run(P, wxy, wz, *model, state, n0=n0, nsteps=nsteps)[:4]
    return g, o


def assert_parity(g, o, bitwise=True):
    for a, b in zip(g, o):
        assert np.isfinite(a).all()
        assert rel_l2(a, b) <= TOL
        if bitwise:
            assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"


def test_c1_full_run():
    """BASELINE configs[0]: 64^3, R=(4,4), homogeneous eps=0.2 delta=0.1, 100 steps, source (32,32,32)."""
    cfg = synth.CONFIGS["C1"]()
    g, o = run_both(cfg, cfg["steps"])
    assert np.abs(o[0]).max() > 0
    assert_parity(g, o)


def test_c1_without_damping():
    cfg = dict(synth.CONFIGS["C1"](), damp_width=0)
    g, o = run_both(cfg, 60)
    assert_parity(g, o)


@pytest.mark.parametrize("r,rz", [(4, 4), (8, 4), (6, 6), (12, 8)])
@pytest.mark.parametrize("shape", [(61, 33, 47), (24, 24, 24), (130, 17, 40), (64, 32, 17)])
def test_random_state_ragged_shapes(r, rz, shape):
    """Random u^n, u^{n-1} and model on ragged grids (partial tiles in x, y and z), 3 steps."""
    nx, ny, nz = shape
    if nz < 2 * rz + 1 or ny < r:
        pytest.skip("grid smaller than the stencil")
    cfg = small_cfg(nx, ny, nz, r, rz, damp=min(4, (min(shape) - 1) // 2), src=(nx // 3, ny // 2, nz // 2))
    st = random_state(cfg)
    g, o = run_both(cfg, 3, state=st, model=random_model(cfg), n0=5)
    assert_parity(g, o)


@pytest.mark.parametrize("mask", [1, 2, 3])
def test_layered_source_masks(mask):
    cfg = small_cfg(72, 70, 66, 4, 4, damp=10, mask=mask, src=(30, 41, 29))
    g, o = run_both(cfg, 40)
    assert np.abs(o[0]).max() > 0 or np.abs(o[1]).max() > 0
    assert_parity(g, o)


def test_source_at_grid_corner_and_edges():
    cfg = small_cfg(40, 36, 30, 4, 4, damp=0, src=(0, 35, 29))
    g, o = run_both(cfg, 12)
    assert_parity(g, o)


def test_isotropic_limit_p_equals_q():
    """eps = delta = 0 with dual injection: p == q bitwise on the GPU (SURVEY 8(c) isotropic pin)."""
    cfg = synth.scaled(synth.CONFIGS["C5"](), 48, 40, 44, steps=30, damp_width=6, mask=3)
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    vx2, vn2, vz2 = (a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    assert np.array_equal(vx2, vn2)
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(vx2, vn2, vz2)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], mask=3)
        v.step(30)
        p, q = v.get_fields(0)
    assert np.abs(p).max() > 0 and np.array_equal(p, q)


def test_split_steps_and_time_index():
    cfg = small_cfg(50, 40, 36, 4, 4, damp=5, src=(20, 20, 18))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    out = []
    for chunks in ([25], [7, 11, 7]):
        with make(cfg, dt, wxy, wz) as v:
            v.set_model(*model)
            v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
            for c in chunks:
                v.step(c)
            out.append(v.get_fields(0))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_device_pointer_io_matches_host_io():
    cfg = small_cfg(40, 33, 30, 4, 4, damp=4)
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    st = random_state(cfg)
    res = []
    for dev in (False, True):
        conv = (lambda a: torch.from_numpy(a).cuda()) if dev else (lambda a: a)
        with make(cfg, dt, wxy, wz) as v:
            v.set_model(*[conv(a) for a in model])
            v.set_fields(*[conv(a) for a in st])
            v.step(4)
            if dev:
                p = torch.empty(cfg["nz"], cfg["ny"], cfg["nx"], device="cuda")
                q = torch.empty_like(p)
                v.get_fields(0, p, q)
                res.append((p.cpu().numpy(), q.cpu().numpy()))
            else:
                res.append(v.get_fields(0))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def test_planes_api_roundtrip():
    cfg = small_cfg(40, 20, 30, 4, 4, damp=0)
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    st = random_state(cfg)
    with make(cfg, dt, wxy, wz) as v:
        for k0 in range(0, 30, 7):
            sl = slice(k0, min(30, k0 + 7))
            v.set_model_planes(k0, *[a[sl] for a in model])
            v.set_fields_planes(k0, *[a[sl] for a in st])
        p, q = v.get_fields(0)
        pm, qm = v.get_fields(1)
        assert np.array_equal(p, st[0]) and np.array_equal(q, st[1])
        assert np.array_equal(pm, st[2]) and np.array_equal(qm, st[3])
        p2, _ = v.get_fields(0, planes=(5, 9))
        assert np.array_equal(p2, st[0][5:14])


def test_model_counts_as_set_only_when_every_plane_was_uploaded():
    """Uploading the same planes twice must not mark the model set (the
    never-uploaded planes keep vz2 = 0); the last missing plane completes it."""
    from paper_1410_1387_b200 import VTIError
    cfg = small_cfg(40, 20, 30, 4, 4, damp=0)
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    with make(cfg, dt, wxy, wz) as v:
        v.set_model_planes(0, *[a[:15] for a in model])
        v.set_model_planes(0, *[a[:15] for a in model])
        with pytest.raises(VTIError) as e:
            v.step(1)
        assert e.value.name == "VTI_E_STATE"
        v.set_model_planes(15, *[a[15:29] for a in model])
        with pytest.raises(VTIError):
            v.step(1)
        v.set_model_planes(29, *[a[29:] for a in model])
        v.step(1)


def test_errors_on_gpu_handle():
    from paper_1410_1387_b200 import VTIError
    cfg = small_cfg(40, 20, 30, 4, 4, damp=0)
    wxy, wz, _ = synth.weights_f32(cfg)
    with make(cfg, 1e-4, wxy, wz) as v:
        with pytest.raises(VTIError) as e:
            v.step(1)
        assert e.value.name == "VTI_E_STATE"
        with pytest.raises(VTIError) as e:
            v.add_source(40, 0, 0)
        assert e.value.name == "VTI_E_INDEX"
        with pytest.raises(VTIError) as e:
            v.add_source(1, 1, 1, mask=4)
        assert e.value.name == "VTI_E_PARAM"
        bad = np.ones((30, 20, 40), np.float32)
        with pytest.raises(VTIError) as e:
            v.set_model(bad, bad, -bad)
        assert e.value.name == "VTI_E_MODEL"
        v.set_model(bad, 2 * bad, bad)
        assert v.model_warnings() == 30 * 20 * 40   # eps < delta everywhere: warn-only


def test_check_every_detects_instability():
    from paper_1410_1387_b200 import VTIError
    cfg = small_cfg(32, 32, 32, 4, 4, damp=0, src=(16, 16, 16))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = 5 * synth.stable_dt(cfg, wxy, wz)   # far beyond the CFL bound
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    with make(cfg, dt, wxy, wz, check_every=25) as v:
        v.set_model(*model)
        v.set_fields(*random_state(cfg, amp=1.0))
        with pytest.raises(VTIError) as e:
            v.step(2000)
        assert e.value.name == "VTI_E_INSTABILITY"


@pytest.mark.parametrize("nranks", [2, 3])
def test_local_group_slabs_bitwise_equal_single(nranks):
    """y-slab decomposition (local group, fused peer-store halo transport) == one slab, bitwise."""
    from paper_1410_1387_b200 import VTI, group_step
    cfg = small_cfg(70, 75, 40, 4, 4, damp=6, src=(30, 37, 20))
    if nranks == 2:
        cfg["src"] = (30, 38, 20)   # first row of rank 1: source on a slab boundary
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    st = random_state(cfg, amp=1e-4)
    g, o = run_both(cfg, 9, state=st, model=model)
    assert_parity(g, o)
    hs = [VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], 4, 4, dt, wxy, wz, damp_width=cfg["damp_width"],
              damp_alpha=cfg["damp_alpha"], device=0, rank=r, nranks=nranks) for r in range(nranks)]
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
    group_step(hs, 4)
    group_step(hs, 5)
    parts = [h.get_fields(0) + h.get_fields(1) for h in hs]
    for f in range(4):
        full = np.concatenate([p[f] for p in parts], axis=1)
        assert np.array_equal(full, g[f])
    for h in hs:
        h.close()


@pytest.mark.parametrize("r,rz", [(4, 4), (8, 4), (6, 6), (12, 8)])
@pytest.mark.parametrize("ty,wp,rpt,px", [(32, 1, 1, 4), (32, 0, 1, 4), (32, 0, 2, 4), (16, -1, 1, 4),
                                         (30, 1, 2, 2), (32, 1, 2, 2)])
def test_every_compiled_variant(r, rz, ty, wp, rpt, px, monkeypatch):
    """Each (tile height, producer-warp, rows-per-thread, points-per-thread) instantiation is bitwise
    equal to the oracle (a combination not compiled for the pair falls back to the default, also checked)."""
    monkeypatch.setenv("VTI_TY", str(ty))
    monkeypatch.setenv("VTI_WP", str(wp))
    monkeypatch.setenv("VTI_RPT", str(rpt))
    monkeypatch.setenv("VTI_PX", str(px))
    cfg = small_cfg(77, 45, 41, r, rz, damp=5, src=(30, 22, 20))
    st = random_state(cfg, seed=9)
    g, o = run_both(cfg, 4, state=st, model=random_model(cfg, seed=5), n0=2)
    assert_parity(g, o)


@pytest.mark.parametrize("r,rz", [(4, 4), (6, 6)])
def test_autotune_then_parity(r, rz):
    """vti_autotune probes every variant on the zero state, then the run is still bitwise exact."""
    from paper_1410_1387_b200 import VTIError
    cfg = small_cfg(96, 70, 60, r, rz, damp=6, src=(40, 33, 30))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        res = v.autotune(probe_steps=2)
        assert res["candidates"] >= 3 and res["tile_y"] in (16, 30, 32) and res["ms_per_step"] > 0
        assert v.time_index == 0
        p0, q0 = v.get_fields(0)
        assert not p0.any() and not q0.any()          # probes left the zero state untouched
        info = v.info()
        assert info["tile_y"] == res["tile_y"] and info["zchunk"] == res["zchunk"]
        v.step(15)
        p, q = v.get_fields(0)
        with pytest.raises(VTIError) as e:
            v.autotune(2)                              # not the initial state any more
        assert e.value.name == "VTI_E_STATE"
    po, qo, _, _, _ = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, None, nsteps=15)
    assert np.abs(po).max() > 0
    assert np.array_equal(p, po) and np.array_equal(q, qo)


def test_set_variant_switches_kernel_mid_run():
    """Switching the compiled variant between steps keeps the result bitwise identical."""
    from paper_1410_1387_b200 import VTIError
    cfg = small_cfg(70, 50, 40, 4, 4, damp=5, src=(30, 25, 20))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        for ty, wp in ((32, 1), (16, -1), (32, 0), (32, 1)):
            v.set_variant(ty, wp)
            assert v.info()["tile_y"] == ty
            v.step(4)
        v.set_variant(32, 0, 2)
        assert v.info()["rows_per_thread"] == 2
        v.step(3)
        with pytest.raises(VTIError) as e:
            v.set_variant(8, 1)
        assert e.value.name == "VTI_E_UNSUPPORTED"
        p, q = v.get_fields(0)
    po, qo, _, _, _ = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, None, nsteps=19)
    assert np.array_equal(p, po) and np.array_equal(q, qo)


@pytest.mark.parametrize("ty", [16, 32])
@pytest.mark.parametrize("ny,nranks", [(66, 2), (67, 2), (100, 3), (98, 2), (140, 4)])
def test_local_group_short_last_tiles(ty, ny, nranks, monkeypatch):
    """Slabs whose last tile row is shorter than R_xy: the rows a neighbour receives span
    two tile rows, and all of them must be in the edge launch (multi-step, bitwise)."""
    from paper_1410_1387_b200 import VTI, group_step
    monkeypatch.setenv("VTI_TY", str(ty))
    cfg = small_cfg(70, ny, 30, 4, 4, damp=5, src=(30, ny // 2, 15))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    st = random_state(cfg, amp=1e-4)
    g, o = run_both(cfg, 6, state=st, model=model)
    assert_parity(g, o)
    hs = [VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], 4, 4, dt, wxy, wz, damp_width=cfg["damp_width"],
              damp_alpha=cfg["damp_alpha"], rank=r, nranks=nranks) for r in range(nranks)]
    for h in hs:
        assert h.info()["tile_y"] == ty
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
    group_step(hs, 2)
    group_step(hs, 4)
    parts = [h.get_fields(0) + h.get_fields(1) for h in hs]
    for f in range(4):
        assert np.array_equal(np.concatenate([p[f] for p in parts], axis=1), g[f])
    for h in hs:
        h.close()


@pytest.mark.parametrize("shape", [(1, 1, 9), (1, 40, 9), (37, 1, 12), (1, 1, 17), (5, 3, 9)])
def test_degenerate_thin_grids(shape):
    """Grids thinner than the stencil in x and/or y (the zero exterior does all the work)."""
    nx, ny, nz = shape
    cfg = small_cfg(nx, ny, nz, 4, 4, damp=0, src=(nx // 2, ny // 2, nz // 2))
    st = random_state(cfg, amp=1e-2)
    g, o = run_both(cfg, 7, state=st, model=random_model(cfg))
    assert_parity(g, o)


def test_zero_steps_and_zero_amplitude():
    cfg = small_cfg(40, 30, 20, 4, 4, damp=3)
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    st = random_state(cfg)
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.set_fields(*st, time_index=7)
        v.step(0)                                   # no-op
        assert v.time_index == 7
        p, q = v.get_fields(0)
        assert np.array_equal(p, st[0]) and np.array_equal(q, st[1])
    with make(cfg, dt, wxy, wz) as v:               # zero state, zero-amplitude source: stays exactly zero
        v.set_model(*model)
        v.add_source(*cfg["src"], amp=0.0)
        v.step(10)
        p, q = v.get_fields(0)
        assert not p.any() and not q.any()


def test_handle_schedule_equals_host_plan():
    """vti_query on a GPU handle reports the schedule vti_plan predicts on the host."""
    import torch
    from paper_1410_1387_b200 import plan
    cfg = small_cfg(300, 200, 96, 4, 4, damp=4)
    wxy, wz, _ = synth.weights_f32(cfg)
    with make(cfg, 1e-4, wxy, wz) as v:
        info = v.info()
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        assert info["tile_y"] == 32                     # default (4,4) variant: one CTA per SM
        p = plan(300, 200, 96, 4, 4, tile_y=32, sms=sms, ctas_per_sm=1)
        assert (info["zchunk"], info["work_items"], info["grid"]) == (p["zchunk"], p["items"], p["grid"])


def test_graph_replays_equal_direct_launches(monkeypatch):
    """Launch-bound grids step through CUDA-graph replays (32 steps each); the result is
    bitwise the direct-launch result, across a source change, an odd remainder and reversal."""
    cfg = small_cfg(60, 44, 40, 4, 4, damp=5, src=(20, 20, 20))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    out = []
    for graph in ("1", "0"):
        monkeypatch.setenv("VTI_GRAPH", graph)
        with make(cfg, dt, wxy, wz) as v:
            v.set_model(*model)
            v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
            v.step(70)                                   # 2 replays + 6 direct steps
            v.add_source(40, 10, 30, f=cfg["f"], t0=0.0, mask=3)   # invalidates the graphs
            v.step(33)
            v.reverse()
            v.step(64)
            assert v.time_index == 70 + 33 - 1 - 64
            out.append(v.get_fields(0) + v.get_fields(1))
    for a, b in zip(*out):
        assert np.array_equal(a, b)
    assert np.abs(out[0][0]).max() > 0


@pytest.mark.parametrize("r,rz", [(8, 4), (6, 6), (12, 8)])
@pytest.mark.parametrize("shape", [(1, 1, None), (5, 3, None), (70, 2, None), (3, 37, None)])
def test_degenerate_thin_grids_every_radius(r, rz, shape):
    """Thin grids at the smallest legal depth nz = 2 R_z + 1 for every compiled radius pair
    (the default variant of the pair, including the float2 x 2-row (12,8) mapping)."""
    nx, ny, _ = shape
    nz = 2 * rz + 1
    cfg = small_cfg(nx, ny, nz, r, rz, damp=0, src=(nx // 2, ny // 2, nz // 2))
    st = random_state(cfg, amp=1e-2)
    g, o = run_both(cfg, 5, state=st, model=random_model(cfg))
    assert_parity(g, o)


def test_widest_damping_band():
    """2W = extent - 1 on the smallest axis: every point of that axis is inside the band."""
    cfg = small_cfg(61, 45, 23, 4, 4, damp=11, src=(30, 22, 11))
    st = random_state(cfg, amp=1e-3)
    g, o = run_both(cfg, 6, state=st, model=random_model(cfg))
    assert_parity(g, o)


@pytest.mark.parametrize("r,rz,shape", [(4, 4, (64, 64, 64)), (8, 4, (77, 45, 41)), (6, 6, (70, 33, 29))])
def test_small_grid_kernel(r, rz, shape, monkeypatch):
    """Small single-slab grids whose plan cuts z into 1-plane items run the small-grid kernel
    (one CTA per tile-plane item, the whole q column in one TMA box): bitwise == oracle, and
    == the persistent kernel (VTI_SMALL=0)."""
    nx, ny, nz = shape
    if os.environ.get("VTI_LAYOUT") == "yzx":
        pytest.skip("the small-grid kernel is [z][y][x]-only")
    cfg = small_cfg(nx, ny, nz, r, rz, damp=5, src=(nx // 2, ny // 2, nz // 2))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    st = random_state(cfg, amp=1e-3)
    model = random_model(cfg)
    with make(cfg, dt, wxy, wz) as v:
        assert v.info()["small_kernel"] == 1 and v.info()["zchunk"] == 1
    g, o = run_both(cfg, 9, state=st, model=model, n0=1)
    assert_parity(g, o)
    monkeypatch.setenv("VTI_SMALL", "0")
    # the switch is read once per process; a fresh handle with an explicit variant uses the main kernel
    monkeypatch.setenv("VTI_TY", "16")
    with make(cfg, dt, wxy, wz) as v:
        assert v.info()["small_kernel"] == 0
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        v.set_fields(*st, time_index=1)
        v.step(9)
        g2 = v.get_fields(0) + v.get_fields(1)
    for a, b in zip(g, g2):
        assert np.array_equal(a, b)


def test_prepare_builds_graphs_without_stepping():
    """vti_prepare captures the step graphs of a small grid without running anything; the
    following steps (graph replays) stay bitwise equal to the oracle."""
    cfg = synth.CONFIGS["C1"]()
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    st = random_state(cfg, seed=5, amp=1e-3)
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        v.set_fields(*st, time_index=2)
        v.prepare()
        assert v.time_index == 2
        p, q = v.get_fields(0)
        assert np.array_equal(p, st[0]) and np.array_equal(q, st[1])   # nothing ran
        v.step(70)                                                      # 2 graph replays + 6 direct steps
        g = v.get_fields(0) + v.get_fields(1)
    o = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, n0=2, nsteps=70)[:4]
    assert_parity(g, o)
