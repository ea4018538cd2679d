"""SURVEY.md 8(f) N4 hooks: receiver traces and time reversal, against the oracle."""
import os

import numpy as np
import pytest

import oracle
import synth
from synth import fields as SF

pytestmark = pytest.mark.gpu


def setup(nx=60, ny=50, nz=40, damp=5, src=(25, 24, 20)):
    cfg = synth.scaled(synth.CONFIGS["C2"](), nx, ny, nz, damp_width=damp, dz=(6.0, 12.0), t0=0.02, src=src)
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = [a.numpy() for a in SF.model_planes(cfg, 0, nz)]
    return cfg, wxy, wz, dt, model


def handle(cfg, dt, wxy, wz, **kw):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], **kw)


REC = np.array([[25, 24, 20], [0, 0, 0], [59, 49, 39], [30, 10, 5], [10, 40, 33], [25, 25, 20]], np.int32)


def test_receiver_traces_match_fields_and_oracle():
    cfg, wxy, wz, dt, model = setup()
    nsteps = 12
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.set_receivers(REC, fields=3, capacity_steps=100)
        sampled = []
        for _ in range(nsteps):
            v.step(1)
            p, q = v.get_fields(0)
            sampled.append(np.stack([p[REC[:, 2], REC[:, 1], REC[:, 0]], q[REC[:, 2], REC[:, 1], REC[:, 0]]], -1))
        ids, tr = v.get_traces()
    assert list(ids) == list(range(len(REC))) and tr.shape == (nsteps, len(REC), 2)
    assert np.array_equal(tr, np.stack(sampled))
    # the same traces from the oracle, one step at a time
    P = oracle.params(cfg, dt)
    st = None
    for n in range(nsteps):
        st = oracle.run(P, wxy, wz, *model, st, n0=n, nsteps=1)[:4]
        assert np.array_equal(tr[n, :, 0], st[0][REC[:, 2], REC[:, 1], REC[:, 0]])
        assert np.array_equal(tr[n, :, 1], st[1][REC[:, 2], REC[:, 1], REC[:, 0]])
    assert np.abs(tr).max() > 0


def test_receiver_capacity_and_errors():
    from paper_1410_1387_b200 import VTIError
    cfg, wxy, wz, dt, model = setup()
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.set_receivers(REC[:2], fields=1, capacity_steps=3)
        v.step(5)
        ids, tr = v.get_traces()
        assert tr.shape == (3, 2, 1)
        with pytest.raises(VTIError) as e:
            v.set_receivers([[60, 0, 0]])
        assert e.value.name == "VTI_E_INDEX"


def test_receivers_across_slabs():
    from paper_1410_1387_b200 import group_step
    cfg, wxy, wz, dt, model = setup(ny=70, src=(25, 35, 20))
    rec = np.array([[25, 34, 20], [25, 35, 20], [3, 0, 1], [40, 69, 30], [12, 36, 7]], np.int32)
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.set_receivers(rec, fields=1, capacity_steps=20)
        v.step(8)
        _, ref = v.get_traces()
    hs = [handle(cfg, dt, wxy, wz, rank=r, nranks=2) for r in range(2)]
    got = np.zeros_like(ref)
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        h.set_receivers(rec, fields=1, capacity_steps=20)
    group_step(hs, 8)
    seen = []
    for h in hs:
        ids, tr = h.get_traces()
        got[:, ids] = tr
        seen += list(ids)
        h.close()
    assert sorted(seen) == list(range(len(rec)))
    assert np.array_equal(got, ref)


def test_reverse_matches_oracle_backwards():
    """vti_reverse then K steps == the oracle applying Eq. 3 with the levels swapped, n decreasing."""
    cfg, wxy, wz, dt, model = setup(damp=6)
    st0 = [SF.random_planes(cfg["nx"], cfg["ny"], 0, cfg["nz"], 8, s, 1e-3).numpy() for s in range(4)]
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.set_fields(*st0, time_index=20)
        v.step(6)                       # forward to level 26
        fwd = v.get_fields(0) + v.get_fields(1)
        v.reverse()
        assert v.direction == -1 and v.time_index == 25
        v.step(9)                       # backward to level 16
        assert v.time_index == 16
        back = v.get_fields(0) + v.get_fields(1)
    P = oracle.params(cfg, dt)
    st = oracle.run(P, wxy, wz, *model, st0, n0=20, nsteps=6)[:4]
    for a, b in zip(fwd, st):
        assert np.array_equal(a, b)
    # swap levels: current = u^25 (stored prev), previous = u^26
    cur = [st[2], st[3], st[0], st[1]]
    for n in range(25, 16, -1):         # Eq. 3 at level n with s(t^n), producing u^{n-1}
        cur = oracle.run(P, wxy, wz, *model, cur, n0=n, nsteps=1)[:4]
    for a, b in zip(back, cur):
        assert np.array_equal(a, b)


def test_reverse_recovers_initial_state_without_damping():
    """W = 0, no source: K steps forward, reverse, K steps back -> the initial state (rounding only)."""
    cfg, wxy, wz, dt, model = setup(damp=0)
    st0 = [SF.random_planes(cfg["nx"], cfg["ny"], 0, cfg["nz"], 9, s, 1e-3).numpy() for s in range(4)]
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.set_fields(*st0)
        v.step(25)                       # level 25 (stored level 24)
        v.reverse()                      # current level 24, stored level 25
        assert v.time_index == 24
        v.step(24)                       # back to level 0
        assert v.time_index == 0
        p0, q0 = v.get_fields(0)
        v.step(1)                        # level -1 = the initial u^{n-1}
        assert v.time_index == -1
        p, q = v.get_fields(0)
    for got, want in ((p0, st0[0]), (q0, st0[1]), (p, st0[2]), (q, st0[3])):
        rel = np.linalg.norm(got.astype(np.float64) - want) / np.linalg.norm(want)
        assert rel < 1e-4, rel


# ---------------------------------------------------------------- trace injection (fused, IO kernels)

def _inj_points(cfg, n_rand, seed, extra=()):
    rng = np.random.default_rng(seed)
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    pts = {tuple(cfg["src"])} | set(extra)
    # tile / row / plane edges, a whole row segment of one plane, the domain corners
    for i in (0, 1, 63, 64, nx - 1):
        pts.add((min(i, nx - 1), ny // 2, nz // 3))
    for i in range(10, 30):
        pts.add((i, 7, 5))
    pts |= {(0, 0, 0), (nx - 1, ny - 1, nz - 1)}
    while len(pts) < n_rand:
        pts.add((int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))))
    return np.array(sorted(pts, key=lambda t: (t[2], t[1], t[0])), np.int32)[rng.permutation(len(pts))]


@pytest.mark.parametrize("grid,nsteps,small", [((60, 50, 40), 70, True), ((96, 96, 72), 50, False)])
def test_injection_and_receivers_match_oracle(grid, nsteps, small):
    """Multi-point trace injection (+ the Ricker source at one of the points) and receivers
    over >= 50 steps: fields and traces bitwise equal to the oracle's vto_run_ex. The small grid
    runs through the small-grid kernel with CUDA-graph replays (70 steps = 2 x 32 + 6 direct);
    the larger one through the persistent TMA step kernel."""
    cfg, wxy, wz, dt, model = setup(*grid, damp=6, src=(grid[0] // 2, grid[1] // 2, grid[2] // 2))
    pts = _inj_points(cfg, 90, 3)
    rng = np.random.default_rng(5)
    t_first, nt = 3, nsteps - 10             # rows outside [t_first, t_first + nt) inject nothing
    tr = (rng.normal(size=(nt, len(pts))) * 5.0).astype(np.float32)
    rec = np.concatenate([pts[:40], REC[:3] % np.array(grid[::1], np.int32)])
    with handle(cfg, dt, wxy, wz) as v:
        if os.environ.get("VTI_LAYOUT") != "yzx":   # the small-grid kernel is [z][y][x]-only
            assert v.info()["small_kernel"] == int(small)
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], mask=1)
        v.set_injection(pts, tr, fields=3, t_first=t_first)
        v.set_receivers(rec, fields=3, capacity_steps=nsteps + 5)
        v.step(nsteps)
        g = v.get_fields(0) + v.get_fields(1)
        ids, traces = v.get_traces()
    P = oracle.params(dict(cfg, mask=1), dt)
    o = oracle.run_ex(P, wxy, wz, *model, None, nsteps=nsteps, inj=(pts, 3, t_first, tr), rec=(rec, 3))
    for a, b in zip(g, o[:4]):
        assert np.abs(b).max() > 0
        assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"
    assert list(ids) == list(range(len(rec))) and traces.shape == (nsteps, len(rec), 2)
    assert np.array_equal(traces, o[4])


def test_injection_fp64_matches_oracle():
    from synth import weights as W
    cfg, _, _, dt, model = setup(60, 50, 40, damp=5)
    wxy = W.xy_weights(cfg["r_xy"])
    wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(cfg["nz"], cfg["r_z"], 6.0, 12.0), cfg["r_z"]))
    model = [a.astype(np.float64) for a in model]
    pts = _inj_points(cfg, 40, 7)
    tr = np.random.default_rng(2).normal(size=(30, len(pts)))
    with handle(cfg, dt, wxy, wz, precision=64) as v:
        v.set_model(*model)
        v.set_injection(pts, tr, fields=1)
        v.set_receivers(pts[:10], fields=2, capacity_steps=40)
        v.step(30)
        g = v.get_fields(0)
        _, traces = v.get_traces()
    o = oracle.run_ex(oracle.params(cfg, dt, src=None), wxy, wz, *model, None, nsteps=30,
                      inj=(pts, 1, 0, tr), rec=(pts[:10], 2), dtype=np.float64)
    assert np.array_equal(g[0], o[0]) and np.array_equal(g[1], o[1]) and np.array_equal(traces, o[4])


def test_reverse_with_injection_matches_oracle():
    """The RTM backward leg: record forward, then reverse and re-inject the recorded traces
    (time index decreasing picks the earlier rows), bitwise against vto_run_ex(direction=-1)."""
    cfg, wxy, wz, dt, model = setup(damp=6)
    rec = _inj_points(cfg, 30, 11)
    K = 40
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.set_receivers(rec, fields=1, capacity_steps=K)
        v.step(K)
        _, traces = v.get_traces()
        fwd = v.get_fields(0) + v.get_fields(1)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=0.0)   # source off for the backward leg
        v.set_receivers(np.zeros((0, 3), np.int32))
        v.set_injection(rec, traces[:, :, 0], fields=1, t_first=1)      # row t = level t + 1
        v.reverse()
        v.step(K - 5)
        back = v.get_fields(0) + v.get_fields(1)
    P = oracle.params(cfg, dt)
    o = oracle.run_ex(P, wxy, wz, *model, None, nsteps=K, rec=(rec, 1))
    for a, b in zip(fwd, o[:4]):
        assert np.array_equal(a, b)
    assert np.array_equal(traces, o[4])
    P0 = oracle.params(dict(cfg, amp=0.0), dt)
    b = oracle.run_ex(P0, wxy, wz, *model, (o[2], o[3], o[0], o[1]), n0=K - 1, nsteps=K - 5, direction=-1,
                      inj=(rec, 1, 1, traces[:, :, 0]))
    for a, c in zip(back, b[:4]):
        assert np.array_equal(a, c)


def test_injection_across_slabs():
    from paper_1410_1387_b200 import group_step
    cfg, wxy, wz, dt, model = setup(ny=70, src=(25, 35, 20))
    pts = _inj_points(cfg, 60, 13, extra=[(25, 34, 20), (25, 36, 20), (3, 0, 1), (40, 69, 30)])
    tr = np.random.default_rng(1).normal(size=(12, len(pts))).astype(np.float32)
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.set_injection(pts, tr, fields=3)
        v.step(10)
        ref = v.get_fields(0)
    hs = [handle(cfg, dt, wxy, wz, rank=r, nranks=2) for r in range(2)]
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        h.set_injection(pts, tr, fields=3)
    group_step(hs, 10)
    for h in hs:
        p, q = h.get_fields(0)
        assert np.array_equal(p, ref[0][:, h.y0:h.y0 + h.ny_local])
        assert np.array_equal(q, ref[1][:, h.y0:h.y0 + h.ny_local])
        h.close()


def test_injection_errors():
    from paper_1410_1387_b200 import VTIError
    cfg, wxy, wz, dt, model = setup()
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        for pts, name in (([[1, 1, 1], [1, 1, 1]], "VTI_E_PARAM"), ([[60, 0, 0]], "VTI_E_INDEX")):
            with pytest.raises(VTIError) as e:
                v.set_injection(np.array(pts, np.int32), np.ones((3, len(pts)), np.float32))
            assert e.value.name == name
        with pytest.raises(VTIError) as e:
            v.set_injection([[1, 1, 1]], np.ones((3, 1), np.float32), fields=4)
        assert e.value.name == "VTI_E_PARAM"
        v.set_injection(np.zeros((0, 3), np.int32), None)   # remove: plain kernels again
        v.step(2)


def test_async_snapshots_every_step():
    """vti_snapshot_async: one enqueued copy per step into a device ring (no host sync in the
    loop), equal to the oracle's level after each step; a pageable host buffer is refused."""
    import torch
    from paper_1410_1387_b200 import VTIError
    cfg, wxy, wz, dt, model = setup()
    nsteps = 8
    ring_p = torch.zeros((nsteps, cfg["nz"], cfg["ny"], cfg["nx"]), dtype=torch.float32, device="cuda")
    ring_q = torch.zeros_like(ring_p)
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], mask=3)
        for n in range(nsteps):
            v.step(1)
            v.snapshot_async(ring_p[n], ring_q[n])
        with pytest.raises(VTIError) as e:
            v.snapshot_async(np.zeros((cfg["nz"], cfg["ny"], cfg["nx"]), np.float32))
        assert e.value.name == "VTI_E_PARAM"
        v.sync()
    P = oracle.params(dict(cfg, mask=3), dt)
    st = None
    got_p, got_q = ring_p.cpu().numpy(), ring_q.cpu().numpy()
    for n in range(nsteps):
        st = oracle.run(P, wxy, wz, *model, st, n0=n, nsteps=1)[:4]
        assert np.array_equal(got_p[n], st[0]) and np.array_equal(got_q[n], st[1])
    assert np.abs(got_p[-1]).max() > 0


@pytest.mark.parametrize("grid", [(60, 50, 40), (96, 96, 72)])
def test_dense_surface_injection_and_receivers(grid):
    """A whole plane of injection points and a whole plane of receivers (the RTM surface
    acquisition): dense CSR rows on the small-grid and the persistent kernels, bitwise."""
    cfg, wxy, wz, dt, model = setup(*grid, damp=6, src=(grid[0] // 2, grid[1] // 2, grid[2] // 2))
    nx, ny, nz = grid
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    surface = lambda k: np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, k)], 1).astype(np.int32)
    inj, rec = surface(3), surface(nz - 9)
    nsteps = 40
    tr = (np.random.default_rng(8).normal(size=(nsteps, len(inj))) * 2.0).astype(np.float32)
    with handle(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.set_injection(inj, tr, fields=1)
        v.set_receivers(rec, fields=3, capacity_steps=nsteps)
        v.step(nsteps)
        g = v.get_fields(0)
        _, traces = v.get_traces()
    o = oracle.run_ex(oracle.params(cfg, dt), wxy, wz, *model, None, nsteps=nsteps, inj=(inj, 1, 0, tr), rec=(rec, 3))
    assert np.array_equal(g[0], o[0]) and np.array_equal(g[1], o[1])
    assert np.array_equal(traces, o[4]) and np.abs(traces).max() > 0


def test_async_snapshots_fp64_planes_and_slabs():
    """Snapshots of a plane range in fp64, and per-slab snapshots of a local group (each slab
    snapshots its own rows), equal to the oracle's level after each step."""
    import torch
    from synth import weights as W
    from paper_1410_1387_b200 import group_step
    cfg, _, _, dt, model = setup(60, 50, 40, damp=5)
    wxy = W.xy_weights(cfg["r_xy"])
    wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(cfg["nz"], cfg["r_z"], 6.0, 12.0), cfg["r_z"]))
    m64 = [a.astype(np.float64) for a in model]
    k0, nk, nsteps = 11, 7, 5
    ring = torch.zeros((nsteps, nk, cfg["ny"], cfg["nx"]), dtype=torch.float64, device="cuda")
    with handle(cfg, dt, wxy, wz, precision=64) as v:
        v.set_model(*m64)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        for n in range(nsteps):
            v.step(1)
            v.snapshot_async(ring[n], None, level=0, planes=(k0, nk))
        v.sync()
    P = oracle.params(cfg, dt)
    st = None
    for n in range(nsteps):
        st = oracle.run(P, wxy, wz, *m64, st, n0=n, nsteps=1, dtype=np.float64)[:4]
        assert np.array_equal(ring[n].cpu().numpy(), st[0][k0:k0 + nk])
    # two slabs, fp32: each snapshots its own rows of u^n after the group's steps
    wxy32, wz32 = wxy.astype(np.float32), wz.astype(np.float32)
    hs = [handle(cfg, dt, wxy32, wz32, rank=r, nranks=2) for r in range(2)]
    outs = []
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
    group_step(hs, 6)
    for h in hs:
        buf = torch.zeros((cfg["nz"], h.ny_local, cfg["nx"]), dtype=torch.float32, device="cuda")
        h.snapshot_async(buf, None)
        h.sync()
        outs.append(buf.cpu().numpy())
        h.close()
    o = oracle.run(oracle.params(cfg, dt), wxy32, wz32, *model, None, nsteps=6)[0]
    assert np.array_equal(np.concatenate(outs, axis=1), o)
