"""GPU tests of the fused peer-memory halo transport.

The edge launch of a y-slab stores p^{n+1} of its first / last R_xy rows into
the neighbours' halo rows itself (a separate PEER instantiation of every
compiled variant), and stream flag operations order the steps. A local group
(several handles in one process on cuda:0) runs exactly that protocol with the
neighbours' own buffers as peer memory, so every case here is a multi-slab run
compared bitwise with the single-domain oracle (or, for time reversal, with the
single-slab library run that tests/test_n4_gpu.py pins to the oracle).
"""
import os
import re

import numpy as np
import pytest

import oracle
import synth
from synth import fields as SF

from test_parity_gpu import random_state, small_cfg

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def compiled_variants():
    """(precision, r, rz, ty, wp, rpt, px) of every entry<...> in csrc/variants/*.cu."""
    out = []
    d = os.path.join(ROOT, "paper_1410_1387_b200", "csrc", "variants")
    for f in sorted(os.listdir(d)):
        if f.endswith(".cu"):
            src = open(os.path.join(d, f)).read()
            pat = r"entry(?:_io)?<(float|double),\s*(\d+),\s*(\d+),\s*(\d+),\s*(\d+),\s*(\d+),\s*\d+,\s*\d+(?:,\s*(\d+))?>"
            for m in re.finditer(pat, src):
                t, r, rz, ty, rpt, wp, px = m.groups()
                out.append((32 if t == "float" else 64, int(r), int(rz), int(ty), int(wp), int(rpt), int(px or 4)))
    return out


def handles(cfg, dt, wxy, wz, nranks, precision=32):
    from paper_1410_1387_b200 import VTI
    return [VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
                damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0, rank=r, nranks=nranks,
                precision=precision) for r in range(nranks)]


def load(hs, model, state=None, n0=0, cfg=None):
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        if state is not None:
            h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in state], time_index=n0)
        if cfg is not None:
            h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])


def gather(hs):
    parts = [h.get_fields(0) + h.get_fields(1) for h in hs]
    return [np.concatenate([p[f] for p in parts], axis=1) for f in range(4)]


def close(hs):
    for h in hs:
        h.close()


def f32_inputs(cfg, seed=7):
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    return wxy, wz, dt, model, random_state(cfg, seed=seed, amp=1e-4)


def f64_inputs(cfg, seed=7):
    from test_fp64_gpu import inputs, weights64
    wxy, wz = weights64(cfg)
    model, st = inputs(cfg, seed=seed)
    return wxy, wz, synth.stable_dt(cfg), tuple(model), st


@pytest.mark.parametrize("prec,r,rz,ty,wp,rpt,px", compiled_variants())
def test_every_peer_instantiation(prec, r, rz, ty, wp, rpt, px):
    """3 slabs (source on a slab boundary, interior tile rows present) in every compiled
    variant: the PEER edge instantiation and the plain interior one, bitwise == oracle."""
    ny = 3 * max(2 * ty + 2 * r, 40)
    cfg = small_cfg(70, ny, 2 * rz + 12, r, rz, damp=5)
    cfg["src"] = (30, ny // 3, cfg["nz"] // 2)   # first row of rank 1
    wxy, wz, dt, model, st = (f64_inputs if prec == 64 else f32_inputs)(cfg)
    hs = handles(cfg, dt, wxy, wz, 3, prec)
    for h in hs:
        h.set_variant(ty, wp, rpt, px)
        info = h.info()
        assert (info["tile_y"], info["producer_warp"], info["rows_per_thread"], info["points_per_thread"]) == \
            (ty, wp, rpt, px)
    load(hs, model, st, 2, cfg)
    from paper_1410_1387_b200 import group_step
    group_step(hs, 5)
    got = gather(hs)
    assert hs[1].halo_transport == "peer"
    close(hs)
    P = oracle.params(cfg, dt)
    ref = oracle.run(P, wxy, wz, *model, st, n0=2, nsteps=5, dtype=np.float64 if prec == 64 else np.float32)[:4]
    for f in range(4):
        assert np.abs(ref[f]).max() > 0
        assert np.array_equal(got[f], ref[f]), f"field {f}"


@pytest.mark.parametrize("r,rz,ny,nranks", [(8, 4, 40, 4), (12, 8, 39, 3), (4, 4, 30, 5)])
def test_slabs_thinner_than_two_radii(r, rz, ny, nranks):
    """nyl < 2R: a boundary row is in both neighbours' halos (stored to both sides)."""
    from paper_1410_1387_b200 import group_step
    cfg = small_cfg(64, ny, 2 * rz + 8, r, rz, damp=3, src=(20, ny // 2, rz + 4))
    wxy, wz, dt, model, st = f32_inputs(cfg)
    hs = handles(cfg, dt, wxy, wz, nranks)
    assert all(r <= h.ny_local < 2 * r for h in hs)
    load(hs, model, st, 0, cfg)
    group_step(hs, 4)
    group_step(hs, 3)
    got = gather(hs)
    close(hs)
    ref = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=7)[:4]
    for f in range(4):
        assert np.array_equal(got[f], ref[f]), f"field {f}"


def test_set_fields_mid_run_republishes():
    """Steps, then a new state from the caller (halos re-published after the last step's
    publication was abandoned), then more steps: bitwise == oracle from the new state."""
    from paper_1410_1387_b200 import group_step
    cfg = small_cfg(70, 90, 30, 4, 4, damp=5, src=(30, 45, 15))
    wxy, wz, dt, model, st = f32_inputs(cfg)
    hs = handles(cfg, dt, wxy, wz, 3)
    load(hs, model, st, 0, cfg)
    group_step(hs, 3)
    st2 = random_state(cfg, seed=11, amp=1e-4)
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st2], time_index=3)
    group_step(hs, 4)
    got = gather(hs)
    close(hs)
    ref = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st2, n0=3, nsteps=4)[:4]
    for f in range(4):
        assert np.array_equal(got[f], ref[f]), f"field {f}"


def test_reverse_in_a_group_equals_single_slab():
    """Forward, vti_reverse (re-publication of the swapped level), backward: the group run
    equals the single-slab run of the same calls bitwise."""
    from paper_1410_1387_b200 import group_step
    cfg = small_cfg(70, 80, 30, 4, 4, damp=5, src=(30, 40, 15))
    wxy, wz, dt, model, st = f32_inputs(cfg)
    (one,) = handles(cfg, dt, wxy, wz, 1)
    load([one], model, st, 0, cfg)
    one.step(6)
    one.reverse()
    one.step(4)
    ref = one.get_fields(0) + one.get_fields(1)
    one.close()
    hs = handles(cfg, dt, wxy, wz, 2)
    load(hs, model, st, 0, cfg)
    group_step(hs, 6)
    for h in hs:
        h.reverse()
    group_step(hs, 4)
    got = gather(hs)
    close(hs)
    for f in range(4):
        assert np.array_equal(got[f], ref[f]), f"field {f}"


def test_yzx_layout_group(monkeypatch):
    """The [y][z][x] layout: different row / plane strides for the peer stores and the
    re-publication copy."""
    from paper_1410_1387_b200 import group_step
    monkeypatch.setenv("VTI_LAYOUT", "yzx")
    cfg = small_cfg(70, 75, 26, 4, 4, damp=5, src=(30, 37, 13))
    wxy, wz, dt, model, st = f32_inputs(cfg)
    hs = handles(cfg, dt, wxy, wz, 3)
    assert hs[0].info()["layout"] == 1
    load(hs, model, st, 0, cfg)
    group_step(hs, 5)
    got = gather(hs)
    close(hs)
    ref = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=5)[:4]
    for f in range(4):
        assert np.array_equal(got[f], ref[f]), f"field {f}"


def test_peer_group_launches_two_kernels_per_step():
    cfg = small_cfg(70, 450, 26, 4, 4, damp=5, src=(30, 100, 13))   # 150-row slabs: edge + interior
    wxy, wz, dt, model, st = f32_inputs(cfg)
    hs = handles(cfg, dt, wxy, wz, 3)
    # local groups default to the edge + interior pair; VTI_FUSED_STEP=1 forces one fused launch
    expect = 1 if os.environ.get("VTI_FUSED_STEP", "") == "1" else 2
    assert [h.info()["launches_per_step"] for h in hs] == [expect] * 3
    close(hs)


def test_group_check_every_detects_instability():
    """check_every also runs in a local group: a blow-up is reported as VTI_E_INSTABILITY."""
    from paper_1410_1387_b200 import VTI, VTIError, group_step
    cfg = small_cfg(70, 80, 30, 4, 4, damp=5, src=(30, 40, 15))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = 5 * synth.stable_dt(cfg, wxy, wz)   # far beyond the CFL bound
    model = tuple(a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"]))
    hs = [VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], 4, 4, dt, wxy, wz, damp_width=cfg["damp_width"],
              damp_alpha=cfg["damp_alpha"], rank=r, nranks=2, check_every=25) for r in range(2)]
    load(hs, model, random_state(cfg, amp=1.0), 0, cfg)
    with pytest.raises(VTIError) as e:
        group_step(hs, 2000)
    assert e.value.name == "VTI_E_INSTABILITY"
    close(hs)


@pytest.mark.parametrize("nranks,ty,r,rz", [(2, 32, 4, 4), (3, 16, 4, 4), (3, 30, 12, 8), (4, 32, 8, 4)])
def test_fused_step_bitwise(nranks, ty, r, rz, monkeypatch):
    """The fused one-launch peer step (edge items first, the last edge CTA raises the
    neighbours' flags from the device; the default of a multi-process rank), forced in a
    local group: bitwise == oracle, across a re-publication and a reverse."""
    from paper_1410_1387_b200 import group_step
    monkeypatch.setenv("VTI_FUSED_STEP", "1")
    ny = nranks * 70
    cfg = small_cfg(70, ny, 2 * rz + 12, r, rz, damp=5)
    cfg["src"] = (30, ny // nranks, cfg["nz"] // 2)   # first row of rank 1
    wxy, wz, dt, model, st = f32_inputs(cfg)
    hs = handles(cfg, dt, wxy, wz, nranks)
    for h in hs:
        h.set_variant(ty, -1, -1, -1)
    assert all(h.info()["launches_per_step"] == 1 for h in hs)
    load(hs, model, st, 0, cfg)
    group_step(hs, 4)
    group_step(hs, 3)
    got = gather(hs)
    ref = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=7)[:4]
    for f in range(4):
        assert np.array_equal(got[f], ref[f]), f"field {f}"
    # a state from the caller (re-publication), then reverse: equals the same calls on one slab
    st2 = random_state(cfg, seed=13, amp=1e-4)
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st2], time_index=7)
    group_step(hs, 3)
    for h in hs:
        h.reverse()
    group_step(hs, 2)
    got2 = gather(hs)
    close(hs)
    (one,) = handles(cfg, dt, wxy, wz, 1)
    load([one], model, st2, 7, cfg)
    one.step(3)
    one.reverse()
    one.step(2)
    ref2 = one.get_fields(0) + one.get_fields(1)
    one.close()
    for f in range(4):
        assert np.array_equal(got2[f], ref2[f]), f"field {f}"


@pytest.mark.parametrize("prec,r,rz,nranks", [(32, 4, 4, 2), (32, 8, 4, 3), (64, 6, 6, 3), (32, 12, 8, 2)])
def test_staged_transport_matches_oracle(prec, r, rz, nranks):
    """The NCCL path's staged transport -- edge launch, pack of the boundary rows, exchange on
    the comm stream (device copies standing in for ncclSend/ncclRecv), unpack into the halo
    rows, interior launch overlapped -- in a local group: bitwise == oracle, including a
    state set mid-run (its halo re-exchanged before the next step)."""
    from paper_1410_1387_b200 import group_step
    ny = nranks * 40
    cfg = small_cfg(70, ny, 2 * rz + 14, r, rz, damp=5)
    cfg["src"] = (30, ny // nranks, cfg["nz"] // 2)   # first row of rank 1
    wxy, wz, dt, model, st = (f64_inputs if prec == 64 else f32_inputs)(cfg)
    dtype = np.float64 if prec == 64 else np.float32
    hs = handles(cfg, dt, wxy, wz, nranks, prec)
    load(hs, model, st, 2, cfg)
    group_step(hs, 4, transport="staged")
    mid = gather(hs)
    P = oracle.params(cfg, dt)
    ref = oracle.run(P, wxy, wz, *model, st, n0=2, nsteps=4, dtype=dtype)[:4]
    for f in range(4):
        assert np.array_equal(mid[f], ref[f]), f"field {f} after 4 steps"
    # a new state mid-run: halos must be re-exchanged (pack of the current level) before stepping
    st2 = [np.ascontiguousarray(a[::-1]) for a in st]
    load(hs, model, st2, 9)
    group_step(hs, 3, transport="staged")
    got = gather(hs)
    close(hs)
    ref2 = oracle.run(P, wxy, wz, *model, st2, n0=9, nsteps=3, dtype=dtype)[:4]
    for f in range(4):
        assert np.abs(ref2[f]).max() > 0
        assert np.array_equal(got[f], ref2[f]), f"field {f} after the reset"


def test_staged_transport_with_receivers_and_injection():
    from paper_1410_1387_b200 import group_step
    cfg = small_cfg(70, 96, 20, 4, 4, damp=5)
    cfg["src"] = (30, 48, 10)
    wxy, wz, dt, model, st = f32_inputs(cfg)
    pts = np.array([[30, 47, 10], [30, 48, 10], [5, 0, 0], [69, 95, 19], [12, 50, 3]], np.int32)
    tr = np.random.default_rng(3).normal(size=(6, len(pts))).astype(np.float32)
    hs = handles(cfg, dt, wxy, wz, 2)
    load(hs, model, st, 0, cfg)
    for h in hs:
        h.set_injection(pts, tr, fields=3)
        h.set_receivers(pts, fields=1, capacity_steps=10)
    group_step(hs, 6, transport="staged")
    got = gather(hs)
    traces = np.zeros((6, len(pts), 1), np.float32)
    for h in hs:
        ids, t = h.get_traces()
        traces[:, ids] = t
    close(hs)
    o = oracle.run_ex(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=6, inj=(pts, 3, 0, tr), rec=(pts, 1))
    for f in range(4):
        assert np.array_equal(got[f], o[f])
    assert np.array_equal(traces, o[4])


@pytest.mark.parametrize("nranks", [2, 3])
def test_fused_step_with_point_sets(nranks, monkeypatch):
    """The fused one-launch peer step (the multi-process default) with trace injection and
    receivers: its PEER + IO instantiation, bitwise == oracle (vto_run_ex)."""
    from paper_1410_1387_b200 import group_step
    monkeypatch.setenv("VTI_FUSED_STEP", "1")
    ny = nranks * 64
    cfg = small_cfg(70, ny, 20, 4, 4, damp=5)
    cfg["src"] = (30, ny // nranks, 10)
    wxy, wz, dt, model, st = f32_inputs(cfg)
    rng = np.random.default_rng(nranks)
    pts = {(30, ny // nranks - 1, 10), (30, ny // nranks, 10), (0, 0, 0), (69, ny - 1, 19)}
    while len(pts) < 40:
        pts.add((int(rng.integers(70)), int(rng.integers(ny)), int(rng.integers(20))))
    pts = np.array(sorted(pts), np.int32)
    tr = rng.normal(size=(8, len(pts))).astype(np.float32)
    hs = handles(cfg, dt, wxy, wz, nranks)
    load(hs, model, st, 0, cfg)
    for h in hs:
        h.set_injection(pts, tr, fields=3)
        h.set_receivers(pts, fields=3, capacity_steps=8)
    group_step(hs, 8)
    assert all(h.info()["launches_per_step"] == 1 for h in hs)
    got = gather(hs)
    traces = np.zeros((8, len(pts), 2), np.float32)
    for h in hs:
        ids, t = h.get_traces()
        traces[:, ids] = t
    close(hs)
    o = oracle.run_ex(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=8, inj=(pts, 3, 0, tr), rec=(pts, 3))
    for f in range(4):
        assert np.array_equal(got[f], o[f]), f"field {f}"
    assert np.array_equal(traces, o[4])
