"""SURVEY.md 8(f) N4 hooks: receiver traces and time reversal, against the oracle."""
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
