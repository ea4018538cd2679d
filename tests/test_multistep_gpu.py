"""The multi-step small-grid kernel (vti_small_multi_kernel, opt-in with VTI_MULTI=1): one
cooperative launch advances a whole vti_step call, every CTA owning one (tile, plane) item and waiting only for its exchange
partners' per-item epoch counters between steps. Bitwise against the oracle: BASELINE C1 at its
stated 100 steps, ragged grids with several x tiles for every radius pair, chunked launches
(> 1024 steps), time reversal, interleaving with one-step launches, and the default path."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth
from synth import fields as SF

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _multi_on(monkeypatch):
    monkeypatch.setenv("VTI_MULTI", "1")   # read by vti_create


def make(cfg, dt, wxy, wz):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0)


def inputs(cfg):
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    model = [a.numpy() for a in SF.model_planes(cfg, 0, cfg["nz"])]
    return wxy, wz, dt, model


def test_c1_stated_100_steps():
    cfg = synth.CONFIGS["C1"]()
    wxy, wz, dt, model = inputs(cfg)
    with make(cfg, dt, wxy, wz) as v:
        info = v.info()
        assert info["small_kernel"] == 1 and info["steps_per_launch"] > 1
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        v.step(cfg["steps"])
        g = v.get_fields(0) + v.get_fields(1)
    o = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, None, nsteps=cfg["steps"])[:4]
    for a, b in zip(g, o):
        assert np.abs(b).max() > 0
        assert np.array_equal(a, b)


@pytest.mark.parametrize("r,rz", [(4, 4), (8, 4), (6, 6)])
def test_ragged_multi_tile_grids(r, rz):
    """3 x tiles (130 wide), ragged y and z, source near a tile corner, random start state."""
    cfg = synth.scaled(synth.CONFIGS["C2"](), 130, 45, 2 * rz + 11, r_xy=r, r_z=rz, damp_width=5,
                       dz=(6.0, 12.0), t0=0.02, src=(64, 16, rz + 2))
    wxy, wz, dt, model = inputs(cfg)
    st = [SF.random_planes(cfg["nx"], cfg["ny"], 0, cfg["nz"], 4, s, 1e-3).numpy() for s in range(4)]
    with make(cfg, dt, wxy, wz) as v:
        assert v.info()["steps_per_launch"] > 1
        v.set_model(*model)
        v.set_fields(*st, time_index=3)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], mask=3)
        v.step(37)
        v.step(1)      # a one-step launch in between
        v.step(12)
        g = v.get_fields(0) + v.get_fields(1)
    o = oracle.run(oracle.params(dict(cfg, mask=3), dt), wxy, wz, *model, st, n0=3, nsteps=50)[:4]
    for a, b in zip(g, o):
        assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max():.3e}"


def test_chunked_launches_and_reverse():
    cfg = synth.scaled(synth.CONFIGS["C2"](), 32, 28, 24, damp_width=6, dz=(6.0, 12.0), t0=0.02)
    wxy, wz, dt, model = inputs(cfg)
    with make(cfg, dt, wxy, wz) as v:
        v.set_model(*model)
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.step(1100)   # two launches (1024 + 76)
        fwd = v.get_fields(0) + v.get_fields(1)
        v.reverse()
        v.step(30)
        back = v.get_fields(0) + v.get_fields(1)
    P = oracle.params(cfg, dt)
    o = oracle.run(P, wxy, wz, *model, None, nsteps=1100)[:4]
    for a, b in zip(fwd, o):
        assert np.array_equal(a, b)
    r = oracle.run_ex(P, wxy, wz, *model, (o[2], o[3], o[0], o[1]), n0=1099, nsteps=30, direction=-1)[:4]
    for a, b in zip(back, r):
        assert np.array_equal(a, b)


def test_default_path_matches():
    """Without VTI_MULTI (CUDA-graph replays of the one-step kernel) the same bits."""
    code = (
        "import numpy as np, synth, oracle\n"
        "from synth import fields as SF\n"
        "from paper_1410_1387_b200 import VTI\n"
        "cfg = synth.CONFIGS['C1']()\n"
        "wxy, wz, _ = synth.weights_f32(cfg); dt = synth.stable_dt(cfg, wxy, wz)\n"
        "m = [a.numpy() for a in SF.model_planes(cfg, 0, 64)]\n"
        "v = VTI(64, 64, 64, cfg['h'], 4, 4, dt, wxy, wz, damp_width=20, device=0)\n"
        "assert v.info()['steps_per_launch'] == 1\n"
        "v.set_model(*m); v.add_source(32, 32, 32, f=15.0, t0=0.0); v.step(70)\n"
        "p, q = v.get_fields(0)\n"
        "o = oracle.run(oracle.params(cfg, dt), wxy, wz, *m, None, nsteps=70)\n"
        "assert np.array_equal(p, o[0]) and np.array_equal(q, o[1])\n"
        "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("VTI_MULTI", None)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
