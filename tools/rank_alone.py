#!/usr/bin/env python
"""One rank's slab timed alone on one GPU: the config's recipe on an nx x ny x nz grid
with ny = the slab height a rank owns at N GPUs. With VTI_FORCE_SPLIT=1 the single
slab runs the multi-GPU two-launch schedule (edge tile rows, then interior; no
transport), so comparing the two runs and the full grid gives the per-GPU schedule
efficiency of strong scaling, before NVLink effects.

  VTI_FORCE_SPLIT=1 python tools/rank_alone.py C4 256 30     # C4 at 8 GPUs
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from synth import fields as SF  # noqa: E402
from paper_1410_1387_b200 import VTI  # noqa: E402

name, ny = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
base = synth.CONFIGS[name]()
cfg = synth.scaled(base, base["nx"], ny, base["nz"])
wxy, wz, _ = synth.weights_f32(cfg)
dt = synth.stable_dt(cfg, wxy, wz)
h = VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
        damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"])
for k0 in range(0, cfg["nz"], 64):
    nk = min(64, cfg["nz"] - k0)
    h.set_model_planes(k0, *[a.contiguous() for a in SF.model_planes(cfg, k0, nk, device="cuda")])
h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
h.step(3)
h.sync()
ms = h.step_timed(steps)
print(name, ny, "split" if os.environ.get("VTI_FORCE_SPLIT", "0") != "0" else "single",
      round(cfg["nx"] * ny * cfg["nz"] * steps / (ms * 1e-3) / 1e9, 2), flush=True)
h.close()
