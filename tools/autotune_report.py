#!/usr/bin/env python
"""vti_autotune on a BASELINE workload: which compiled variant x z-chunk is fastest on this
GPU, next to the library default (bench.py's schedule).  python tools/autotune_report.py C5"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from synth import fields as SF  # noqa: E402
from paper_1410_1387_b200 import VTI  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = synth.CONFIGS[name]()
wxy, wz, _ = synth.weights_f32(cfg)
dt = synth.stable_dt(cfg, wxy, wz)
h = VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
        damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"])
for k0 in range(0, cfg["nz"], 64):
    h.set_model_planes(k0, *[a.contiguous() for a in SF.model_planes(cfg, k0, min(64, cfg["nz"] - k0), device="cuda")])
npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
default = {k: h.info()[k] for k in ("tile_y", "producer_warp", "rows_per_thread", "points_per_thread", "zchunk", "grid")}
h.step(3)
ms = h.step_timed(20) / 20
h.close()
h = VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
        damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"])
for k0 in range(0, cfg["nz"], 64):
    h.set_model_planes(k0, *[a.contiguous() for a in SF.model_planes(cfg, k0, min(64, cfg["nz"] - k0), device="cuda")])
res = h.autotune(probe_steps=5)
h.close()
print(json.dumps({"config": name, "default": dict(default, gpoints_s=round(npts / (ms * 1e-3) / 1e9, 1)),
                  "autotune": dict(res, gpoints_s=round(npts / (res["ms_per_step"] * 1e-3) / 1e9, 1))}))
