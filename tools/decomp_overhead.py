#!/usr/bin/env python
"""Cost of the y-slab decomposition on ONE GPU (not a scaling number).

Runs the C2 grid as 1, 2 and 4 local-group slabs in one process on cuda:0
(vti_group_step: edge tile rows, pack, device-to-device halo copy, unpack,
interior rows -- the same schedule as the NCCL path with a copy transport)
and prints Gpoints/s for each, so the overhead of the multi-slab step itself
(extra launches, edge/interior split, halo traffic) is visible.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from synth import fields as SF  # noqa: E402
from paper_1410_1387_b200 import VTI, group_step  # noqa: E402


def run(cfg, nslabs, steps, warmup):
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    hs = [VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
              damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], rank=r, nranks=nslabs)
          for r in range(nslabs)]
    for h in hs:
        for k0 in range(0, cfg["nz"], 64):
            nk = min(64, cfg["nz"] - k0)
            m = SF.model_planes(cfg, k0, nk, device="cuda", j0=h.y0, nyl=h.ny_local)
            h.set_model_planes(k0, *[a.contiguous() for a in m])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
    step = (lambda n: hs[0].step(n)) if nslabs == 1 else (lambda n: group_step(hs, n))
    step(warmup)
    for h in hs:
        h.sync()
    t0 = time.perf_counter()
    step(steps)
    for h in hs:
        h.sync()
    t = time.perf_counter() - t0
    info = hs[0].info()
    for h in hs:
        h.close()
    torch.cuda.empty_cache()
    return cfg["nx"] * cfg["ny"] * cfg["nz"] * steps / t / 1e9, info


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = synth.CONFIGS[name]()
    out = {}
    for n in (1, 2, 4):
        v, info = run(cfg, n, 200, 10)
        out[n] = {"gpoints_s": round(v, 2), "rank0_launches_per_step": info["launches_per_step"]}
        print(n, out[n], flush=True)
    print(json.dumps({"config": name, "slabs_on_one_gpu": out}))
