#!/usr/bin/env python
"""Cost of the y-slab decomposition on ONE GPU (not a scaling number).

Default: the C2 grid split into 1, 2 and 4 local-group slabs in one process
on cuda:0. --weak: n slabs of the full C2 ny each (grid nx x n*ny x nz, the
bench's weak-scaling workload per GPU), n = 1, 2, 4, 8.

Both run vti_group_step, i.e. the multi-GPU step schedule: edge tile rows with
the fused peer stores into the neighbours' halo rows, flag waits and writes,
then the interior rows. They print Gpoints/s, so the overhead of the
multi-slab step itself is visible: extra launch, edge/interior split, halo
stores. NVLink and the other GPUs are not part of it.
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
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    weak = "--weak" in sys.argv
    name = args[0] if args else "C2"
    slabs = tuple(int(x) for x in args[1].split(",")) if len(args) > 1 else ((1, 2, 4, 8) if weak else (1, 2, 4))
    steps = int(args[2]) if len(args) > 2 else 200
    base = synth.CONFIGS[name]()
    out = {}
    for n in slabs:
        cfg = base
        if weak:   # the bench's weak-scaling workload: n slabs of the base ny rows each
            cfg = synth.scaled(base, base["nx"], base["ny"] * n, base["nz"])
            cfg["src"] = base["src"]
        v, info = run(cfg, n, steps if not weak else max(25, steps // n), 5)
        out[n] = {"gpoints_s": round(v, 2), "rank0_launches_per_step": info["launches_per_step"]}
        if 1 in out:
            out[n]["vs_1_slab"] = round(v / out[1]["gpoints_s"], 4)
        print(n, out[n], flush=True)
    print(json.dumps({"config": name, "mode": "weak (n slabs of ny rows)" if weak else "split one grid",
                      "slabs_on_one_gpu": out}))
