#!/usr/bin/env python
"""Throughput of vti_step_adjoint (the transpose recurrence, N4) on a BASELINE grid, CUDA events
around K adjoint steps (after W warm-up steps); the forward step on the same handle for scale.

  python tools/adjoint_rate.py [--config C2] [--steps 20] [--warmup 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import synth
    from synth import fields as SF
    from paper_1410_1387_b200 import VTI
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", type=int, default=32, choices=[32, 64])
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]()
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    if a.precision == 64:
        from synth import weights as W
        wxy = W.xy_weights(cfg["r_xy"])
        wz = W.z_weights(W.z_coords_ramp(cfg["nz"], cfg["r_z"], cfg["dz"][0], cfg["dz"][1]), cfg["r_z"])
    npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
    with VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
             damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=0, precision=a.precision) as v:
        for k0 in range(0, cfg["nz"], 32):
            m = SF.model_planes(cfg, k0, min(32, cfg["nz"] - k0), device="cuda")
            v.set_model_planes(k0, *[(x.double() if a.precision == 64 else x).contiguous() for x in m])
        torch.cuda.synchronize()
        v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"])
        v.step(a.warmup)
        fwd_ms = v.step_timed(a.steps)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.ExternalStream(v.stream)
        v.step_adjoint(a.warmup)
        v.sync()
        s0.record(stream)
        v.step_adjoint(a.steps)
        s1.record(stream)
        s1.synchronize()
        adj_ms = s0.elapsed_time(s1)
    out = {"config": a.config, "precision": a.precision, "grid": [cfg["nx"], cfg["ny"], cfg["nz"]], "steps": a.steps,
           "forward_gpoints_s": round(npts * a.steps / (fwd_ms * 1e-3) / 1e9, 2),
           "adjoint_gpoints_s": round(npts * a.steps / (adj_ms * 1e-3) / 1e9, 2),
           "adjoint_ms_per_step": round(adj_ms / a.steps, 4),
           "adjoint_algorithmic_bytes_per_point": 9 * a.precision // 8,
           "note": "bytes per point = the forward step's 36 (72); the one-pass adjoint reads psi, vx2, vn2, "
                   "vz2, psi^{m+1} and writes psi^{m-1}, the two-pass form adds s1 / s2 (60 / 120 B per point)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
