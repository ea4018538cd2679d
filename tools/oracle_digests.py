#!/usr/bin/env python
"""Write tests/golden/oracle_digests.json: the CPU oracle's fields after the stated step count
of BASELINE.json's configurations (north_star: "GPU fields must match the oracle ... after the
stated step count"; "integrated in time for a thousand time steps").

Calls only oracle/ and synth/ (never the CUDA path). For each workload -- the bench's start:
the seeded synthetic model, zero initial state, the Ricker source at the centre (SURVEY.md
8(d) recipe) -- it runs the oracle for the config's steps and stores the sha256 of the raw
little-endian bytes (user layout [z][y][x], x fastest) of u^N = (p, q) and of the stored
u^{N-1} (pm, qm), plus the digests of the three model arrays so that a GPU-side generator
mismatch is diagnosed separately, and a few scalar summaries. tests/test_digests_gpu.py steps
the library the same N steps and compares digests (bitwise parity).

  python tools/oracle_digests.py [C2 N1 C3 C5] [--threads T] [--out PATH]

Runtime on 8 host cores: roughly 0.5-1.5 h per config (x86 subnormal arithmetic in the
decaying far field dominates); each config is merged into the JSON as soon as it finishes.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import fields as SF  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_digests.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<f4", copy=False).tobytes()).hexdigest()


def host_model(cfg, chunk=32):
    """The synth model on the host, generated plane-chunk by plane-chunk into preallocated arrays."""
    shape = (cfg["nz"], cfg["ny"], cfg["nx"])
    out = [np.empty(shape, np.float32) for _ in range(3)]
    for k0 in range(0, cfg["nz"], chunk):
        nk = min(chunk, cfg["nz"] - k0)
        for dst, src in zip(out, SF.model_planes(cfg, k0, nk, device="cpu")):
            dst[k0:k0 + nk] = src.numpy()
    return out


def run_one(name: str, threads: int) -> dict:
    cfg = synth.CONFIGS[name]()
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    nsteps = cfg["steps"]
    t0 = time.time()
    model = host_model(cfg)
    t_model = time.time() - t0
    mdig = [sha(a) for a in model]
    p, q, pm, qm, secs = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, None, nsteps=nsteps,
                                    nthreads=threads)
    del model
    ent = {
        "grid": [cfg["nx"], cfg["ny"], cfg["nz"]], "r_xy": cfg["r_xy"], "r_z": cfg["r_z"],
        "steps": nsteps, "dt": dt, "src": list(cfg["src"]), "t0": cfg["t0"], "mask": cfg["mask"],
        "start": "zero state (u^0 = u^-1 = 0), Ricker source at cfg['src'] (bench.py's workload)",
        "model_sha256": {"vx2": mdig[0], "vn2": mdig[1], "vz2": mdig[2]},
        "sha256": {"p": sha(p), "q": sha(q), "pm": sha(pm), "qm": sha(qm)},
        "max_abs": {"p": float(np.abs(p).max()), "q": float(np.abs(q).max())},
        "l2": {"p": float(np.linalg.norm(p.astype(np.float64))), "q": float(np.linalg.norm(q.astype(np.float64)))},
        "oracle_seconds": round(secs, 1), "model_seconds": round(t_model, 1), "threads": threads,
        "host": platform.processor() or platform.machine(),
    }
    return ent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["C2", "C3", "C5", "N1"])
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=OUT, help="JSON to merge the entries into (default tests/golden/...)")
    a = ap.parse_args()
    oracle.build()
    for name in a.names:
        ent = run_one(name, a.threads or oracle.max_threads())
        out = a.out
        d = json.load(open(out)) if os.path.exists(out) else {
            "what": "sha256 of the oracle's float32 fields after each config's stated step count",
            "written_by": "tools/oracle_digests.py (oracle/ + synth/ only)"}
        d[name] = ent
        tmp = out + ".tmp"
        with open(tmp, "w") as f:
            json.dump(d, f, indent=1)
        os.replace(tmp, out)
        print(name, json.dumps(ent), flush=True)


if __name__ == "__main__":
    main()
