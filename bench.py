#!/usr/bin/env python
"""Benchmark: VTI time steps per second on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl native|reference]

One "step" = one time step of the reduced elastic VTI propagator (PAPER.md
Eqs. 1-3) over the whole grid: every row of SURVEY.md 8(a) runs inside the
fused sm_100a kernel (plus, for N > 1, the NCCL halo exchange of p).

Workload (N = 1): BASELINE.json configs[1] = C2, 512^3, R_xy = R_z = 4,
layered VTI with variable dz, Cerjan W = 20, Ricker source at the centre,
starting from the zero state. N > 1: weak scaling, one 512^3 C2 block per GPU
stacked along y (global 512 x 512N x 512), one y-slab per rank, NCCL halo
exchange of p every step. Inputs (4.8 GB/step at N = 1) are far larger than
the 126 MB L2, so no explicit flush is needed between steps.

Metric: Gpoints/s = (global grid points) x K / t, t = max over ranks of the
CUDA-event time of the K steps on the library's stream. ``roofline`` uses
36 algorithmic bytes per point-update against the measured
HBM copy bandwidth in MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_POINT = 36   # reads p^n, q^n, p^{n-1}, q^{n-1}, vx2, vn2, vz2; writes p^{n+1}, q^{n+1}
METRIC = "Gpoints/s per VTI step (1/2/4/8 B200) and % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5", "N1"])
    ap.add_argument("--scaling", default=None, choices=[None, "weak", "strong"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--zchunk", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--precision", type=int, default=32, choices=[32, 64],
                    help="64 = the fp64 path (SURVEY.md 8(f) N3, 72 B/point)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload(args, world):
    import synth
    base = synth.CONFIGS[args.config]() if args.config != "C5" else synth.CONFIGS["C5"](world)
    # C3 = y-slabs of 1024/G rows and C4 = strong scaling (fixed grid); C2 = 512^3
    # per GPU and C5 = 1024 x 1024G x 1024 (weak)
    scaling = args.scaling or ("strong" if args.config in ("C3", "C4") else "weak")
    if world > 1 and scaling == "weak" and args.config != "C5":
        cfg = synth.scaled(base, base["nx"], base["ny"] * world, base["nz"])
    else:
        cfg = dict(base)
    return cfg, scaling


def describe(cfg, world, scaling, bpp=BYTES_PER_POINT, transport="none"):
    return {
        "workload": f"{cfg['name']}: {cfg['nx']}x{cfg['ny']}x{cfg['nz']} global, R_xy={cfg['r_xy']} R_z={cfg['r_z']}, "
                    f"{cfg['model']['kind']} VTI, W={cfg['damp_width']}, Ricker f={cfg['f']:g} Hz at the centre",
        "grid": [cfg["nx"], cfg["ny"], cfg["nz"]],
        "r_xy": cfg["r_xy"], "r_z": cfg["r_z"], "config_steps": cfg["steps"],
        "decomposition": f"y-slabs x{world}" if world > 1 else "single GPU",
        "halo_transport": transport,
        "scaling": scaling,
        "l2_flush": f"not needed: per-step working set ({bpp} B/pt) >> 126 MB L2",
        "bytes_per_point": bpp,
    }


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9 and f[1].isdigit():
                    rows.append(f)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.remove(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(int(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace('.', '', 1).isdigit())}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def mix_ceiling():
    """Best streaming rate of the step's own DRAM mix (7 streams read, 2 written), measured by
    tools/stream_probe.cu (plain loads) and tools/stream_probe_bulk.cu (TMA bulk loads, the way
    the kernel moves data) -- profiles/stream_probe*_r01.txt: the practical ceiling of this
    kernel, above the 1:1 copy figure of MEASURED_PEAKS.json. Context for roofline.frac > 1."""
    import glob
    import re
    vals = []
    for p in glob.glob(os.path.join(ROOT, "profiles", "stream_probe*_r01.txt")):
        for line in open(p):
            m = None if line.startswith("#") else re.search(r"([0-9.]+) TB/s", line)
            if m:
                vals.append(float(m.group(1)))
    return max(vals) * 1000.0 if vals else None


def ncu_traffic(cfg, precision=32):
    """dram bytes per launch from the committed ncu --set full summary, if one matches this workload."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))
        e = d.get(cfg["name"] if precision == 32 else cfg["name"] + "_f64")
        if e and e.get("grid") == [cfg["nx"], cfg["ny"], cfg["nz"]]:
            return e.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return None


def cpu_baseline(cfg, budget_s=12.0, precision=32):
    """The oracle as it stands, on this host's cores, on a bounded sample of the same workload."""
    import numpy as np
    import torch

    import oracle
    import synth
    from synth import fields as SF
    oracle.build()
    wxy, wz = weights(cfg, precision)
    dt = synth.stable_dt(cfg)
    dt_np = np.float32 if precision == 32 else np.float64
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    nz = cfg["nz"]
    model = [a.cpu().numpy() for a in SF.model_planes(cfg, 0, nz, device=dev)]
    state = [SF.random_planes(cfg["nx"], cfg["ny"], 0, nz, 11, s, 1e-6, device=dev).cpu().numpy()
             for s in range(4)]
    P = oracle.params(cfg, dt)
    npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
    _, _, _, _, t1 = oracle.run(P, wxy, wz, *model, state, n0=100, nsteps=1, dtype=dt_np)
    k = int(max(1, min(50, budget_s / max(t1, 1e-3))))
    _, _, _, _, tk = oracle.run(P, wxy, wz, *model, state, n0=100, nsteps=k, dtype=dt_np)
    del model, state
    return {"value": round(npts * k / tk / 1e9, 6), "unit": "Gpoints/s", "cores": oracle.max_threads(),
            "kind": "oracle",
            "sample": f"oracle fp{precision} (C, OpenMP) on the full {cfg['nx']}x{cfg['ny']}x{cfg['nz']} {cfg['name']} grid, "
                      f"{k} time steps from a seeded random state (step loop only, {tk:.1f} s)"}


def run_reference(args):
    """--impl reference: the oracle (test infrastructure), timed on host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synth
    from synth import fields as SF
    cfg_full, scaling = workload(args, world)
    oracle.build()
    # bounded sample: the same recipe on a smaller grid, sized so W + K steps take ~2 minutes
    probe = synth.scaled(cfg_full, 128, 128, 128)

    def setup(c):
        wxy, wz, _ = synth.weights_f32(c)
        dt = synth.stable_dt(c, wxy, wz)
        model = [a.numpy() for a in SF.model_planes(c, 0, c["nz"])]
        state = [SF.random_planes(c["nx"], c["ny"], 0, c["nz"], 11, s, 1e-6).numpy() for s in range(4)]
        return oracle.params(c, dt), wxy, wz, model, state

    P, wxy, wz, model, state = setup(probe)
    _, _, _, _, t = oracle.run(P, wxy, wz, *model, state, nsteps=2)
    rate = 2 * 128 ** 3 / t
    pts = max(32 ** 3, min(cfg_full["nx"] * cfg_full["ny"] * cfg_full["nz"],
                           int(rate * 120.0 / max(1, args.steps + args.warmup))))
    side = int(round(pts ** (1.0 / 3.0)))
    side = max(2 * cfg_full["damp_width"] + 2, max(2 * cfg_full["r_z"] + 1, side))
    sample = synth.scaled(cfg_full, side, side, side)
    P, wxy, wz, model, state = setup(sample)
    st = oracle.run(P, wxy, wz, *model, state, nsteps=args.warmup)[:4] if args.warmup else state
    _, _, _, _, secs = oracle.run(P, wxy, wz, *model, st, n0=args.warmup, nsteps=args.steps)
    npts = side ** 3
    value = npts * args.steps / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gpoints/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / args.steps, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded)",
        "config": describe(cfg_full, world, scaling),
        "cpu_baseline": {"value": round(value, 6), "unit": "Gpoints/s", "cores": oracle.max_threads(),
                         "kind": "oracle",
                         "sample": f"oracle fp32 (C, OpenMP) on the {cfg_full['name']} recipe at {side}^3 "
                                   f"(bounded sample of {cfg_full['nx']}x{cfg_full['ny']}x{cfg_full['nz']}), "
                                   f"{args.warmup} warm-up + {args.steps} timed steps"},
        "e2e": {"value": round(value, 6), "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def make_handle(cfg, dt, wxy, wz, rank, world, local, nccl_id, precision=32):
    from paper_1410_1387_b200 import VTI
    return VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], cfg["r_xy"], cfg["r_z"], dt, wxy, wz,
               damp_width=cfg["damp_width"], damp_alpha=cfg["damp_alpha"], device=local, rank=rank,
               nranks=world, nccl_id=nccl_id, precision=precision)


def weights(cfg, precision):
    """float32 weights (the BASELINE path) or float64 weights for the fp64 path."""
    import numpy as np

    import synth
    from synth import weights as W
    if precision == 32:
        wxy, wz, _ = synth.weights_f32(cfg)
        return wxy, wz
    zc = W.z_coords_ramp(cfg["nz"], cfg["r_z"], cfg["dz"][0], cfg["dz"][1])
    return W.xy_weights(cfg["r_xy"]), np.ascontiguousarray(W.z_weights(zc, cfg["r_z"]))


def set_model_from_device(v, cfg, chunk=64):
    """Generate this rank's model slab on the GPU (synth, chunked by planes) and upload it."""
    import torch
    from synth import fields as SF
    for k0 in range(0, cfg["nz"], chunk):
        nk = min(chunk, cfg["nz"] - k0)
        m = SF.model_planes(cfg, k0, nk, device="cuda", j0=v.y0, nyl=v.ny_local)
        if v.precision == 64:
            m = [a.double() for a in m]
        v.set_model_planes(k0, *[a.contiguous() for a in m])
        del m
    torch.cuda.synchronize()


def run_native(args):
    import torch
    import torch.distributed as dist

    import synth
    import paper_1410_1387_b200 as vti

    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, scaling = workload(args, world)
    prec = args.precision
    from paper_1410_1387_b200 import perfmodel
    bpp = perfmodel.bytes_per_point(prec)   # 36 B/point in fp32, 72 in fp64
    wxy, wz = weights(cfg, prec)
    dt = synth.stable_dt(cfg)

    from paper_1410_1387_b200 import multi

    def fresh_nccl_id():
        return multi.broadcast_nccl_id(dist, rank, world)

    halo = os.environ.get("VTI_HALO", "peer") if world > 1 else "none"

    def open_handle():
        """A rank's handle with its halo transport: peer stores over CUDA IPC by default,
        NCCL if requested or if any rank cannot connect (collective fallback)."""
        if world > 1 and halo != "nccl":
            h = make_handle(cfg, dt, wxy, wz, rank, world, local, None, prec)
            if multi.connect_peer(dist, h, rank, world):
                return h
            h.close()
        return make_handle(cfg, dt, wxy, wz, rank, world, local, fresh_nccl_id(), prec)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return multi.max_over_ranks(dist, world, x, device="cuda")

    npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
    v = open_handle()
    transport = v.halo_transport
    if args.zchunk or args.ctas_per_sm:
        v.set_tuning(args.zchunk, args.ctas_per_sm)
    set_model_from_device(v, cfg)
    v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
    info = v.info()

    # warm-up (untimed), then exactly K timed steps bracketed by barrier + synchronize
    v.step(args.warmup)
    v.prepare()   # small grids: capture the step graphs now, not inside the timed region
    if world > 1:   # the first exchanges prove the transport; fail loudly rather than hang
        multi.sync_or_die(v, 120.0, f"warm-up ({transport} halo transport)")
    v.sync()
    barrier()
    with Clocks(local) as clk:
        ms = v.step_timed(args.steps)
    barrier()
    t_ms = max_over_ranks(ms)
    clocks = clk.summary()

    value = npts * args.steps / (t_ms * 1e-3) / 1e9
    launches = info["launches_per_step"] * args.steps
    pts_rank = cfg["nx"] * info["ny_local"] * cfg["nz"]
    # dominant kernel: the step kernel; at N = 1 one launch per step covers every point
    kern_ms = ms / args.steps
    achieved = bpp * pts_rank / (kern_ms * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    traffic = ncu_traffic(cfg, prec) if world == 1 else None
    v.close()

    e2e = None
    if not args.no_e2e:
        # through the public API with HOST buffers (pinned): model upload, K steps, read back u^K
        tdt = torch.float32 if prec == 32 else torch.float64
        pin = lambda shape: torch.empty(shape, dtype=tdt, pin_memory=True)
        shape = (cfg["nz"], info["ny_local"], cfg["nx"])
        host_model = [pin(shape) for _ in range(3)]
        from synth import fields as SF
        for k0 in range(0, cfg["nz"], 64):
            nk = min(64, cfg["nz"] - k0)
            m = SF.model_planes(cfg, k0, nk, device="cuda", j0=info["y0"], nyl=info["ny_local"])
            for dst, src in zip(host_model, m):
                dst[k0:k0 + nk].copy_(src)
        out_p, out_q = pin(shape), pin(shape)
        w = open_handle()
        if args.zchunk or args.ctas_per_sm:
            w.set_tuning(args.zchunk, args.ctas_per_sm)
        barrier()
        t0 = time.perf_counter()
        w.set_model(*host_model)
        w.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        w.step(args.steps)
        w.get_fields(0, out_p, out_q)
        w.sync()
        te = time.perf_counter() - t0
        barrier()
        te = max_over_ranks(te)
        w.close()
        nbytes = (prec // 8) * cfg["nx"] * cfg["ny"] * cfg["nz"]
        e2e = {"value": round(npts * args.steps / te / 1e9, 4), "unit": "Gpoints/s",
               "h2d_bytes_per_step": int(3 * nbytes / args.steps), "d2h_bytes_per_step": int(2 * nbytes / args.steps),
               "what": "vti_set_model (pinned host) + vti_add_source + vti_step(K) + vti_get_fields(u^K to pinned host), wall clock, max over ranks"}
        del host_model

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, precision=prec)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 5),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": f"f{prec}",
            "data": "synthetic (seeded layered VTI model generated on device; zero initial state + Ricker source)",
            "config": describe(cfg, world, scaling, bpp, transport),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                         "mix_ceiling": ({"gbs": mc, "frac": round(achieved / mc, 4),
                                          "source": "profiles/stream_probe*_r01.txt (7 read + 2 write streams, "
                                                    "best of plain and TMA-bulk loads)"}
                                         if (mc := mix_ceiling()) else None),
                         "kernel": "vti::vti_step_kernel<4,4>" if cfg["r_xy"] == 4 else f"vti::vti_step_kernel<{cfg['r_xy']},{cfg['r_z']}>",
                         "algorithmic_bytes_per_launch": bpp * pts_rank,
                         "flops_per_point": {"paper_count": perfmodel.flops_per_point(cfg["r_xy"], cfg["r_z"]),
                                             "canonical_order": perfmodel.step_flops_per_point(cfg["r_xy"], cfg["r_z"])},
                         "gflops": round(perfmodel.step_flops_per_point(cfg["r_xy"], cfg["r_z"]) * value, 1)},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "schedule": {k: info[k] for k in ("tile_x", "tile_y", "producer_warp", "rows_per_thread", "points_per_thread",
                                              "small_kernel",
                                              "zchunk", "grid", "work_items")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
