#!/usr/bin/env python
"""Benchmark: VTI time steps per second on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--reps R] [--config C4]
                  [--impl native|reference]

One "step" = one time step of the reduced elastic VTI propagator (PAPER.md
Eqs. 1-3) over the whole grid: every row of SURVEY.md 8(a) runs inside the
fused sm_100a kernel (for N > 1 the halo exchange of p is fused into it as
peer stores over NVLink, or NCCL send/recv when CUDA IPC is unavailable).

Workload (default at every N): BASELINE.json configs[3] = C4, 2048 x 2048 x
1024, R_xy = R_z = 4, layered VTI with variable dz, Cerjan W = 20, Ricker source
at the centre, starting from the zero state -- north_star's ">= 85 % at 8 GPUs
on a 2048x2048x1024 grid" workload and the largest single-GPU configuration
(120 GB of HBM at N = 1). N > 1: strong scaling, one y-slab of 2048/N rows per
rank. --config C1/C2/C3/C5/N1 time the other BASELINE configurations (C2/N1
and C5 weak-scaled along y for N > 1). Inputs (155 GB/step at N = 1) are far
larger than the 126 MB L2, so no explicit flush is needed between steps.

Metric: Gpoints/s = (global grid points) x K / t, t = max over ranks of the
CUDA-event time of K steps on the library's stream; the K-step region is timed
--reps times (default 5, each bracketed by barrier + synchronize) and `value`
is the median. ``roofline`` uses 36 algorithmic bytes per point-update
 against the measured HBM copy bandwidth in
MEASURED_PEAKS.json, with the nominal 8 TB/s fraction alongside.
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5, help="timed K-step regions; value = their median")
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5", "N1"])
    ap.add_argument("--scaling", default=None, choices=[None, "weak", "strong"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps of the end-to-end job (0 = the config's stated step count)")
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
    import synth
    npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
    return {
        "workload": f"{cfg['name']}: {cfg['nx']}x{cfg['ny']}x{cfg['nz']} global, R_xy={cfg['r_xy']} R_z={cfg['r_z']}, "
                    f"{cfg['model']['kind']} VTI, W={cfg['damp_width']}, Ricker f={cfg['f']:g} Hz at the centre",
        "grid": [cfg["nx"], cfg["ny"], cfg["nz"]],
        "r_xy": cfg["r_xy"], "r_z": cfg["r_z"], "config_steps": cfg["steps"],
        "dt": synth.stable_dt(cfg), "h": cfg["h"], "dz": list(cfg["dz"]), "src": list(cfg["src"]),
        "damping": {"width": cfg["damp_width"], "alpha": cfg["damp_alpha"]},
        "decomposition": f"y-slabs x{world}" if world > 1 else "single GPU",
        "halo_transport": transport,
        "scaling": scaling,
        "l2_flush": (f"not needed: per-step working set {bpp * npts / 1e9:.1f} GB ({bpp} B/pt) >> 126 MB L2"
                     if bpp * npts > 4 * 126e6 else
                     f"none: the whole per-step working set ({bpp * npts / 1e6:.1f} MB) stays L2-resident "
                     "across steps (a small-grid, latency-bound workload)"),
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


NOMINAL_HBM_GBS = 8000.0   # B200 nominal HBM3e bandwidth (north_star "~8 TB/s")


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
    """(dram bytes per launch, source) from the committed ncu --set full summary
    (profiles/ncu_summary.json, tools/ncu_summary.py) if it holds this workload's grid."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))
        e = d.get(cfg["name"] if precision == 32 else cfg["name"] + "_f64")
        if e and e.get("grid") == [cfg["nx"], cfg["ny"], cfg["nz"]]:
            return e.get("dram_bytes_per_launch"), f"prior ncu --set full capture ({e.get('source', 'profiles/')})"
    except (OSError, ValueError):
        pass
    return None, None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


REF_MAX_POINTS = 320 ** 3   # the reference arm's largest sample cube (~1.2 GB of oracle arrays)


def reference_side(cfg_full, rate, steps, warmup, budget_s=120.0):
    """Edge of the reference arm's sample cube: W + K oracle steps in about budget_s at the
    probed rate (points/s), at most REF_MAX_POINTS (host memory and input generation stay
    small whatever the config), at least what the damping band and the z stencil need."""
    pts = max(32 ** 3, min(cfg_full["nx"] * cfg_full["ny"] * cfg_full["nz"], REF_MAX_POINTS,
                           int(rate * budget_s / max(1, steps + warmup))))
    side = int(round(pts ** (1.0 / 3.0)))
    return max(2 * cfg_full["damp_width"] + 2, max(2 * cfg_full["r_z"] + 1, side))


def host_inputs(c, chunk=32, dtype=None):
    """The recipe's model and a seeded random state on the host, generated plane-chunk by
    plane-chunk into preallocated arrays (bounded temporaries)."""
    import numpy as np

    from synth import fields as SF
    shape = (c["nz"], c["ny"], c["nx"])
    model = [np.empty(shape, np.float32) for _ in range(3)]
    state = [np.empty(shape, np.float32) for _ in range(4)]
    for k0 in range(0, c["nz"], chunk):
        nk = min(chunk, c["nz"] - k0)
        for dst, src in zip(model, SF.model_planes(c, k0, nk)):
            dst[k0:k0 + nk] = src.numpy()
        for s, dst in enumerate(state):
            dst[k0:k0 + nk] = SF.random_planes(c["nx"], c["ny"], k0, nk, 11, s, 1e-6).numpy()
    return model, state


def cpu_baseline(cfg, budget_s=12.0, precision=32):
    """The oracle as it stands, on this host's cores, on a bounded sample of the same workload:
    the config's recipe on SURVEY.md 8(d)'s reduced grid (256 x 256 x 128 for C4/C5, the full
    grid for C1, else at most 256^3), from a seeded random state; all threads, then 1 thread."""
    import numpy as np

    import oracle
    import synth
    oracle.build()
    if cfg["nx"] * cfg["ny"] * cfg["nz"] > 256 ** 3:
        sample = synth.scaled(cfg, min(cfg["nx"], 256), min(cfg["ny"], 256), 128 if cfg["nz"] >= 1024 else
                              min(cfg["nz"], 256))
    else:
        sample = cfg
    wxy, wz = weights(sample, precision)
    dt = synth.stable_dt(sample)
    dt_np = np.float32 if precision == 32 else np.float64
    model, state = host_inputs(sample)
    P = oracle.params(sample, dt)
    npts = sample["nx"] * sample["ny"] * sample["nz"]
    threads = host_threads()
    _, _, _, _, t1 = oracle.run(P, wxy, wz, *model, state, n0=100, nsteps=1, dtype=dt_np, nthreads=threads)
    k = int(max(1, min(400, budget_s / max(t1, 1e-3))))
    _, _, _, _, tk = oracle.run(P, wxy, wz, *model, state, n0=100, nsteps=k, dtype=dt_np, nthreads=threads)
    k1 = int(max(1, min(10, 0.25 * budget_s / max(t1 * threads, 1e-3))))
    _, _, _, _, t1t = oracle.run(P, wxy, wz, *model, state, n0=100, nsteps=k1, dtype=dt_np, nthreads=1)
    return {"value": round(npts * k / tk / 1e9, 6), "unit": "Gpoints/s", "cores": threads,
            "kind": "oracle", "cpu": cpu_model(),
            "one_thread": {"value": round(npts * k1 / t1t / 1e9, 6), "steps": k1},
            "sample": f"oracle fp{precision} (C, OpenMP, {threads} threads) on the {cfg['name']} recipe at "
                      f"{sample['nx']}x{sample['ny']}x{sample['nz']} (bounded sample of "
                      f"{cfg['nx']}x{cfg['ny']}x{cfg['nz']}), {k} time steps from a seeded random state "
                      f"(step loop only, {tk:.1f} s); one_thread: {k1} steps on 1 thread"}


def run_reference(args):
    """--impl reference: the oracle (test infrastructure), timed on host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synth
    cfg_full, scaling = workload(args, world)
    oracle.build()
    # bounded sample: the same recipe on a smaller grid, sized so W + K steps take ~2 minutes
    probe = synth.scaled(cfg_full, 128, 128, 128)

    def setup(c):
        wxy, wz, _ = synth.weights_f32(c)
        dt = synth.stable_dt(c, wxy, wz)
        model, state = host_inputs(c)
        return oracle.params(c, dt), wxy, wz, model, state

    threads = host_threads()
    P, wxy, wz, model, state = setup(probe)
    _, _, _, _, t = oracle.run(P, wxy, wz, *model, state, nsteps=2, nthreads=threads)
    rate = 2 * 128 ** 3 / t
    side = reference_side(cfg_full, rate, args.steps, args.warmup)
    sample = synth.scaled(cfg_full, side, side, side)
    P, wxy, wz, model, state = setup(sample)
    st = oracle.run(P, wxy, wz, *model, state, nsteps=args.warmup, nthreads=threads)[:4] if args.warmup else state
    _, _, _, _, secs = oracle.run(P, wxy, wz, *model, st, n0=args.warmup, nsteps=args.steps, nthreads=threads)
    npts = side ** 3
    value = npts * args.steps / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gpoints/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / args.steps, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded)",
        "config": describe(cfg_full, world, scaling),
        "cpu_baseline": {"value": round(value, 6), "unit": "Gpoints/s", "cores": threads,
                         "kind": "oracle", "cpu": cpu_model(),
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


def open_handle(cfg, dt, wxy, wz, rank, world, local, prec, dist, halo="peer"):
    """A rank's handle with its halo transport: fused peer stores over CUDA IPC by default
    (multi.connect_peer), NCCL if requested (VTI_HALO=nccl) or if any rank cannot connect
    (the decision is collective). world == 1: a single-slab handle."""
    from paper_1410_1387_b200 import multi
    if world > 1 and halo != "nccl":
        h = make_handle(cfg, dt, wxy, wz, rank, world, local, None, prec)
        if multi.connect_peer(dist, h, rank, world):
            return h
        h.close()
    nccl_id = multi.broadcast_nccl_id(dist, rank, world) if world > 1 else None
    return make_handle(cfg, dt, wxy, wz, rank, world, local, nccl_id, prec)


def warm_up(v, steps, world, transport, timeout_s=120.0):
    """W untimed steps, graph capture for small grids, and -- for N > 1 -- the guard that
    turns a transport that never delivers into a loud exit instead of a hang."""
    from paper_1410_1387_b200 import multi
    v.step(steps)
    v.prepare()   # small grids: capture the step graphs now, not inside the timed region
    if world > 1:
        multi.sync_or_die(v, timeout_s, f"warm-up ({transport} halo transport)")
    v.sync()


class Watchdog:
    """Exit the process loudly (code 4) if a guarded region outlives timeout_s -- a halo
    transport that stops delivering mid-run must fail the job, not hang it (N > 1 only;
    the warm-up is guarded by multi.sync_or_die)."""

    def __init__(self, timeout_s, what, enabled=True):
        self.timeout_s, self.what, self.enabled, self.t = timeout_s, what, enabled, None

    def _fire(self):
        print(f"error: {self.what} did not finish within {self.timeout_s:.0f} s; aborting", file=sys.stderr,
              flush=True)
        os._exit(4)

    def __enter__(self):
        if self.enabled:
            import threading
            self.t = threading.Timer(self.timeout_s, self._fire)
            self.t.daemon = True
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.t:
            self.t.cancel()


def setup_rank(args, cfg, dt, wxy, wz, rank, world, local, dist, halo):
    """Everything a rank does before the timed region: handle + transport, tuning, model,
    source and warm-up. Returns (handle, transport name)."""
    v = open_handle(cfg, dt, wxy, wz, rank, world, local, args.precision, dist, halo)
    transport = v.halo_transport
    if args.zchunk or args.ctas_per_sm:
        v.set_tuning(args.zchunk, args.ctas_per_sm)
    set_model_from_device(v, cfg)
    v.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
    warm_up(v, args.warmup, world, transport)
    return v, transport


def end_to_end(args, cfg, dt, wxy, wz, rank, world, local, dist, halo, info, barrier, max_over_ranks):
    """The config's whole job through the public API with HOST buffers (pinned): model upload,
    source, e2e_steps steps, read back u^N. Wall clock, max over ranks."""
    import torch

    from synth import fields as SF
    import numpy as np
    prec = args.precision
    nsteps = args.e2e_steps or cfg["steps"]
    shape = (cfg["nz"], info["ny_local"], cfg["nx"])
    rt = torch.cuda.cudart()
    registered = []

    def pinned():
        # exact-size page-locked host arrays (cudaHostRegister on numpy memory): torch's pinned
        # caching allocator rounds large blocks up, which C4 (17 GB per array) cannot afford
        a = np.empty(shape, np.float32 if prec == 32 else np.float64)
        err = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        if int(err) != 0:
            raise RuntimeError(f"cudaHostRegister({a.nbytes} B) failed: {err}")
        registered.append(a)
        return a

    host_model = [pinned() for _ in range(3)]
    for k0 in range(0, cfg["nz"], 64):
        nk = min(64, cfg["nz"] - k0)
        m = SF.model_planes(cfg, k0, nk, device="cuda", j0=info["y0"], nyl=info["ny_local"])
        for dst, src in zip(host_model, m):
            torch.from_numpy(dst[k0:k0 + nk]).copy_(src.to(torch.float32 if prec == 32 else torch.float64))
        del m
    out_p, out_q = pinned(), pinned()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    w = open_handle(cfg, dt, wxy, wz, rank, world, local, prec, dist, halo)
    if args.zchunk or args.ctas_per_sm:
        w.set_tuning(args.zchunk, args.ctas_per_sm)
    barrier()
    t0 = time.perf_counter()
    w.set_model(*host_model)
    w.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
    w.step(nsteps)
    w.get_fields(0, out_p, out_q)
    w.sync()
    te = time.perf_counter() - t0
    barrier()
    te = max_over_ranks(te)
    w.close()
    npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
    nbytes = (prec // 8) * npts
    for a in registered:
        rt.cudaHostUnregister(a.ctypes.data)
    del host_model, out_p, out_q, registered
    return {"value": round(npts * nsteps / te / 1e9, 4), "unit": "Gpoints/s", "steps": nsteps,
            "h2d_bytes_per_step": int(3 * nbytes / nsteps), "d2h_bytes_per_step": int(2 * nbytes / nsteps),
            "seconds": round(te, 3),
            "what": f"the config's whole job: vti_set_model (pinned host model, {3 * nbytes / 1e9:.1f} GB) + "
                    f"vti_add_source + vti_step({nsteps}) + vti_get_fields(u^N, {2 * nbytes / 1e9:.1f} GB to "
                    "pinned host), wall clock, max over ranks"}


def run_native(args):
    import statistics

    import torch
    import torch.distributed as dist

    import synth
    from paper_1410_1387_b200 import multi, perfmodel

    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, scaling = workload(args, world)
    prec = args.precision
    bpp = perfmodel.bytes_per_point(prec)   # 36 B/point in fp32, 72 in fp64
    wxy, wz = weights(cfg, prec)
    dt = synth.stable_dt(cfg)
    halo = os.environ.get("VTI_HALO", "peer") if world > 1 else "none"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return multi.max_over_ranks(dist, world, x, device="cuda")

    npts = cfg["nx"] * cfg["ny"] * cfg["nz"]
    v, transport = setup_rank(args, cfg, dt, wxy, wz, rank, world, local, dist, halo)
    info = v.info()

    # --reps timed regions of exactly K steps, each bracketed by barrier + synchronize
    reps = []
    barrier()
    with Clocks(local) as clk, Watchdog(600.0 + 2.0 * args.reps * args.steps, "timed region", world > 1):
        for _ in range(max(1, args.reps)):
            barrier()
            ms = v.step_timed(args.steps)
            barrier()
            reps.append(max_over_ranks(ms))
    clocks = clk.summary()
    t_ms = statistics.median(reps)

    value = npts * args.steps / (t_ms * 1e-3) / 1e9
    spl = info.get("steps_per_launch", 1)   # > 1: the multi-step small-grid kernel
    launches = info["launches_per_step"] * (args.steps if spl <= 1 else -(-args.steps // spl))
    pts_rank = cfg["nx"] * info["ny_local"] * cfg["nz"]
    # dominant kernel: the step kernel; one launch per step covers every point of the slab
    kern_ms = t_ms / args.steps
    achieved = bpp * pts_rank / (kern_ms * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    traffic, traffic_src = ncu_traffic(cfg, prec) if world == 1 else (None, None)
    v.close()
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        with Watchdog(1800.0, "end-to-end job", world > 1):
            e2e = end_to_end(args, cfg, dt, wxy, wz, rank, world, local, dist, halo, info, barrier, max_over_ranks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, precision=prec)

    if rank == 0:
        mc = mix_ceiling()
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 7),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": f"f{prec}",
            "data": "synthetic (seeded layered VTI model generated on device; zero initial state + Ricker source)",
            "config": describe(cfg, world, scaling, bpp, transport),
            "repetitions": {"n": len(reps), "statistic": "median", "ms_per_region": [round(x, 4) for x in reps],
                            "gpoints_s": [round(npts * args.steps / (x * 1e-3) / 1e9, 3) for x in reps]},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "nominal": {"peak": NOMINAL_HBM_GBS, "frac": round(achieved / NOMINAL_HBM_GBS, 4),
                                     "source": "B200 nominal HBM3e bandwidth (north_star ~8 TB/s)"},
                         "mix_ceiling": ({"gbs": mc, "frac": round(achieved / mc, 4),
                                          "source": "profiles/stream_probe*_r01.txt (7 read + 2 write streams, "
                                                    "best of plain and TMA-bulk loads)"} if mc else None),
                         "kernel": f"vti::vti_step_kernel<{'float' if prec == 32 else 'double'},"
                                   f"{cfg['r_xy']},{cfg['r_z']},...>"
                                   + (" (small-grid kernel vti_small_kernel)" if info["small_kernel"] else ""),
                         "algorithmic_bytes_per_launch": bpp * pts_rank,
                         "bytes_per_point": bpp, "points_per_launch": pts_rank,
                         "flops_per_point": {"paper_count": perfmodel.flops_per_point(cfg["r_xy"], cfg["r_z"]),
                                             "canonical_order": perfmodel.step_flops_per_point(cfg["r_xy"], cfg["r_z"])},
                         "gflops": round(perfmodel.step_flops_per_point(cfg["r_xy"], cfg["r_z"]) * value, 1)},
            "e2e": e2e,
            "gpu_launches": launches,
            "timed_regions": len(reps),
            "clocks": clocks,
            "cpu_baseline": cpu,
            "schedule": {k: info[k] for k in ("tile_x", "tile_y", "producer_warp", "rows_per_thread", "points_per_thread",
                                              "small_kernel", "zchunk", "grid", "work_items", "launches_per_step",
                                              "steps_per_launch")},
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
