"""Multi-process y-slab stepping across GPUs: one process per
GPU, each owning one slab, the halo exchange over the fused CUDA-IPC peer step (the default) or
over NCCL send/recv (VTI_HALO=nccl); the gathered fields after K steps must equal the oracle's
single-domain run bitwise. Also `torchrun bench.py --gpus 2`.

These tests need >= 2 GPUs in one node and SKIP otherwise; the round's GPU box has one, and
ranks that wait on one another must not share a GPU (B200_PROFILING.md). The one-rank run of the
same harness checks the harness itself on one GPU. The one-GPU evidence for the
same code is tests/test_ipc_gpu.py (the one-sided IPC step), tests/test_peer_gpu.py (local
groups, both transports' kernels) and tests/test_peer_protocol_cpu.py (the flag protocol).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from synth import fields as SF

pytestmark = pytest.mark.gpu


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _need(n):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs in one node")


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(r, rz, ny, prec=32):
    cfg = synth.scaled(synth.CONFIGS["C2"](), 72, ny, 2 * rz + 12, r_xy=r, r_z=rz, damp_width=5,
                       dz=(6.0, 12.0), t0=0.02)
    cfg["src"] = (36, ny // 2, cfg["nz"] // 2)   # on or next to a slab boundary for even worlds
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    if prec == 64:
        from synth import weights as W
        wxy = W.xy_weights(r)
        wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(cfg["nz"], rz, 6.0, 12.0), rz))
    return cfg, wxy, wz, dt


def _worker(rank, world, port, q, halo, r, rz, ny, K):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        sys.path.insert(0, ROOT)
        import bench
        cfg, wxy, wz, dt = _case(r, rz, ny)
        h = bench.open_handle(cfg, dt, wxy, wz, rank, world, rank, 32, dist, halo)
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a.numpy()[:, sl]) for a in SF.model_planes(cfg, 0, cfg["nz"])])
        h.add_source(*cfg["src"], f=cfg["f"], t0=cfg["t0"], amp=cfg["amp"], mask=cfg["mask"])
        from paper_1410_1387_b200 import multi
        h.step(K // 2)
        multi.sync_or_die(h, 60.0, f"{halo} steps")
        h.step(K - K // 2)
        multi.sync_or_die(h, 60.0, f"{halo} steps")
        res = {"transport": h.halo_transport, "y0": h.y0, "fields": h.get_fields(0) + h.get_fields(1)}
        dist.barrier()
        h.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(world, halo, r=4, rz=4, ny=None, K=24):
    ny = ny or 40 * world + 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q, halo, r, rz, ny, K)) for rk in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=600) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    cfg, wxy, wz, dt = _case(r, rz, ny)
    model = SF.model_planes(cfg, 0, cfg["nz"])
    o = oracle.run(oracle.params(cfg, dt), wxy, wz, *[a.numpy() for a in model], nsteps=K)
    order = sorted(got, key=lambda k: got[k]["y0"])
    for f in range(4):
        g = np.concatenate([got[k]["fields"][f] for k in order], axis=1)
        assert np.abs(o[f]).max() > 0
        assert np.array_equal(g, o[f]), f"field {f}: max |diff| {np.abs(g - o[f]).max():.3e}"
    return [got[k]["transport"] for k in order]


def test_harness_one_rank():
    """The same spawn / bench.open_handle / oracle comparison with one rank (no transport)."""
    _need(1)
    assert _run(1, "peer") == ["none"]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_peer_slabs_equal_oracle(world):
    _need(world)
    assert _run(world, "peer") == ["peer"] * world


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_slabs_equal_oracle(world):
    _need(world)
    assert _run(world, "nccl") == ["nccl"] * world


@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_paper_radii_thin_slabs(halo):
    """(12,8) radii with slabs of 16 rows: every row of a slab is some neighbour's halo row."""
    _need(2)
    assert _run(2, halo, r=12, rz=8, ny=32, K=12) == [halo] * 2


def _adj_worker(rank, world, port, q, r, rz, prec, ny, K, halo):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        sys.path.insert(0, ROOT)
        import bench
        cfg, wxy, wz, dt = _case(r, rz, ny, prec)
        h = bench.open_handle(cfg, dt, wxy, wz, rank, world, rank, prec, dist, halo)
        sl = slice(h.y0, h.y0 + h.ny_local)
        dtype = np.float32 if prec == 32 else np.float64
        model = [np.ascontiguousarray(a.numpy()[:, sl].astype(dtype)) for a in SF.model_planes(cfg, 0, cfg["nz"])]
        st = [np.ascontiguousarray(SF.random_planes(cfg["nx"], ny, 0, cfg["nz"], 7, s, 1e-3).numpy()[:, sl].astype(dtype))
              for s in range(4)]
        h.set_model(*model)
        h.set_fields(*st, time_index=40)
        h.step_adjoint(K)
        h.sync()
        res = {"transport": h.halo_transport, "y0": h.y0, "fields": h.get_fields(0) + h.get_fields(1)}
        dist.barrier()
        h.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("halo", ["nccl", "peer"])
@pytest.mark.parametrize("r,rz,prec", [(4, 4, 32), (12, 8, 32), (6, 6, 64)])
def test_adjoint_slabs_equal_oracle(r, rz, prec, halo):
    """vti_step_adjoint over y-slabs, one process per GPU: the chained two-pass TMA form with the
    s1 boundary rows exchanged each step over NCCL or CUDA IPC; bitwise equal to the oracle."""
    _need(2)
    world, K = 2, 10
    ny = 40 * world + 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_adj_worker, args=(rk, world, port, q, r, rz, prec, ny, K, halo))
             for rk in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=600) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    cfg, wxy, wz, dt = _case(r, rz, ny, prec)
    dtype = np.float32 if prec == 32 else np.float64
    model = [a.numpy().astype(dtype) for a in SF.model_planes(cfg, 0, cfg["nz"])]
    st = [SF.random_planes(cfg["nx"], ny, 0, cfg["nz"], 7, s, 1e-3).numpy().astype(dtype) for s in range(4)]
    o = oracle.adjoint_ex(oracle.params(cfg, dt, src=None), wxy, wz, *model, st, m0=40, nsteps=K, dtype=dtype)
    order = sorted(got, key=lambda k: got[k]["y0"])
    assert [got[k]["transport"] for k in order] == [halo] * world
    for f in range(4):
        g = np.concatenate([got[k]["fields"][f] for k in order], axis=1)
        assert np.array_equal(g, o[f]), f"field {f}: max |diff| {np.abs(g - o[f]).max():.3e}"


@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_torchrun_bench_two_gpus(halo):
    _need(2)
    env = dict(os.environ, VTI_HALO=halo)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--config", "C3", "--steps", "10", "--warmup", "3", "--reps", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["halo_transport"] == halo
