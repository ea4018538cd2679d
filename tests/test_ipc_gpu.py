"""Multi-process fused peer transport over CUDA IPC on one GPU.

Two processes on cuda:0, each owning one y-slab handle (nranks = 2, nccl_id = NULL).
* Bootstrap: bench.py's own rank setup (bench.open_handle -> multi.connect_peer over a
  gloo group) exports the IPC blobs, all-gathers them and opens the neighbour's buffers
  and flag words; the handles report the peer transport and the fused one-launch step,
  and bench.py's N > 1 guards run on them (multi.sync_or_die on the idle library stream,
  multi.max_over_ranks with a device tensor).
* One-sided stepping: ranks that wait on one another must not share one GPU
  (B200_PROFILING.md), so rank 0 steps with its own flag words pre-set (test-only hook
  vti_debug_flags) while rank 1 stays idle, then rank 1 checks what arrived in its memory.
The two-sided protocol is covered by the local-group GPU tests (same kernels and flag
sequence), the CPU model check (tests/test_peer_protocol_cpu.py) and, on >= 2 GPUs,
tests/test_multigpu_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1410_1387_b200 import VTI, VTIError, multi
        nz = 20
        h = VTI(64, 192, nz, 10.0, 4, 4, 1e-3, np.zeros(5, np.float32), np.zeros(nz * 9, np.float32),
                damp_width=0, device=0, rank=rank, nranks=world)
        before = h.halo_transport
        ok = multi.connect_peer(dist, h, rank, world)
        res = {"before": before, "ok": ok, "after": h.halo_transport, "launches": h.info()["launches_per_step"]}
        # bench.py's own rank setup and N > 1 guards (no stepping: see the module docstring)
        import bench
        import synth
        cfg = synth.scaled(synth.CONFIGS["C4"](), 64, 192, 24, damp_width=4)
        wxy, wz, _ = synth.weights_f32(cfg)
        b = bench.open_handle(cfg, 1e-3, wxy, wz, rank, world, 0, 32, dist, "peer")
        res["bench_transport"] = b.halo_transport
        multi.sync_or_die(b, 5.0, "idle stream")   # must return (nothing enqueued)
        res["max"] = multi.max_over_ranks(dist, world, float(rank) + 0.25, device="cuda")
        b.close()
        # a blob of the wrong rank is refused
        try:
            h.ipc_connect(h.ipc_export() if rank > 0 else None, h.ipc_export() if rank < world - 1 else None)
            res["self_blob"] = "accepted"
        except VTIError as e:
            res["self_blob"] = e.name
        dist.barrier()
        h.close()
        dist.barrier()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_connect():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=240) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert got[r]["before"] == "none", got
        assert got[r]["ok"] is True, got
        assert got[r]["after"] == "peer", got
        assert got[r]["launches"] == 1, got   # a multi-process peer rank runs the fused one-launch step
        assert got[r]["self_blob"] == "VTI_E_PARAM", got
        assert got[r]["bench_transport"] == "peer" and got[r]["max"] == 1.25, got
    for p in procs:
        assert p.exitcode == 0


def _one_sided_worker(rank, world, port, q):
    """Rank 0 steps with its neighbour's flags pre-satisfied (no process waits on another's GPU
    work); rank 1 stays idle and afterwards inspects what arrived in its memory over CUDA IPC."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import synth
        from synth import fields as SF
        from paper_1410_1387_b200 import VTI, multi
        cfg = synth.scaled(synth.CONFIGS["C2"](), 70, 96, 20, damp_width=4, dz=(6.0, 12.0), t0=0.02)
        wxy, wz, _ = synth.weights_f32(cfg)
        dt = synth.stable_dt(cfg, wxy, wz)
        h = VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], 4, 4, dt, wxy, wz, damp_width=4, device=0,
                rank=rank, nranks=world)
        assert multi.connect_peer(dist, h, rank, world)
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a.numpy()[:, sl]) for a in SF.model_planes(cfg, 0, cfg["nz"])])
        res = {"launches": h.info()["launches_per_step"]}
        K = 3
        dist.barrier()
        if rank == 0:
            h.debug_flags(set8=[1 << 20] * 8)   # the neighbour's DATA / ACK: every wait passes
            st = [SF.random_planes(cfg["nx"], cfg["ny"], 0, cfg["nz"], 5, s, 1e-3).numpy()[:, sl] for s in range(4)]
            h.set_fields(*[np.ascontiguousarray(a) for a in st], time_index=0)
            h.step(K)   # the fused one-launch peer step: PEER stores + device-side flag release over IPC
            h.sync()
            res["last_rows"] = h.get_fields(0)[0][:, -4:, :].copy()
        dist.barrier()
        if rank == 1:
            # rank 0's output buffer of step K has index K % 2; this idle rank's cur is 0
            res["halo"] = h.debug_halo(level=K % 2, side=0)
            res["flags"] = h.debug_flags().tolist()
        dist.barrier()
        h.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_one_sided_step():
    """The multi-process fused peer step across two processes on cuda:0 without mutual waiting:
    rank 0's last R_xy rows of u^K land in rank 1's halo rows through CUDA-IPC peer stores, and
    rank 0's last edge CTA raises rank 1's flag words (st.release.sys) to the publication count."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_one_sided_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=300) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert got[0]["launches"] == 1 and got[1]["launches"] == 1
    assert np.abs(got[0]["last_rows"]).max() > 0
    assert np.array_equal(got[1]["halo"], got[0]["last_rows"])
    # publications: the re-publication of the state set by the caller, then one per step
    assert got[1]["flags"] == [4, 0, 3, 0, 0, 0, 0, 0], got[1]["flags"]
    for p in procs:
        assert p.exitcode == 0


def _one_sided_adjoint_worker(rank, world, port, q):
    """The multi-process adjoint over CUDA IPC, one-sided: rank 0 (flags pre-set) runs K chained
    adjoint steps, each publishing its s1 boundary rows straight into rank 1's receive buffer;
    rank 1 stays idle and then reads that buffer and its flag words."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import synth
        from synth import fields as SF
        from paper_1410_1387_b200 import VTI, multi
        cfg = synth.scaled(synth.CONFIGS["C2"](), 70, 96, 20, damp_width=4, dz=(6.0, 12.0), t0=0.02)
        wxy, wz, _ = synth.weights_f32(cfg)
        dt = synth.stable_dt(cfg, wxy, wz)
        h = VTI(cfg["nx"], cfg["ny"], cfg["nz"], cfg["h"], 4, 4, dt, wxy, wz, damp_width=4, device=0,
                rank=rank, nranks=world)
        assert multi.connect_peer(dist, h, rank, world)
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a.numpy()[:, sl]) for a in SF.model_planes(cfg, 0, cfg["nz"])])
        res = {}
        K = 3
        dist.barrier()
        if rank == 0:
            h.debug_flags(set8=[1 << 20] * 8)
            st = [SF.random_planes(cfg["nx"], cfg["ny"], 0, cfg["nz"], 5, s, 1e-3).numpy()[:, sl] for s in range(4)]
            h.set_fields(*[np.ascontiguousarray(a) for a in st], time_index=30)
            h.step_adjoint(K)
            h.sync()
            # publications: s1 of the initial state (scratch 0), then of each chained step's output
            # (scratch 1, 0, ...): the last, publication K, is in scratch (K - 1) % 2
            res["last_rows"] = h.debug_rows(2 * ((K - 1) % 2) + 1)
            res["time_index"] = h.time_index
        dist.barrier()
        if rank == 1:
            res["rbuf"] = h.debug_rows(4)
            res["flags"] = h.debug_flags().tolist()
        dist.barrier()
        h.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_one_sided_adjoint():
    """vti_step_adjoint on a multi-process peer rank: rank 0's s1 boundary rows of its last
    publication arrive bitwise in rank 1's receive buffer over CUDA IPC, and rank 0 raises rank
    1's S1DATA and S1ACK words to the publication count (K chained steps publish K times)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_one_sided_adjoint_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=300) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert got[0]["time_index"] == 27
    assert np.abs(got[0]["last_rows"]).max() > 0
    assert np.array_equal(got[1]["rbuf"], got[0]["last_rows"])
    assert got[1]["flags"] == [0, 0, 0, 0, 3, 0, 3, 0], got[1]["flags"]
    for p in procs:
        assert p.exitcode == 0
