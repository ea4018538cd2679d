"""World-size-2 (and 3) gloo tests of the y-slab decomposition on CPU.

The multi-GPU path splits y into slabs with the library's
own partition rule (vti_slab), keeps a R_xy-row halo of p only (q has no x-y
derivative, Eqs. 1-2), injects the source on the owning rank only, and
exchanges p's boundary rows with rank -/+ 1 after every step. Here each rank
steps its slab with the oracle on an (ny_local + 2R)-row subgrid, exchanging
halos through torch.distributed (gloo) send/recv in the same neighbour
pattern as the library's NCCL group, and the gathered result must equal a
single-domain oracle run bitwise. Also covered: per-rank model-slab
generation equals the global model's rows, and bench.py's bootstrap
(paper_1410_1387_b200.multi: library ncclUniqueId broadcast, max over ranks).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import oracle
    import synth
    cfg = synth.scaled(synth.CONFIGS["C2"](), 28, 23, 20, damp_width=0, dz=(6.0, 12.0), t0=0.01,
                       src=(13, 11, 9))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    return oracle, synth, cfg, wxy, wz, dt


def _exchange(p_halo, R, nyl, rank, world):
    """Fill the R halo rows of p (axis 1 = y, rows [0,R) and [R+nyl, 2R+nyl)) from the neighbours."""
    reqs = []
    recv_lo = torch.zeros_like(torch.from_numpy(p_halo[:, :R].copy()))
    recv_hi = torch.zeros_like(recv_lo)
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(p_halo[:, R:2 * R].copy()), rank - 1))
        reqs.append(dist.irecv(recv_lo, rank - 1))
    if rank < world - 1:
        reqs.append(dist.isend(torch.from_numpy(p_halo[:, nyl:nyl + R].copy()), rank + 1))
        reqs.append(dist.irecv(recv_hi, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        p_halo[:, :R] = recv_lo.numpy()
    if rank < world - 1:
        p_halo[:, R + nyl:] = recv_hi.numpy()


def _worker(rank, world, port, nsteps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1410_1387_b200 as V
        from synth import fields as SF
        oracle, synth, cfg, wxy, wz, dt = _setup()
        nx, ny, nz, R = cfg["nx"], cfg["ny"], cfg["nz"], cfg["r_xy"]
        y0, nyl = V.slab(ny, rank, world)

        # per-rank model slab == rows of the global model
        mg = [a.numpy() for a in SF.model_planes(cfg, 0, nz)]
        ms = [a.numpy() for a in SF.model_planes(cfg, 0, nz, j0=y0, nyl=nyl)]
        for a, b in zip(mg, ms):
            assert np.array_equal(a[:, y0:y0 + nyl], b)

        # seeded random initial state, each rank generating only its rows
        st = [SF.random_planes(nx, ny, 0, nz, 5, s, 1e-3, j0=y0, nyl=nyl).numpy() for s in range(4)]
        sub = dict(cfg, ny=nyl + 2 * R)
        si, sj, sk = cfg["src"]
        own = y0 <= sj < y0 + nyl
        P = oracle.params(sub, dt, src=(si, sj - y0 + R, sk) if own else None)
        pad = lambda a: np.concatenate([np.zeros((nz, R, nx), np.float32), a, np.zeros((nz, R, nx), np.float32)], axis=1)
        p, qf, pm, qm = (pad(a) for a in st)
        model = [pad(a) for a in ms]
        _exchange(p, R, nyl, rank, world)          # initial halo of u^n
        for n in range(nsteps):
            p, qf, pm, qm, _ = oracle.run(P, wxy, wz, *model, (p, qf, pm, qm), n0=n, nsteps=1)
            for a in (qf, pm, qm):                  # rows outside the slab carry no state
                a[:, :R] = 0
                a[:, R + nyl:] = 0
            p[:, :R] = 0
            p[:, R + nyl:] = 0
            _exchange(p, R, nyl, rank, world)      # p^{n+1} boundary rows to the neighbours
        mine = [a[:, R:R + nyl] for a in (p, qf, pm, qm)]

        # bench.py's N > 1 bootstrap: a real ncclUniqueId from the library on rank 0,
        # identical on every rank after the broadcast; fresh per call; max over ranks
        from paper_1410_1387_b200 import multi
        ids = [multi.broadcast_nccl_id(dist, rank, world) for _ in range(2)]
        assert all(len(i) == 128 for i in ids) and ids[0] != ids[1]
        allids = [None] * world
        dist.all_gather_object(allids, ids[0])
        assert all(i == ids[0] for i in allids)
        assert multi.max_over_ranks(dist, world, float(rank + 1)) == float(world)

        # peer transport bootstrap: each rank connects to the blobs of rank-1 / rank+1,
        # and one rank failing makes every rank fall back (collective decision)
        class MockHandle:
            def __init__(self, fail):
                self.fail, self.got = fail, None

            def ipc_export(self):
                return b"blob-%d" % rank

            def ipc_connect(self, lo, hi):
                self.got = (lo, hi)
                if self.fail:
                    raise RuntimeError("no peer access")

        h = MockHandle(fail=False)
        assert multi.connect_peer(dist, h, rank, world)
        assert h.got == (b"blob-%d" % (rank - 1) if rank > 0 else None,
                         b"blob-%d" % (rank + 1) if rank < world - 1 else None)
        assert not multi.connect_peer(dist, MockHandle(fail=(rank == world - 1)), rank, world)

        gathered = [None] * world
        dist.all_gather_object(gathered, (y0, [m.copy() for m in mine]))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_domain(world):
    nsteps = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nsteps, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from synth import fields as SF
    oracle, synth, cfg, wxy, wz, dt = _setup()
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    model = [a.numpy() for a in SF.model_planes(cfg, 0, nz)]
    st = [SF.random_planes(nx, ny, 0, nz, 5, s, 1e-3).numpy() for s in range(4)]
    ref = oracle.run(oracle.params(cfg, dt), wxy, wz, *model, st, nsteps=nsteps)[:4]
    gathered.sort(key=lambda g: g[0])
    for f in range(4):
        full = np.concatenate([g[1][f] for g in gathered], axis=1)
        assert np.abs(ref[f]).max() > 0
        assert np.array_equal(full, ref[f]), f"field {f}: max diff {np.abs(full - ref[f]).max()}"
