"""Host logic of the N > 1 bench path, on CPU (no GPU needed).

* multi.sync_or_die: reads the handle's ``stream`` PROPERTY (an int, vti_stream) -- the
  round-1 bug called it -- polls until done, calls sync(); exits loudly on a timeout.
* multi.max_over_ranks: the max over a world-size-2 gloo group.
* bench.py's default workload is BASELINE C4 (2048 x 2048 x 1024, strong scaling) at every N,
  and its explicit configs keep their stated scaling.
"""
import os
import socket
import sys
import types

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1410_1387_b200 import multi  # noqa: E402


class FakeHandle:
    halo_transport = "peer"

    def __init__(self):
        self.synced = 0

    @property
    def stream(self):   # like VTI.stream: an int, not a method
        return 0xDEAD

    def sync(self):
        self.synced += 1


def test_sync_or_die_uses_stream_property(monkeypatch):
    import torch
    seen = []

    class FakeExternalStream:
        def __init__(self, ptr, device=None):
            assert isinstance(ptr, int)
            seen.append(ptr)
            self.n = 0

        def query(self):
            self.n += 1
            return self.n >= 3   # done on the third poll

    monkeypatch.setattr(torch.cuda, "ExternalStream", FakeExternalStream)
    h = FakeHandle()
    multi.sync_or_die(h, 5.0)
    assert seen == [0xDEAD] and h.synced == 1


def test_sync_or_die_times_out_loudly(capsys):
    h = FakeHandle()
    codes = []
    multi.sync_or_die(h, 0.05, "warm-up", query=lambda: False, die=codes.append)
    assert codes == [3] and h.synced == 0
    assert "warm-up did not complete" in capsys.readouterr().err


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, multi.max_over_ranks(dist, world, 1.5 + rank, device="cpu")))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 2.5, 1: 2.5}


def _bench_args(*argv):
    import bench
    old = sys.argv
    sys.argv = ["bench.py", *argv]
    try:
        return bench, bench.parse()
    finally:
        sys.argv = old


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bench_default_workload_is_c4_strong(world):
    bench, args = _bench_args("--gpus", str(world))
    assert args.config == "C4" and args.reps >= 3 and args.warmup >= 3
    cfg, scaling = bench.workload(args, world)
    assert (cfg["name"], cfg["nx"], cfg["ny"], cfg["nz"]) == ("C4", 2048, 2048, 1024)
    assert (cfg["r_xy"], cfg["r_z"], cfg["steps"]) == (4, 4, 200) and scaling == "strong"
    d = bench.describe(cfg, world, scaling)
    assert d["workload"].startswith("C4: 2048x2048x1024")
    assert ">> 126 MB L2" in d["l2_flush"]


def test_bench_explicit_configs_keep_their_scaling():
    bench, args = _bench_args("--config", "C5")
    cfg, scaling = bench.workload(args, 4)
    assert scaling == "weak" and (cfg["nx"], cfg["ny"], cfg["nz"]) == (1024, 4096, 1024)
    bench, args = _bench_args("--config", "C3")
    cfg, scaling = bench.workload(args, 8)
    assert scaling == "strong" and (cfg["nx"], cfg["ny"], cfg["nz"]) == (1024, 1024, 512)
    bench, args = _bench_args("--config", "C1")
    cfg, scaling = bench.workload(args, 1)
    assert "L2-resident" in bench.describe(cfg, 1, scaling)["l2_flush"]


def test_bench_watchdog_fires_and_cancels():
    """bench.Watchdog: cancelled on exit; otherwise it ends the process with code 4."""
    import subprocess
    import bench
    with bench.Watchdog(0.5, "quick region"):
        pass
    code = ("import sys, time; sys.path.insert(0, %r); import bench\n"
            "with bench.Watchdog(0.2, 'stuck region'):\n    time.sleep(5)\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
    assert r.returncode == 4 and "stuck region did not finish" in r.stderr
