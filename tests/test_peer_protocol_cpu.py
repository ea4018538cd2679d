"""Model check of the fused peer-memory halo protocol.

The multi-process form of the transport cannot run on the single GPU of this
environment, so its ordering logic is checked here on the CPU. The model
replays, per rank, the operation sequence `vti_step` (vti_runtime.cu, vti_transport.cu) enqueues on the
rank's stream:

  step consuming publication j  (peer_pre_step, launch_edge, peer_post_edge):
      wait DATA_lo >= j, wait ACK_lo >= j-1, wait DATA_hi >= j, wait ACK_hi >= j-1
      EDGE: read own halo (parity of j), write neighbours' halo (parity of j+1)
      write nb_lo.ACK_hi = j, nb_lo.DATA_hi = j+1, nb_hi.ACK_lo = j, nb_hi.DATA_lo = j+1
  re-publication (peer_release, peer_publish) after set_fields / reverse:
      write nb.ACK = xseq;  j0 = xseq + 1;  wait ACK >= j0-1;  COPY into nb halo (parity cur);
      write nb.DATA = j0

and checks, for random interleavings of the ranks' streams:
  * no deadlock;
  * every halo read sees exactly the publication it consumes (no stale data,
    no overwrite before the neighbour has read the previous content);
and, for the local group, that the host enqueue order is deadlock-free even if
every stream of every handle shares ONE in-order hardware channel (the
enqueue-order rule: a value-wait may only wait on an earlier-enqueued write).
The adjoint's s1 row exchange between peer ranks (rows_exchange_peer) is checked
the same way at the end of the file.
"""
import random

import pytest

LO, HI = 0, 1
DATA, ACK = 0, 1


class Rank:
    def __init__(self, r, n):
        self.r, self.n = r, n
        self.flags = {(DATA, LO): 0, (DATA, HI): 0, (ACK, LO): 0, (ACK, HI): 0}
        # halo[parity][side] = publication number whose rows are stored there (0 = initial zero state)
        self.halo = [[0, 0], [0, 0]]
        self.xseq = 0
        self.cur = 0
        self.ops = []

    def sides(self):
        return [s for s in (LO, HI) if (s == LO and self.r > 0) or (s == HI and self.r < self.n - 1)]


def nb(ranks, r, side):
    return ranks[r - 1] if side == LO else ranks[r + 1]


def other(side):
    return HI if side == LO else LO


def enqueue_step(ranks, R):
    """peer_pre_step + launch_edge + peer_post_edge (+ interior, which touches no halo)."""
    j = R.xseq
    for s in R.sides():
        R.ops.append(("wait", (DATA, s), j))
        if j >= 1:
            R.ops.append(("wait", (ACK, s), j - 1))
    R.ops.append(("edge", j, R.cur))   # reads halo parity cur (publication j), writes nb halo parity 1-cur (j+1)
    for s in R.sides():
        R.ops.append(("write", s, (ACK, other(s)), j))
        R.ops.append(("write", s, (DATA, other(s)), j + 1))
    R.xseq = j + 1
    R.cur = 1 - R.cur


def enqueue_release(R):
    for s in R.sides():
        R.ops.append(("write", s, (ACK, other(s)), R.xseq))


def enqueue_publish(R):
    R.xseq += 1
    j0 = R.xseq
    for s in R.sides():
        R.ops.append(("wait", (ACK, s), j0 - 1))
        R.ops.append(("copy", s, j0, R.cur))
        R.ops.append(("write", s, (DATA, other(s)), j0))


def ready(ranks, R, op):
    return op[0] != "wait" or R.flags[op[1]] >= op[2]


def execute(ranks, R, op, errors):
    kind = op[0]
    if kind == "edge":
        _, j, par = op
        for s in R.sides():
            if R.halo[par][s] != j:
                errors.append(f"rank {R.r} step reading publication {j} saw {R.halo[par][s]} on side {s}")
        for s in R.sides():
            N = nb(ranks, R.r, s)
            N.halo[1 - par][other(s)] = j + 1
    elif kind == "copy":
        _, s, j0, par = op
        nb(ranks, R.r, s).halo[par][other(s)] = j0
    elif kind == "write":
        _, s, key, v = op
        nb(ranks, R.r, s).flags[key] = v


def run_streams(ranks, rng):
    """Each rank's stream in order; ranks interleave at random. Returns errors (deadlock included)."""
    pcs = [0] * len(ranks)
    errors = []
    while True:
        live = [i for i, R in enumerate(ranks) if pcs[i] < len(R.ops)]
        if not live:
            return errors
        runnable = [i for i in live if ready(ranks, ranks[i], ranks[i].ops[pcs[i]])]
        if not runnable:
            return errors + [f"deadlock at {[(i, ranks[i].ops[pcs[i]]) for i in live]}"]
        i = rng.choice(runnable)
        execute(ranks, ranks[i], ranks[i].ops[pcs[i]], errors)
        pcs[i] += 1


def scenario(n, script, group_order):
    """script: list of ('step', k) / ('republish',) / ('reverse',). Returns ranks with ops enqueued and the
    global host enqueue order (rank, op index) of a local group."""
    ranks = [Rank(r, n) for r in range(n)]
    order = []

    def mark(R, before):
        order.extend((R.r, i) for i in range(before, len(R.ops)))

    for item in script:
        if item[0] == "step":
            for _ in range(item[1]):
                if group_order:
                    for R in ranks:   # edges (with their waits and writes) for every handle, then interiors
                        b = len(R.ops)
                        enqueue_step(ranks, R)
                        mark(R, b)
                else:
                    for R in ranks:
                        enqueue_step(ranks, R)
        else:
            if item[0] == "reverse":
                for R in ranks:
                    R.cur = 1 - R.cur
            for R in ranks:   # every release before any publish
                b = len(R.ops)
                enqueue_release(R)
                mark(R, b)
            for R in ranks:
                b = len(R.ops)
                enqueue_publish(R)
                mark(R, b)
    return ranks, order


SCRIPTS = [
    [("step", 12)],
    [("republish",), ("step", 5)],
    [("step", 3), ("republish",), ("step", 4)],
    [("step", 5), ("reverse",), ("step", 4), ("reverse",), ("step", 2)],
    [("step", 1), ("republish",), ("republish",), ("step", 3), ("reverse",), ("step", 1)],
]


@pytest.mark.parametrize("n", [2, 3, 5])
@pytest.mark.parametrize("si", range(len(SCRIPTS)))
def test_random_interleavings_deliver_every_publication(n, si):
    for seed in range(200):
        ranks, _ = scenario(n, SCRIPTS[si], group_order=False)
        errs = run_streams(ranks, random.Random(seed))
        assert not errs, (seed, errs[:3])


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("si", range(len(SCRIPTS)))
def test_group_enqueue_order_is_deadlock_free_on_one_channel(n, si):
    """Worst case of channel sharing: all handles' operations in ONE in-order queue, in the host
    enqueue order of vti_group_step. Every wait must be satisfied by an earlier operation."""
    ranks, order = scenario(n, SCRIPTS[si], group_order=True)
    assert len(order) == sum(len(R.ops) for R in ranks)
    errors = []
    for r, i in order:
        R = ranks[r]
        op = R.ops[i]
        assert ready(ranks, R, op), f"wait {op} of rank {r} would block the shared channel"
        execute(ranks, R, op, errors)
    assert not errors, errors[:3]


def test_step_ack_waits_are_implied_by_data():
    """In steady state the DATA chain already orders a rank's halo write after the neighbour's
    previous read of that parity (the neighbour writes DATA = j only after the edge launch that read
    publication j-1), so the steps' ACK waits are defence in depth: without them every interleaving
    still delivers every publication."""
    global enqueue_step
    orig = enqueue_step

    def no_ack(ranks, R):
        j = R.xseq
        for s in R.sides():
            R.ops.append(("wait", (DATA, s), j))
        R.ops.append(("edge", j, R.cur))
        for s in R.sides():
            R.ops.append(("write", s, (ACK, other(s)), j))
            R.ops.append(("write", s, (DATA, other(s)), j + 1))
        R.xseq = j + 1
        R.cur = 1 - R.cur

    enqueue_step = no_ack
    try:
        for seed in range(200):
            ranks, _ = scenario(3, [("step", 8)], group_order=False)
            assert not run_streams(ranks, random.Random(seed))
    finally:
        enqueue_step = orig


def test_model_catches_a_missing_publish_ack_wait():
    """The checker is not vacuous: without the ACK wait of a re-publication (after vti_reverse the
    re-published level lands in the parity the neighbour's last step read), some interleaving
    overwrites a halo before the neighbour has read it."""
    global enqueue_publish
    orig = enqueue_publish

    def no_ack(R):
        R.xseq += 1
        j0 = R.xseq
        for s in R.sides():
            R.ops.append(("copy", s, j0, R.cur))
            R.ops.append(("write", s, (DATA, other(s)), j0))

    enqueue_publish = no_ack
    try:
        bad = 0
        for seed in range(300):
            ranks, _ = scenario(3, [("step", 3), ("reverse",), ("step", 2)], group_order=False)
            bad += bool(run_streams(ranks, random.Random(seed)))
        assert bad > 0
    finally:
        enqueue_publish = orig


def test_model_catches_a_wait_before_the_write_in_one_channel():
    """The one-channel check is not vacuous: the first copy-engine version enqueued each handle's
    whole exchange (send, DATA write, then DATA wait) handle by handle, so handle 0's wait came
    before handle 1's write of the same exchange -- the deadlock seen on the GPU."""
    ranks = [Rank(r, 2) for r in range(2)]
    order = []
    for R in ranks:
        s = R.sides()[0]
        R.ops += [("write", s, (DATA, other(s)), 1), ("wait", (DATA, s), 1)]
        order += [(R.r, 0), (R.r, 1)]
    blocked = None
    for r, i in order:
        if not ready(ranks, ranks[r], ranks[r].ops[i]):
            blocked = (r, i)
            break
        execute(ranks, ranks[r], ranks[r].ops[i], [])
    assert blocked == (0, 1)


# ---- the adjoint's s1 rows between multi-process peer ranks (rows_exchange_peer, vti_transport.cu):
# one receive buffer per side; publication j of a rank, enqueued on its stream:
#   per side: wait S1ACK >= j-1; PACK into the neighbour's receive buffer; write nb.S1DATA = j
#   per side: wait S1DATA >= j; UNPACK own receive buffer (must hold exactly j); write nb.S1ACK = j
S1DATA, S1ACK = 2, 3


class S1Rank(Rank):
    def __init__(self, r, n):
        super().__init__(r, n)
        self.flags.update({(S1DATA, LO): 0, (S1DATA, HI): 0, (S1ACK, LO): 0, (S1ACK, HI): 0})
        self.rbuf = [0, 0]       # publication in the receive buffer of each side
        self.consumed = [0, 0]   # last publication unpacked from each side
        self.adj_xseq = 0


def enqueue_s1(R, ack_wait=True):
    R.adj_xseq += 1
    j = R.adj_xseq
    for s in R.sides():
        if ack_wait and j >= 2:
            R.ops.append(("wait", (S1ACK, s), j - 1))
        R.ops.append(("s1pack", s, j))
        R.ops.append(("write", s, (S1DATA, other(s)), j))
    for s in R.sides():
        R.ops.append(("wait", (S1DATA, s), j))
        R.ops.append(("s1unpack", s, j))
        R.ops.append(("write", s, (S1ACK, other(s)), j))


def execute_s1(ranks, R, op, errors):
    if op[0] == "s1pack":
        _, s, j = op
        N = nb(ranks, R.r, s)
        if N.rbuf[other(s)] != N.consumed[other(s)]:
            errors.append(f"rank {R.r} overwrote publication {N.rbuf[other(s)]} in rank {N.r}'s buffer unread")
        N.rbuf[other(s)] = j
    elif op[0] == "s1unpack":
        _, s, j = op
        if R.rbuf[s] != j:
            errors.append(f"rank {R.r} unpacking publication {j} from side {s} found {R.rbuf[s]}")
        R.consumed[s] = j
    else:
        execute(ranks, R, op, errors)


def run_s1(ranks, rng):
    pcs = [0] * len(ranks)
    errors = []
    while True:
        live = [i for i, R in enumerate(ranks) if pcs[i] < len(R.ops)]
        if not live:
            return errors
        runnable = [i for i in live if ready(ranks, ranks[i], ranks[i].ops[pcs[i]])]
        if not runnable:
            return errors + [f"deadlock at {[(i, ranks[i].ops[pcs[i]]) for i in live]}"]
        i = rng.choice(runnable)
        execute_s1(ranks, ranks[i], ranks[i].ops[pcs[i]], errors)
        pcs[i] += 1


@pytest.mark.parametrize("n", [2, 3, 5])
def test_s1_exchange_delivers_every_publication(n):
    """vti_step_adjoint on peer ranks publishes once per call plus once per chained step; every
    interleaving of the ranks' streams is deadlock-free and unpacks exactly the publication it
    expects, with no receive buffer overwritten before it was unpacked."""
    for seed in range(300):
        ranks = [S1Rank(r, n) for r in range(n)]
        for _ in range(9):
            for R in ranks:
                enqueue_s1(R)
        errs = run_s1(ranks, random.Random(seed))
        assert not errs, (seed, errs[:3])


def test_s1_model_catches_a_missing_ack_wait():
    bad = 0
    for seed in range(300):
        ranks = [S1Rank(r, 3) for r in range(3)]
        for _ in range(6):
            for R in ranks:
                enqueue_s1(R, ack_wait=False)
        bad += bool(run_s1(ranks, random.Random(seed)))
    assert bad > 0
