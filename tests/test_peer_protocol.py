"""Model check of the peer-transport flag protocol (store.cu k_put / digest_pull, peer.cu
AGG) on the host: the exact wait/raise conditions of the C code, executed by M simulated
ranks in random interleavings of the synchronous schedule (Alg. 1 guards).

Checks, for FLIP and COPY pulls, N in {1, 2, 3, 5}, M in {2, 3, 4}:
  * progress: the protocol never deadlocks (some rank can always take its next step);
  * a push always lands in the receiver's ACTUAL back buffer (the sender computes the
    index from its own front: same schedule on every rank);
  * a push never overwrites rows the receiver has not consumed yet;
  * a flip / copy exposes exactly the version every owner pushed (no torn levels);
  * the rank-order AGG slot protocol never rewrites a slot a peer may still read.
"""
import random

import pytest

from paper_2206_00057_b200.dist import Schedule


def ops_of(N, R, fresh=False):
    s = Schedule(N)
    out = []
    for e in range(1, R + 1):
        if fresh:   # zero staleness: push then pull in the same epoch (engine.forward_fresh)
            out += [("push", e), ("pull", e + 1), ("agg", e)]
            continue
        if s.pull(e):
            out.append(("pull", e))
        if s.push(e):
            out.append(("push", e))
        out.append(("agg", e))
    return out


class Rank:
    def __init__(self, r, M, ops):
        self.r, self.ops, self.i = r, ops, 0
        self.front, self.ver, self.last_pull = 0, [0, 0], 0
        self.pulled = 0                          # window word kWinPulled
        self.arrived = [0] * M                   # window words kWinArrived[src]
        self.data = [[0] * M, [0] * M]           # version of each owner's segment per buffer
        self.ar_ready = [0] * M                  # window words kWinArReady[src]
        self.ar_seq = 0
        self.slot_writer_seq = [0, 0]            # seq whose data sits in my AGG slot (parity)
        self.pending_reduce = None               # (seq) published but not yet reduced

    def done(self):
        return self.i >= len(self.ops) and self.pending_reduce is None


def step(ranks, r, mode, M):
    """Try rank r's next step; return True if it made progress."""
    me = ranks[r]
    if me.pending_reduce is not None:            # k_ar_reduce: wait for every ar_ready >= seq
        seq = me.pending_reduce
        if any(me.ar_ready[k] < seq for k in range(M)):
            return False
        for k in range(M):                       # reads every rank's slot of parity seq & 1
            assert ranks[k].slot_writer_seq[seq & 1] == seq, "AGG slot rewritten too early"
        me.pending_reduce = None
        return True
    if me.i >= len(me.ops):
        return False
    op, e = me.ops[me.i]
    if op == "push":
        back = 1 - me.front
        if any(ranks[k].pulled < me.last_pull for k in range(M) if k != r):
            return False                          # k_put's per-block wait
        assert e > me.ver[0] and e > me.ver[1]
        for k in range(M):
            if k == r:
                continue
            rk = ranks[k]
            assert back == 1 - rk.front, "push would land in the receiver's front buffer"
            if mode == "copy":   # rows of the previous push were copied out already
                assert rk.data[back][r] == rk.data[rk.front][r], "unconsumed rows overwritten"
            else:                # FLIP: the back buffer holds rows the receiver no longer reads
                assert rk.data[back][r] <= rk.data[rk.front][r]
            rk.data[back][r] = e
            rk.arrived[r] = e                     # last block: fence + st.release.sys
        me.ver[back] = e
    elif op == "pull":
        back = 1 - me.front
        assert me.ver[back] < e
        if me.ver[back] > me.ver[me.front]:
            v = me.ver[back]
            if any(me.arrived[k] < v for k in range(M) if k != r):
                return False                      # flag_sync wait before the flip / copy
            assert all(me.data[back][k] == v for k in range(M) if k != r), "torn level"
            if mode == "flip":
                me.front = back
            else:
                me.data[me.front] = list(me.data[back])
                me.ver[me.front] = v
        me.pulled = e
        me.last_pull = e
    else:  # agg: k_ar_publish (slot seq & 1, then raise ar_ready[me] everywhere)
        me.ar_seq += 1
        seq = me.ar_seq
        me.slot_writer_seq[seq & 1] = seq
        for k in range(M):
            ranks[k].ar_ready[r] = seq
        me.pending_reduce = seq
    me.i += 1
    return True


@pytest.mark.parametrize("mode", ["flip", "copy"])
@pytest.mark.parametrize("M,N,fresh", [(2, 1, False), (3, 2, False), (4, 3, False),
                                       (3, 5, False), (2, 3, False), (3, 1, True),
                                       (4, 1, True)])
def test_protocol_random_interleavings(mode, M, N, fresh):
    R = 13
    for seed in range(60):
        rng = random.Random(seed * 31 + M * 7 + N)
        ranks = [Rank(r, M, ops_of(N, R, fresh)) for r in range(M)]
        speed = [rng.uniform(0.1, 1.0) for _ in range(M)]   # some ranks much slower
        while not all(x.done() for x in ranks):
            live = [r for r in range(M) if not ranks[r].done()]
            order = sorted(live, key=lambda r: -speed[r] * rng.random())
            if not any(step(ranks, r, mode, M) for r in order):
                raise AssertionError(f"deadlock (seed {seed}) at ops "
                                     f"{[ranks[r].ops[ranks[r].i] if ranks[r].i < len(ranks[r].ops) else None for r in range(M)]}")
        for x in ranks:
            assert x.last_pull == (R + 1 if fresh else (R // N) * N)
