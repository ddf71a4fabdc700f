"""The cross-rank matching ledger (host logic of the Transport), CPU only.
Ports R/tests/test_collective.cpp's matching / mismatch / watchdog /
independence / trace cases onto the ledger-only transport (rank threads), and
runs the POSIX-shm ledger across 2 processes (gloo plumbing)."""
import multiprocessing as mp
import socket
import threading
import time

import pytest

from kvhelpers import on_ranks
from paper_1802_06949_b200 import (ConfigError, DeadlockTimeout, MismatchError, TraceSink, Transport,
                                   UsageError)

F32 = 1


def ar(t, comm, rank, count, key=-1):
    t.allreduce_sum(comm, rank, 0, trace_key=key, dtype=F32, count=count)


def test_construction():
    with pytest.raises(ConfigError):
        Transport.ledger_only(0, 1000)
    with pytest.raises(ConfigError):
        Transport.ledger_only(4, 0)
    t = Transport.ledger_only(4, 1000)
    assert t.num_ranks() == 4 and t.num_communicators() == 1


def test_single_rank_degenerates():
    t = Transport.ledger_only(1, 1000)
    ar(t, 0, 0, 2)
    t.broadcast(0, 0, 0, 0, dtype=F32, count=2)
    t.barrier(0, 0)


def test_kind_mismatch_names_both_calls():
    t = Transport.ledger_only(2, 5000)
    msgs = {}

    def rank(r):
        try:
            if r == 0:
                ar(t, 0, 0, 6)
            else:
                t.barrier(0, 1)
        except MismatchError as e:
            msgs[r] = str(e)

    on_ranks(2, rank)
    assert msgs[0] == msgs[1]
    assert "allreduce(count=6)" in msgs[0] and "barrier" in msgs[0]


def test_count_mismatch():
    t = Transport.ledger_only(2, 5000)
    n = []

    def rank(r):
        try:
            ar(t, 0, r, 4 if r == 0 else 5)
        except MismatchError:
            n.append(r)

    on_ranks(2, rank)
    assert sorted(n) == [0, 1]


def test_broadcast_root_disagreement_and_invalid_root():
    t = Transport.ledger_only(2, 5000)
    n = []

    def rank(r):
        try:
            t.broadcast(0, r, r, 0, dtype=F32, count=3)
        except MismatchError:
            n.append(r)

    on_ranks(2, rank)
    assert sorted(n) == [0, 1]
    with pytest.raises(UsageError):
        Transport.ledger_only(2, 5000).broadcast(0, 0, 5, 0, dtype=F32, count=3)


def test_failure_latch_fails_later_calls_fast():
    t = Transport.ledger_only(2, 5000)
    on_ranks(2, lambda r: pytest.raises(MismatchError, ar, t, 0, r, 3 + r))
    t0 = time.time()
    with pytest.raises(MismatchError):
        t.barrier(0, 0)
    assert time.time() - t0 < 1.0


def test_missing_rank_trips_watchdog_with_report():
    t = Transport.ledger_only(2, 200)
    with pytest.raises(DeadlockTimeout) as e:
        t.barrier(0, 0)
    assert "rank 0: barrier" in str(e.value) and "rank 1: no call issued" in str(e.value)


def test_different_communicators_never_match():
    t = Transport.ledger_only(2, 200)
    extra = t.new_communicator()
    n = []

    def rank(r):
        try:
            if r == 0:
                t.barrier(0, 0)
            else:
                ar(t, extra, 1, 2)
        except DeadlockTimeout:
            n.append(r)

    on_ranks(2, rank)
    assert sorted(n) == [0, 1]


def test_communicator_setup_only():
    t = Transport.ledger_only(2, 1000)
    assert t.new_communicator() == 1 and t.new_communicator() == 2
    assert t.num_communicators() == 3
    on_ranks(2, lambda r: t.barrier(0, r))
    with pytest.raises(UsageError):
        t.new_communicator()


def test_eight_independent_sequence_spaces():
    t = Transport.ledger_only(2, 5000)
    comms = [t.new_communicator() for _ in range(8)]

    def rank(r):
        for c in range(8):
            for _ in range(c + 1):
                ar(t, comms[c], r, c + 1)

    on_ranks(2, rank)


def test_independence_with_arrival_skew():
    t = Transport.ledger_only(2, 5000)
    for _ in range(3):
        t.new_communicator()

    def rank(r):
        for _ in range(10):
            if r == 1:
                time.sleep(0.02)
            ar(t, 0, r, 4)

    on_ranks(2, rank)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_matching_fuzz_sequences_identical(seed):
    """test_collective.cpp:249-291 shape: R=3, 30 calls with jitter; every rank
    sees the same (comm, seq) -> signature pairing."""
    import random
    sink = TraceSink()
    t = Transport.ledger_only(3, 5000, sink)
    sched = [(random.Random(seed + i).choice([0, 1]), 1 + (i * 5) % 9) for i in range(30)]
    t.new_communicator()

    def rank(r):
        rng = random.Random(seed * 7 + r)
        for i, (comm, n) in enumerate(sched):
            time.sleep(rng.random() * 0.002)
            ar(t, comm, r, n, key=i)

    on_ranks(3, rank)
    per = {}
    for e in sink.snapshot():
        if e["event"] == "coll_enqueued":
            per.setdefault(e["rank"], []).append((e["comm"], e["seq"], e["key"]))
    assert per[0] == per[1] == per[2]


def test_concurrent_same_rank_calls_sequenced_by_arrival():
    t = Transport.ledger_only(2, 5000)
    done = []
    th = [threading.Thread(target=lambda r=r: (ar(t, 0, r, 3), done.append(r))) for r in (0, 0, 1, 1)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert len(done) == 4


def test_injected_latency_delays_every_rendezvous():
    sink = TraceSink()
    t = Transport.ledger_only(2, 5000, sink)
    t.set_inject_latency(20000)
    t0 = time.time()
    on_ranks(2, lambda r: [ar(t, 0, r, 4) for _ in range(3)])
    assert time.time() - t0 >= 0.06
    assert sink.gauges()[0] == 1


def test_trace_lifecycle():
    sink = TraceSink()
    t = Transport.ledger_only(2, 5000, sink)
    on_ranks(2, lambda r: ar(t, 0, r, 4, key=5))
    ev = sink.snapshot()
    assert all(e["comm"] == 0 and e["seq"] == 0 and e["kind"] == "allreduce" and e["key"] == 5 for e in ev)
    names = [e["event"] for e in ev]
    assert names.count("coll_enqueued") == 2 and names.count("coll_matched") == 1 and names.count("coll_done") == 2


# ------------------------------------------------- 2 processes, shm ledger

def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(case):
    import mp_ledger_worker as w
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=w.run, args=(r, 2, port, case, q)) for r in range(2)]
    for p in ps:
        p.start()
    outs = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=lambda o: o["rank"])


def test_shm_ledger_two_processes_identical_order():
    outs = _spawn("order")
    assert "error" not in outs[0] and "error" not in outs[1]
    ev0 = [e for e in outs[0]["events"]]
    ev1 = [e for e in outs[1]["events"]]
    assert [e[1:] for e in ev0] == [e[1:] for e in ev1]
    assert len(ev0) == 20 + 7 + 1


def test_shm_ledger_two_processes_mismatch():
    outs = _spawn("mismatch")
    assert [o.get("error") for o in outs] == ["MismatchError", "MismatchError"]
    assert "allreduce(count=4)" in outs[0]["message"] and "allreduce(count=5)" in outs[0]["message"]


def test_shm_ledger_two_processes_deadlock_report():
    outs = _spawn("deadlock")
    assert outs[0].get("error") == "DeadlockTimeout"
    assert "rank 1: no call issued" in outs[0]["message"]
