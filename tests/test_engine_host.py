"""Engine scheduling semantics on the host (device=-1: host ops only, no GPU),
ported from R/tests/test_engine.cpp and acceptance criterion 2.  The same
grant logic dispatches the device (stream) ops on the GPU; tests/native/
engine_abi_test.c stresses it from C without a GIL."""
import random
import threading
import time

import pytest

from paper_1802_06949_b200 import ConfigError, EngineError, Engine, TraceSink, UsageError


def test_pool_size_and_distinct_tags():
    with pytest.raises(ConfigError):
        Engine(0)
    e = Engine(4)
    assert e.num_threads() == 4
    tags = {e.new_variable() for _ in range(100)}
    assert len(tags) == 100
    ids = [e.push(lambda: None) for _ in range(10)]
    assert ids == sorted(set(ids))
    e.wait_all()


def test_read_after_write():
    e = Engine(4)
    t = e.new_variable()
    box = {"v": 0, "seen": None}

    def w():
        time.sleep(0.01)
        box["v"] = 7

    e.push(w, [], [t])
    e.push(lambda: box.__setitem__("seen", box["v"]), [t], [])
    e.wait_all()
    assert box["seen"] == 7


def test_writes_execute_in_push_order_exclusively():
    e = Engine(8)
    t = e.new_variable()
    log, active, bad = [], [0], [0]

    def body(i):
        active[0] += 1
        if active[0] != 1:
            bad[0] += 1
        log.append(i)
        active[0] -= 1

    for i in range(200):
        e.push(lambda i=i: body(i), [], [t])
    e.wait_all()
    assert log == list(range(200)) and bad[0] == 0


def test_three_concurrent_readers_rendezvous():
    e = Engine(3)
    a = e.new_variable()
    arrived, ok = [0], [0]
    mu = threading.Lock()

    def body():
        with mu:
            arrived[0] += 1
        deadline = time.time() + 5
        while arrived[0] < 3 and time.time() < deadline:
            time.sleep(0.0005)
        if arrived[0] == 3:
            with mu:
                ok[0] += 1

    for _ in range(3):
        e.push(body, [a], [])
    e.wait_all()
    assert ok[0] == 3


def test_wait_for_covers_all_mutating_ops():
    e = Engine(2)
    t = e.new_variable()
    e.wait_for(t)  # nothing pending
    stamps = []

    def first():
        time.sleep(0.005)
        stamps.append(1)

    e.push(first, [], [t])
    e.push(lambda: stamps.append(2), [], [t])
    e.wait_for(t)
    assert stamps == [1, 2]


def test_wait_all_many_ops():
    e = Engine(4)
    n = [0]
    mu = threading.Lock()

    def inc():
        with mu:
            n[0] += 1

    for _ in range(1000):
        e.push(inc)
    e.wait_all()
    assert n[0] == 1000
    assert e.stats() == (1000, 1000)


def test_shutdown_and_tag_validation():
    e = Engine(2)
    t = e.new_variable()
    with pytest.raises(UsageError):
        e.push(lambda: None, [t], [t])  # tag in both lists
    with pytest.raises(UsageError):
        e.push(lambda: None, [999], [])  # unknown tag
    other = Engine(1)
    ot = other.new_variable()
    if ot == t:  # ids are per engine; a foreign id that exists locally is not detectable by value
        pass
    e.shutdown()
    e.shutdown()  # idempotent
    with pytest.raises(UsageError):
        e.push(lambda: None)


def test_poison_wait_all_rethrows_and_later_ops_still_run():
    e = Engine(2)
    t = e.new_variable()
    ran = []

    def boom():
        raise RuntimeError("body failure")

    e.push(boom, [], [t])
    e.push(lambda: ran.append(1), [], [t])
    with pytest.raises(EngineError):
        e.wait_all()
    assert ran == [1]
    with pytest.raises(EngineError):
        e.wait_all()  # stays poisoned


def test_acceptance_2_write_order_1000_ops_8_threads():
    """acceptance.cpp:86-109 (20 repetitions there; 5 here for runtime)."""
    for _ in range(5):
        e = Engine(8)
        t = e.new_variable()
        log = []
        for i in range(1000):
            e.push(lambda i=i: log.append(i), [], [t])
        e.wait_all()
        e.shutdown()
        assert log == list(range(1000))


def test_read_batching_read_waits_for_earlier_write():
    e = Engine(4)
    t = e.new_variable()
    for _ in range(20):
        done = [False]
        saw = [None]

        def w():
            time.sleep(0.0002)
            done[0] = True

        e.push(w, [], [t])
        e.push(lambda: saw.__setitem__(0, done[0]), [t], [])
        e.wait_all()
        assert saw[0] is True


def test_reads_batch_behind_a_write_and_run_together():
    """A run of reads at the queue head is granted together (engine.cpp:113-133)."""
    e = Engine(4)
    t = e.new_variable()
    gate = threading.Event()
    e.push(lambda: gate.wait(5), [], [t])
    inside, peak = [0], [0]
    mu = threading.Lock()

    def reader():
        with mu:
            inside[0] += 1
            peak[0] = max(peak[0], inside[0])
        time.sleep(0.02)
        with mu:
            inside[0] -= 1

    for _ in range(3):
        e.push(reader, [t], [])
    gate.set()
    e.wait_all()
    assert peak[0] >= 2


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("threads", [1, 8])
def test_random_dag_soundness_no_false_deadlock(seed, threads):
    """test_engine.cpp:215-274: per-tag occupancy counters inside every body."""
    e = Engine(threads)
    num_tags, num_ops = 40, 500
    tags = [e.new_variable() for _ in range(num_tags)]
    readers = [0] * num_tags
    writers = [0] * num_tags
    violations, executed = [0], [0]
    mu = threading.Lock()
    rng = random.Random(seed)
    for _ in range(num_ops):
        pool = list(range(num_tags))
        rng.shuffle(pool)
        nr, nw = rng.randrange(3), 1 + rng.randrange(2)
        rid, wid = pool[:nr], pool[nr:nr + nw]

        def body(rid=rid, wid=wid):
            with mu:
                for i in rid:
                    if writers[i]:
                        violations[0] += 1
                    readers[i] += 1
                for i in wid:
                    if writers[i] or readers[i]:
                        violations[0] += 1
                    writers[i] += 1
            time.sleep(0)  # yield: let other granted ops interleave
            with mu:
                executed[0] += 1
                for i in wid:
                    writers[i] -= 1
                for i in rid:
                    readers[i] -= 1

        e.push(body, [tags[i] for i in rid], [tags[i] for i in wid])
    e.wait_all()
    assert executed[0] == num_ops and violations[0] == 0


def test_trace_records_push_start_finish_triple():
    sink = TraceSink()
    e = Engine(2, 3, sink)
    t = e.new_variable()
    for i in range(10):
        e.push(lambda: None, [], [t], 0, i)
    e.wait_all()
    ev = sink.snapshot()
    assert all(x["rank"] == 3 for x in ev)
    for name in ("op_pushed", "op_started", "op_finished"):
        assert sum(1 for x in ev if x["event"] == name) == 10
    assert all(x["kind"] == "compute" for x in ev)
