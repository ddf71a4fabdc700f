"""run_synthetic (runner.cpp:47-135 over the GPU path): metrics file in the
reference schema and a replay-consistent trace (port of
test_harness.cpp:64-114)."""
import json
from collections import defaultdict

import pytest

pytestmark = pytest.mark.gpu

from paper_1802_06949_b200.metrics import metrics_from_json, run_synthetic  # noqa: E402


@pytest.mark.parametrize("mode", ["funnel", "depcha", "concom"])
def test_trace_files_are_replay_consistent(gpu, tmp_path, mode):
    trace, mpath = tmp_path / "t.jsonl", tmp_path / "m.json"
    m = run_synthetic(mode=mode, workers=2, engine_threads=4, outstanding=2, epochs=2, steps_per_epoch=2,
                      sizes=[64, 1000, 4096, 7, 300, 2048], backward_ms=0.2, trace_path=str(trace),
                      metrics_path=str(mpath))
    assert m.ok(), m.error
    assert len(m.epoch_times_s) == 2 and all(t > 0 for t in m.epoch_times_s)
    back = metrics_from_json(mpath.read_text())
    assert back == m
    assert m.max_concurrent_collectives >= 1
    s0, s1 = m.b200["weight_checksums"]
    assert s0 == s1  # every rank trains the same weights
    ops, colls, enq = defaultdict(list), defaultdict(list), defaultdict(int)
    last_t = defaultdict(int)
    for line in trace.read_text().splitlines():
        j = json.loads(line)
        ev, rank, t = j["event"], j["rank"], j["t_us"]
        assert t >= last_t[rank]  # per-worker t_us nondecreasing
        last_t[rank] = t
        if ev.startswith("op_"):
            ops[(rank, j["op"])].append(ev)
        else:
            slot = (j["comm"], j["seq"])
            colls[slot].append(ev)
            if ev == "coll_enqueued":
                enq[slot] += 1
    assert ops and colls
    for evs in ops.values():
        assert evs == ["op_pushed", "op_started", "op_finished"]
    for evs in colls.values():
        seen = False
        for ev in evs:
            seen |= ev == "coll_matched"
            if ev == "coll_done":
                assert seen
    assert set(enq.values()) == {2}  # every rendezvous carries exactly R enqueues


def test_failed_run_reports_primary_error(gpu):
    # 2 workers, ConCom with outstanding 0 is a config error before any work
    from paper_1802_06949_b200 import ConfigError
    with pytest.raises(ConfigError, match="outstanding"):
        run_synthetic(mode="concom", outstanding=0)
