"""collsim-metrics-v1 round trip and error priority (ports of
test_harness.cpp:36-61 and runner.cpp:37-43); CPU only."""
import json

import pytest

from paper_1802_06949_b200 import ConfigError
from paper_1802_06949_b200.metrics import (Metrics, metrics_from_json, metrics_to_json, primary_error,
                                           SCHEMA)


def _sample():
    return Metrics(mode="depcha", model="resnet50", workers=4, engine_threads=4, outstanding=1, epochs=2,
                   global_batch=256, seed=7, epoch_times_s=[0.5, 0.25], final_train_loss=1.25,
                   test_accuracy=0.5, max_concurrent_collectives=1, compute_overlap_observed=True,
                   b200={"devices": 4})


def test_round_trip():
    m = _sample()
    back = metrics_from_json(metrics_to_json(m))
    assert back == m
    assert back.ok()


def test_schema_layout_matches_reference_writer():
    j = json.loads(metrics_to_json(_sample()))
    assert j["schema"] == SCHEMA
    assert j["error"] is None and j["error_classes"] == []  # metrics.cpp:36-41
    text = metrics_to_json(_sample())
    keys = [line.split('"')[1] for line in text.splitlines() if line.startswith('  "')]
    assert keys == sorted(keys)  # nlohmann object keys are ordered
    failed = metrics_from_json(metrics_to_json(Metrics(mode="concom", error="MismatchError",
                                                       error_classes=["DeadlockTimeout", "MismatchError"])))
    assert not failed.ok() and failed.error == "MismatchError"


def test_rejects_bad_input():
    with pytest.raises(ConfigError, match="invalid JSON"):
        metrics_from_json("{")
    with pytest.raises(ConfigError, match="unrecognized schema"):
        metrics_from_json('{"schema":"nope"}')
    j = json.loads(metrics_to_json(_sample()))
    del j["workers"]
    with pytest.raises(ConfigError, match="missing or mistyped"):
        metrics_from_json(json.dumps(j))
    j = json.loads(metrics_to_json(_sample()))
    j["workers"] = "four"
    with pytest.raises(ConfigError, match="missing or mistyped"):
        metrics_from_json(json.dumps(j))


def test_primary_error_priority():
    assert primary_error([]) == ""
    assert primary_error(["EngineError", "UsageError"]) == "UsageError"
    assert primary_error(["DeadlockTimeout", "MismatchError", "UsageError"]) == "MismatchError"
    assert primary_error(["CudaError", "EngineError"]) == "EngineError"


def test_run_config_validation_before_any_work():
    """runner.cpp:16-34 `validate`: every bad run configuration is a
    ConfigError raised before a transport or a GPU is touched."""
    from paper_1802_06949_b200.metrics import run_synthetic
    bad = [dict(workers=0), dict(engine_threads=0), dict(epochs=0), dict(global_batch=0),
           dict(workers=3, global_batch=64), dict(mode="concom", outstanding=0), dict(inject_latency_us=-1)]
    msgs = ["workers", "engine-threads", "epochs", "divide evenly", "divide evenly", "outstanding", "latency"]
    for kw, msg in zip(bad, msgs):
        with pytest.raises(ConfigError, match=msg):
            run_synthetic(**kw)
