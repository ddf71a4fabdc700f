"""`collsim-metrics-v1` from the GPU path.

The reference writes one metrics file per run (R/core/src/metrics.cpp:21-44,
parsed back by metrics_from_json 46-82) and fills it in run_scenario
(R/core/src/runner.cpp:47-135).  This module emits the same schema -- same
field names, types and null convention, keys in nlohmann's sorted order with
indent 2 -- so the reference's compare tool and its replay checks can read a
B200 run.  B200-only details go under an extra "b200" object, which the
reference parser ignores.

run_synthetic() is the run_scenario analogue: rank threads over the local
transport (one process, the ranks sharing one GPU), each with its own engine
and the native synthetic-backward trainer (trainer.cpp), with a trace sink.
"""
from __future__ import annotations

import json
import threading
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

from ._lib import ConfigError, CsError

SCHEMA = "collsim-metrics-v1"


@dataclass
class Metrics:
    """R/core/include/collsim/metrics.hpp fields (metrics.cpp:21-44)."""
    mode: str = ""
    model: str = ""
    workers: int = 0
    engine_threads: int = 0
    outstanding: int = 0
    epochs: int = 0
    global_batch: int = 0
    seed: int = 0
    epoch_times_s: list = field(default_factory=list)
    final_train_loss: float = 0.0
    test_accuracy: float = 0.0
    max_concurrent_collectives: int = 0
    compute_overlap_observed: bool = False
    error: str = ""
    error_classes: list = field(default_factory=list)
    b200: dict = field(default_factory=dict)

    def ok(self) -> bool:
        return not self.error


def metrics_to_json(m: Metrics) -> str:
    """metrics.cpp:21-44: schema tag, every field, error null when empty."""
    j = {
        "schema": SCHEMA, "mode": m.mode, "model": m.model, "workers": int(m.workers),
        "engine_threads": int(m.engine_threads), "outstanding": int(m.outstanding), "epochs": int(m.epochs),
        "global_batch": int(m.global_batch), "seed": int(m.seed),
        "epoch_times_s": [float(t) for t in m.epoch_times_s], "final_train_loss": float(m.final_train_loss),
        "test_accuracy": float(m.test_accuracy), "max_concurrent_collectives": int(m.max_concurrent_collectives),
        "compute_overlap_observed": bool(m.compute_overlap_observed), "error": m.error or None,
        "error_classes": list(m.error_classes),
    }
    if m.b200:
        j["b200"] = m.b200
    return json.dumps(j, indent=2, sort_keys=True)


def metrics_from_json(text: str) -> Metrics:
    """metrics.cpp:46-82, same ConfigError messages."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(-1, f"metrics: invalid JSON: {e}") from None
    if not isinstance(j, dict) or j.get("schema", "") != SCHEMA:
        raise ConfigError(-1, "metrics: unrecognized schema")
    try:
        def get(k, typ):
            v = j[k]
            if typ is float and isinstance(v, int) and not isinstance(v, bool):
                v = float(v)
            if typ is int and (isinstance(v, bool) or not isinstance(v, int)):
                raise TypeError(k)
            if typ is not int and not isinstance(v, typ):
                raise TypeError(k)
            return v

        m = Metrics(mode=get("mode", str), model=get("model", str), workers=get("workers", int),
                    engine_threads=get("engine_threads", int), outstanding=get("outstanding", int),
                    epochs=get("epochs", int), global_batch=get("global_batch", int), seed=get("seed", int),
                    epoch_times_s=[float(x) for x in get("epoch_times_s", list)],
                    final_train_loss=get("final_train_loss", float), test_accuracy=get("test_accuracy", float),
                    max_concurrent_collectives=get("max_concurrent_collectives", int),
                    compute_overlap_observed=get("compute_overlap_observed", bool),
                    error="" if j["error"] is None else get("error", str),
                    error_classes=[str(x) for x in get("error_classes", list)], b200=j.get("b200", {}))
    except (KeyError, TypeError, ValueError) as e:
        raise ConfigError(-1, f"metrics: missing or mistyped field: {e}") from None
    return m


def write_metrics(m: Metrics, path) -> None:
    Path(path).write_text(metrics_to_json(m) + "\n")


def error_priority(cls: str) -> int:
    """runner.cpp:37-43: the class that wins the primary "error" slot."""
    return {"MismatchError": 5, "DeadlockTimeout": 4, "UsageError": 3, "EngineError": 2}.get(cls, 1)


def primary_error(classes: Sequence[str]) -> str:
    err = ""
    for c in classes:
        if not err or error_priority(c) > error_priority(err):
            err = c
    return err


def run_synthetic(mode: str = "depcha", workers: int = 2, engine_threads: int = 4, outstanding: int = 2,
                  epochs: int = 2, steps_per_epoch: int = 3, sizes: Sequence[int] = (4096,) * 8,
                  bucket_bytes: int = 0, seed: int = 1, global_batch: int = 64, momentum: float = 0.0,
                  backward_ms: float = 0.0, watchdog_ms: int = 30000, model_name: str = "synthetic",
                  trace_path: str | None = None, metrics_path: str | None = None, device: int = 0,
                  inject_latency_us: int = 0, lr: float = 0.1) -> Metrics:
    """runner.cpp:47-135 over the GPU path: validate, one transport + trace
    sink, communicators for ConCom, rank threads each running the native
    trainer loop shape, then the metrics (epoch wall time averaged over
    workers, gauges from the sink, the primary error by priority).  The rank
    threads share `device` (the reference's ranks share one host); one
    process per GPU is the NCCL / NVLink transport's job."""
    from . import api
    if workers < 1:
        raise ConfigError(-1, "run: workers must be >= 1")
    if engine_threads < 1:
        raise ConfigError(-1, "run: engine-threads must be >= 1")
    if epochs < 1:
        raise ConfigError(-1, "run: epochs must be >= 1")
    if global_batch < 1 or global_batch % workers:
        raise ConfigError(-1, "run: global batch size must divide evenly across workers")
    if mode == "concom" and outstanding < 1:
        raise ConfigError(-1, "run: concom requires outstanding >= 1")
    if inject_latency_us < 0:
        raise ConfigError(-1, "run: injected latency must be >= 0")
    sink = api.TraceSink()
    transport = api.Transport.local(workers, watchdog_ms, sink)
    transport.set_inject_latency(inject_latency_us)
    comms = api.create_communicators(transport, outstanding) if mode == "concom" else []
    walls = [[] for _ in range(workers)]
    sums = [0.0] * workers
    classes: list[list[str]] = [[] for _ in range(workers)]
    messages: list[str] = []

    def worker(r):
        eng = model = None
        try:
            eng = api.Engine(engine_threads, r, sink, device)
            model = api.SynthModel(eng, transport, r, workers, list(sizes), mode=mode,
                                   bucket_bytes=bucket_bytes, outstanding=outstanding if mode == "concom" else 1,
                                   lr=lr, rescale=1.0 / global_batch, momentum=momentum,
                                   backward_ns=int(backward_ms * 1e6), concom_comms=comms)
            model.init()
            for _ in range(epochs):
                t0 = time.perf_counter()
                model.run(steps_per_epoch, api.SynthModel.BACKWARD | api.SynthModel.COMM)
                walls[r].append(time.perf_counter() - t0)
            sums[r] = model.checksum()
        except CsError as e:
            classes[r].append(e.kind)
            messages.append(f"rank {r}: {e}")
            transport.abort()  # fail_slot analogue: release the other ranks (collective.cpp:92-105)
        finally:
            try:
                if eng is not None:
                    eng.wait_all()
            except CsError as e:
                if e.kind not in classes[r]:
                    classes[r].append(e.kind)
            if model is not None:
                model.close()
            if eng is not None:
                eng.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(workers)]
    for t in th:
        t.start()
    for t in th:
        t.join()

    m = Metrics(mode=mode, model=model_name, workers=workers, engine_threads=engine_threads,
                outstanding=outstanding, epochs=epochs, global_batch=global_batch, seed=seed)
    done = min(len(w) for w in walls)
    m.epoch_times_s = [sum(w[e] for w in walls) / workers for e in range(done)]
    for cl in classes:
        for c in cl:
            if c not in m.error_classes:
                m.error_classes.append(c)
    m.error = primary_error(m.error_classes)
    gauge_max, overlap = sink.gauges()
    m.max_concurrent_collectives, m.compute_overlap_observed = gauge_max, overlap
    m.b200 = {"path": "local transport rank threads, kernel (b) rank-order sums", "device": device,
              "error_messages": messages,
              "keys": len(sizes), "params": int(sum(sizes)), "steps_per_epoch": steps_per_epoch,
              "bucket_bytes": bucket_bytes, "weight_checksums": sums,
              "final_train_loss": "n/a (synthetic backward: no loss)"}
    if trace_path:
        sink.write_jsonl(trace_path)
    if metrics_path:
        write_metrics(m, metrics_path)
    transport.close()
    sink.close()
    return m
