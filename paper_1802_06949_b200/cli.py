"""`collsim run` / `collsim compare` drop-in over the B200 path.

    python -m paper_1802_06949_b200 run --mode depcha --workers 2 --epochs 2 \
        [--model mlp|diamond|resnet50|...] [--trace t.jsonl] [--metrics m.json]
    python -m paper_1802_06949_b200 compare a.json b.json

Mirrors R/tools/main.cpp:31-79: the same `run` flags (mode, workers,
engine-threads, outstanding, epochs, batch-size, model, seed, watchdog-ms,
inject-latency-us, lr, samples, trace, metrics), `collsim-metrics-v1` on
stdout, exit status 0 / 2 (the run failed: primary error class on stderr) /
1 (a configuration error before the run), and `compare`'s report text
(metrics.cpp:99-125).  `run` drives metrics.run_synthetic: every worker is a
rank thread with its own engine over the local transport on one GPU, and the
backward is the synthetic producer (no loss: final_train_loss reads 0).
"""
from __future__ import annotations

import argparse
import sys

from ._lib import ConfigError, CsError
from .metrics import Metrics, metrics_from_json, metrics_to_json, run_synthetic

# R/core/include/collsim/runner.hpp:26-28 (features, classes) and
# R/core/src/model.cpp:123-166 (hidden sizes, key shapes in key order)
_FEATURES, _CLASSES = 16, 4
_TOPOLOGIES = {
    "mlp": [_FEATURES * 64, 64, 64 * _CLASSES, _CLASSES],
    "diamond": [_FEATURES * 32, 32, 32 * 24, 24, 32 * 24, 24, 2 * 24 * _CLASSES, _CLASSES],
}


def model_sizes(name: str) -> list[int]:
    if name in _TOPOLOGIES:
        return list(_TOPOLOGIES[name])
    from . import keysets
    try:
        return keysets.load(name)
    except Exception:
        raise ConfigError(-1, f"unknown model: {name}") from None


def compare_report(a: Metrics, b: Metrics) -> str:
    """metrics.cpp:99-125: same shape check, same report lines."""
    if (a.model != b.model or a.epochs != b.epochs or a.global_batch != b.global_batch
            or len(a.epoch_times_s) != len(b.epoch_times_s)):
        raise ConfigError(-1, "compare: runs have different scenario shapes")
    ma = sum(a.epoch_times_s) / len(a.epoch_times_s) if a.epoch_times_s else 0.0
    mb = sum(b.epoch_times_s) / len(b.epoch_times_s) if b.epoch_times_s else 0.0
    ratio = mb / ma if ma > 0.0 else 0.0
    return (f"                          A({a.mode})  B({b.mode})\n"
            f"mean epoch time (s)       {ma:.6f}  {mb:.6f}\n"
            f"epoch time ratio B/A      {ratio:.4f}\n"
            f"max concurrent colls      {a.max_concurrent_collectives}  {b.max_concurrent_collectives}\n"
            f"compute/comm overlap      {'yes' if a.compute_overlap_observed else 'no'}  "
            f"{'yes' if b.compute_overlap_observed else 'no'}\n")


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="collsim", description="B200 gradient-aggregation path of arXiv 1802.06949")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="run a training scenario and emit metrics")
    run.add_argument("--backend", default="b200", choices=["b200"])
    run.add_argument("--mode", default="funnel", choices=["funnel", "depcha", "concom", "naive"])
    run.add_argument("--workers", type=int, default=2)
    run.add_argument("--engine-threads", type=int, default=4)
    run.add_argument("--outstanding", type=int, default=2)
    run.add_argument("--epochs", type=int, default=1)
    run.add_argument("--batch-size", type=int, default=64)
    run.add_argument("--model", default="diamond")
    run.add_argument("--seed", type=int, default=1)
    run.add_argument("--watchdog-ms", type=int, default=30000)
    run.add_argument("--inject-latency-us", type=int, default=0)
    run.add_argument("--lr", type=float, default=0.1)
    run.add_argument("--samples", type=int, default=1024)
    run.add_argument("--trace", default=None)
    run.add_argument("--metrics", default=None)
    run.add_argument("--bucket-mb", type=float, default=0.0, help="B200: fusion bucket size (0 = 1:1 comm_buf)")
    run.add_argument("--backward-ms", type=float, default=1.0, help="B200: synthetic backward per step")
    cmp = sub.add_parser("compare", help="compare two metrics files")
    cmp.add_argument("a")
    cmp.add_argument("b")
    return ap


def main(argv=None) -> int:
    a = _parser().parse_args(argv)
    try:
        if a.cmd == "compare":
            with open(a.a) as fa, open(a.b) as fb:
                print(compare_report(metrics_from_json(fa.read()), metrics_from_json(fb.read())), end="")
            return 0
        if a.lr <= 0.0:
            raise ConfigError(-1, "run: learning rate must be positive")
        if a.watchdog_ms <= 0:
            raise ConfigError(-1, "run: watchdog must be positive")
        m = run_synthetic(mode=a.mode, workers=a.workers, engine_threads=a.engine_threads,
                          outstanding=a.outstanding, epochs=a.epochs,
                          steps_per_epoch=max(1, a.samples // max(1, a.batch_size)), sizes=model_sizes(a.model),
                          bucket_bytes=int(a.bucket_mb * 2**20), seed=a.seed, global_batch=a.batch_size,
                          backward_ms=a.backward_ms, watchdog_ms=a.watchdog_ms, model_name=a.model,
                          trace_path=a.trace, metrics_path=a.metrics, inject_latency_us=a.inject_latency_us,
                          lr=a.lr)
        print(metrics_to_json(m))
        if not m.ok():
            print(f"error: {m.error}", file=sys.stderr)
            return 2
        return 0
    except CsError as e:
        print(f"error: {e.kind}: {e}", file=sys.stderr)
        return 1
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
