"""The collsim CLI drop-in (R/tools/main.cpp): compare's report and shape
check, and the exit status of a configuration error -- CPU only (the run
itself is exercised on the GPU in test_cli_gpu)."""
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1802_06949_b200 import ConfigError
from paper_1802_06949_b200.cli import compare_report, model_sizes
from paper_1802_06949_b200.metrics import Metrics, write_metrics

ROOT = Path(__file__).resolve().parent.parent


def _m(mode, times, conc, ov):
    return Metrics(mode=mode, model="diamond", workers=2, engine_threads=4, outstanding=2, epochs=len(times),
                   global_batch=64, seed=1, epoch_times_s=times, max_concurrent_collectives=conc,
                   compute_overlap_observed=ov)


def test_compare_report_matches_reference_layout():
    text = compare_report(_m("funnel", [0.5, 0.25], 1, False), _m("depcha", [0.25, 0.125], 1, True))
    assert text.splitlines() == [
        "                          A(funnel)  B(depcha)",
        "mean epoch time (s)       0.375000  0.187500",
        "epoch time ratio B/A      0.5000",
        "max concurrent colls      1  1",
        "compute/comm overlap      no  yes",
    ]
    with pytest.raises(ConfigError, match="different scenario shapes"):
        compare_report(_m("funnel", [0.5], 1, False), _m("depcha", [0.25, 0.1], 1, True))


def test_cli_compare_and_config_error_exit_codes(tmp_path):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    write_metrics(_m("funnel", [0.5], 1, False), a)
    write_metrics(_m("concom", [0.25], 2, True), b)
    r = subprocess.run([sys.executable, "-m", "paper_1802_06949_b200", "compare", str(a), str(b)],
                       capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "epoch time ratio B/A      0.5000" in r.stdout
    r = subprocess.run([sys.executable, "-m", "paper_1802_06949_b200", "run", "--mode", "concom", "--outstanding",
                        "0"], capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert r.returncode == 1 and "ConfigError" in r.stderr


def test_model_key_sizes_follow_the_reference_topologies():
    assert model_sizes("mlp") == [16 * 64, 64, 64 * 4, 4]          # model.cpp:153-157
    assert len(model_sizes("diamond")) == 8                        # model.cpp:159-166
    assert len(model_sizes("resnet50")) == 161
    with pytest.raises(ConfigError):
        model_sizes("nope")
