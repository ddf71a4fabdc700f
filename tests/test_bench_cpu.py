"""bench.py's reference arm on the CPU (the driver's `--impl reference` line):
the JSON contract holds and the numbers come from the reference library
(oracle/_ref, built from /root/reference) -- no GPU needed."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "uniform16",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    if "unavailable" in line:  # oracle/_ref not built in this checkout
        return
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"] == "uniform16-funnel"


def test_reference_arm_runs_n_rank_threads_without_the_package():
    """`--impl reference --gpus 2` runs R = 2 reference rank threads, honours
    --steps / --warmup exactly, and never maps libcollsim_b200.so (the
    driver's reference_class check); its config equals the GPU arm's."""
    code = (
        "import runpy, sys, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'uniform16', '--gpus', '2',\n"
        "            '--steps', '2', '--warmup', '1']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'so_loaded': 'libcollsim_b200' in maps}))\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert lines[-1] == {"so_loaded": False}
    line = lines[0]
    if "unavailable" in line:
        return
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["warmup"] == 1
    assert line["config"]["parallelism"] == "dp2"
    sys.path.insert(0, str(ROOT))
    import bench
    keyset, mode, outstanding, dtype, bucket_mb, _ = bench.CONFIGS["uniform16"]
    keys = bench.load_keys(keyset)

    class A:
        config, issue_order, momentum, grad_views = "uniform16", "descending", 0.9, False
        direct, comm = True, None
    assert line["config"] == bench.config_dict(A, keys, mode, outstanding, dtype, bucket_mb, 2)
