"""One process per GPU over NCCL (NVLink): parity of the allreduce and of the
three schedules against the oracle / golden fixtures, and the cross-process
matching ledger turning a misordered or missing call into MismatchError /
DeadlockTimeout before anything is enqueued on NVLink.
Needs >= 2 GPUs (gpurun --gpus 2); skipped otherwise."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import _oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = Path(__file__).resolve().parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_case(case, n, tmp_path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(HERE / "mp_worker.py"), case,
           str(tmp_path)]
    for _ in range(3):  # a freshly picked port can be taken before torchrun binds it
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=240,
                           env={**os.environ, "OMP_NUM_THREADS": "1"})
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr:
            break
        cmd[5] = f"--master-port={_free_port()}"
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [json.loads((tmp_path / f"{case}_r{i}.json").read_text()) for i in range(n)]


def world_sizes(ngpus):
    return [w for w in (2, 4) if w <= ngpus]


def test_nccl_allreduce_acceptance_1(two_gpus, tmp_path):
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("allreduce", R, d)
        outs = [np.load(d / f"allreduce_r{r}.npz") for r in range(R)]
        for i in range(100):
            n = 1 + (i * 7) % 64
            exp = O.rank_order_sum([O.random_uniform(n, O.mix_seed(R * 1000 + i, r)) for r in range(R)])
            for r in range(R):
                got = outs[r][f"arr_{i}"]
                if R == 2:
                    np.testing.assert_array_equal(got, exp)  # a + b: order-free, exact
                else:
                    assert np.max(np.abs(got - exp)) <= 1e-12  # reference tolerance
            for r in range(1, R):  # every rank holds the same result
                np.testing.assert_array_equal(outs[r][f"arr_{i}"], outs[0][f"arr_{i}"])


@pytest.mark.parametrize("mode", ["funnel", "depcha", "concom"])
def test_nccl_schedules_match_reference(two_gpus, tmp_path, mode):
    gold = np.load(HERE / "golden" / "train_steps.npz")
    K = len(gold["sizes"])
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        outs = run_case(mode, R, d)
        for r in range(R):
            w = np.load(d / f"{mode}_r{r}.npz")
            for k in range(K):
                exp = gold[f"{mode}_R{R}_r{r}_k{k}"]
                if R == 2:
                    np.testing.assert_array_equal(w[f"arr_{k}"], exp)
                else:
                    np.testing.assert_allclose(w[f"arr_{k}"], exp, rtol=0, atol=1e-12)
        # identical per-comm issue sequences on every rank
        for r in range(1, R):
            for comm in {s.split(":")[1] for s in outs[0]["trace"]}:
                assert [s for s in outs[r]["trace"] if s.split(":")[1] == comm] == \
                    [s for s in outs[0]["trace"] if s.split(":")[1] == comm]


@pytest.mark.parametrize("mode,variant", [("depcha", "p2p"), ("funnel", "p2p"), ("depcha", "p2pzero")])
def test_p2p_fused_allreduce_update_bit_exact(two_gpus, tmp_path, mode, variant):
    """DepCha / Funnel over the NVLink peer-memory path: one fused
    allreduce+SGD kernel per bucket (16 KiB fusion buckets).  Rank-order sums
    make the result bit-identical to the reference KvStore at every world
    size.  p2pzero: ZeRO-1 (each rank updates master weights of its shard
    only, then the kernel all-gathers the weights) -- still bit-identical."""
    gold = np.load(HERE / "golden" / "train_steps.npz")
    K = len(gold["sizes"])
    case = f"{mode}_{variant}"
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        outs = run_case(case, R, d)
        for r in range(R):
            w = np.load(d / f"{case}_r{r}.npz")
            for k in range(K):
                np.testing.assert_array_equal(w[f"arr_{k}"], gold[f"{mode}_R{R}_r{r}_k{k}"])
        for r in range(1, R):
            assert outs[r]["trace"] == outs[0]["trace"]


def test_p2p_split_pulls_bit_exact(two_gpus, tmp_path):
    """Same, but one pull_update per key: the first pull of a bucket fuses only
    its own key's update, so the kernel keeps the whole sum in every bucket
    (shard_only off) and the later pulls read it."""
    gold = np.load(HERE / "golden" / "train_steps.npz")
    K = len(gold["sizes"])
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("depcha_p2psplit", R, d)
        for r in range(R):
            w = np.load(d / f"depcha_p2psplit_r{r}.npz")
            for k in range(K):
                np.testing.assert_array_equal(w[f"arr_{k}"], gold[f"depcha_R{R}_r{r}_k{k}"])


def test_p2p_c_abi_reduce_and_shard_only(two_gpus, tmp_path):
    """cs_allreduce_p2p on a 16 MiB fp32 bucket: the reduce-only sum is the
    fp32 rank-order sum bit for bit; the fused update gives identical weights
    and momentum with shard_only 0 and 1; shard_only 0 leaves the whole sum in
    the bucket, shard_only 1 exactly the own shard; weights and momentum match
    the f32 oracle update bit for bit."""
    n = 4 << 20
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("p2p_api", R, d)
        gs = [O.random_uniform(n, 1000 + r).astype(np.float32) for r in range(R)]
        exp = gs[0].copy()
        for x in gs[1:]:
            exp = exp + x  # float32 IEEE round-to-nearest, rank order
        w0 = O.random_uniform(n, O.mix_seed(7, 0)).astype(np.float32)
        w_exp, m_exp = O.sgd_update(w0, exp, 0.1, 1.0 / 64, 0.9, np.zeros(n, np.float32), kind="f32")
        groups = n // 8
        outs = [np.load(d / f"p2p_api_r{r}.npz") for r in range(R)]
        for r, o in enumerate(outs):
            np.testing.assert_array_equal(o["sum"], exp)
            np.testing.assert_array_equal(o["buf0"], exp)
            np.testing.assert_array_equal(o["w0"], o["w1"])
            np.testing.assert_array_equal(o["m0"], o["m1"])
            a, b = 8 * (groups * r // R), 8 * (groups * (r + 1) // R)
            np.testing.assert_array_equal(o["buf1"][a:b], exp[a:b])
            np.testing.assert_array_equal(o["m0"], m_exp)
            np.testing.assert_array_equal(o["w0"], w_exp)
            np.testing.assert_array_equal(o["w0"], outs[0]["w0"])


@pytest.mark.parametrize("case", ["torch_dp", "torch_dp_zero"])
def test_torch_producer_over_nvlink_bit_exact(two_gpus, tmp_path, case):
    """PyTorch autograd as the producer (torch_dp.TorchKvStoreDP, 2-3 fusion
    buckets, fused NVLink kernel; torch_dp_zero: ZeRO-1 sharded momentum and
    master weights): every rank's weights after each step are the f32 oracle
    update with the rank-order sum of the ranks' gradients."""
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case(case, R, d)
        outs = [np.load(d / f"{case}_r{r}.npz") for r in range(R)]
        assert int(outs[0]["buckets"]) >= 2
        w = outs[0]["w0"].astype(np.float32)
        mom = np.zeros_like(w)
        for r in range(R):
            np.testing.assert_array_equal(outs[r]["w0"], w)  # rank 0's weights were broadcast
        for step in range(3):
            g = outs[0][f"g{step}"].astype(np.float32)
            for r in range(1, R):
                g = g + outs[r][f"g{step}"].astype(np.float32)  # rank order, f32 round-to-nearest
            w, mom = O.sgd_update(w, g, 0.05, 1.0 / R, 0.9, mom, kind="f32")
            for r in range(R):
                np.testing.assert_array_equal(outs[r][f"w{step + 1}"], w, err_msg=f"R={R} rank {r} step {step}")


def test_stress_random_completion_order_is_deadlock_free_and_order_independent(two_gpus, tmp_path):
    """96 stress keys (1 KiB-256 KiB), every rank's synthetic backward in its
    own random order: DepCha (fused kernel, replicated and ZeRO-1), Funnel
    (fused kernel) and DepCha over NCCL all finish (no deadlock, no mismatch)
    and every rank ends with the same weights as the in-order run."""
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        outs = run_case("stress_order", R, d)
        sums = [o["sums"] for o in outs]
        for name in sums[0]:
            for r in range(R):
                assert sums[r][name] == sums[0][name], (R, name)
            if name.endswith("_s11"):
                assert sums[0][name] == sums[0][name[:-3] + "s0"], (R, name)


def test_zero_equals_replicated_update_fp32_and_bf16(two_gpus, tmp_path):
    """ZeRO-1 (sharded master weights + momentum, weight all-gather) gives
    bit-identical weights to the replicated fused update, with fp32 and with
    bf16 comm buckets (the kernel reproduces the bucket's bf16 rounding of
    the sum), momentum 0.9, 3 steps, keys straddling shard boundaries."""
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("zero_vs_replicated", R, d)
        outs = [np.load(d / f"zero_vs_replicated_r{r}.npz") for r in range(R)]
        for r in range(R):
            for name in outs[r].files:
                if name.startswith("z1_"):
                    np.testing.assert_array_equal(outs[r][name], outs[r]["z0_" + name[3:]], err_msg=f"R={R} {name}")
                np.testing.assert_array_equal(outs[r][name], outs[0][name])


def test_nvls_fused_allreduce_update_within_tolerance(two_gpus, tmp_path):
    """fp32 DepCha through the NVSwitch multicast path (multimem.ld_reduce /
    multimem.st) fused with the momentum update: within the north-star fp32
    tolerance of the fp64 oracle, and identical on every rank."""
    sizes = [1, 7, 64, 300, 4097, 70000]
    K = len(sizes)
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("nvls", R, d)
        ws = [np.load(d / f"nvls_r{r}.npz") for r in range(R)]
        for k, n in enumerate(sizes):
            g = [O.random_uniform(n, 1000 + r * K + k).astype(np.float32).astype(np.float64) for r in range(R)]
            s = O.rank_order_sum(g, "f64")
            w0 = O.random_uniform(n, O.mix_seed(7, k)).astype(np.float32).astype(np.float64)
            exp, _ = O.sgd_update(w0, s, 0.1, 1.0 / 64, 0.9, np.zeros(n))
            scale = np.abs(w0) + 0.1 / 64 * np.sum([np.abs(x) for x in g], axis=0)
            for r in range(R):
                got = ws[r][f"arr_{k}"].astype(np.float64)
                assert np.all(np.abs(got - exp) <= 1e-6 * scale + 1e-7), (R, k)
                np.testing.assert_array_equal(ws[r][f"arr_{k}"], ws[0][f"arr_{k}"])


def test_cross_process_mismatch_raises_before_nccl(two_gpus, tmp_path):
    outs = run_case("mismatch", 2, tmp_path)
    assert [o["error"] for o in outs] == ["MismatchError", "MismatchError"]
    assert "allreduce(count=4)" in outs[0]["message"] and "allreduce(count=6)" in outs[0]["message"]


def test_cross_process_deadlock_report(two_gpus, tmp_path):
    outs = run_case("deadlock", 2, tmp_path)
    assert outs[0]["error"] == "DeadlockTimeout"
    assert "rank 1: no call issued" in outs[0]["message"]
