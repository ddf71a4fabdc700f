"""One process per GPU over NCCL (NVLink): parity of the allreduce and of the
three schedules against the oracle / golden fixtures, and the cross-process
matching ledger turning a misordered or missing call into MismatchError /
DeadlockTimeout before anything is enqueued on NVLink.
Needs >= 2 GPUs (gpurun --gpus 2); skipped otherwise.  The same peer-memory
cases run on ONE GPU (rank threads, colocated grids) in test_peer_local_gpu.py."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import _oracle as O
from peer_cases import (check_direct, check_direct_mismatch, check_p2p_api, check_schedule_weights,
                        check_stress_order, check_torch_dp, check_zero_vs_oracle, check_zero_vs_replicated)

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
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        outs = run_case(mode, R, d)
        check_schedule_weights(d, mode, mode, R, outs, exact=(R == 2))


@pytest.mark.parametrize("mode,variant", [("depcha", "p2p"), ("funnel", "p2p"), ("depcha", "p2pzero"),
                                          ("concom", "p2p")])
def test_p2p_fused_allreduce_update_bit_exact(two_gpus, tmp_path, mode, variant):
    """DepCha / Funnel over the NVLink peer-memory path: one fused
    allreduce+SGD kernel per bucket (16 KiB fusion buckets).  Rank-order sums
    make the result bit-identical to the reference KvStore at every world
    size.  p2pzero: ZeRO-1 (each rank updates master weights of its shard
    only, then the kernel all-gathers the weights) -- still bit-identical.
    concom: two communicators' peer kernels running concurrently, each grid
    capped to half the device so both are always co-resident."""
    case = f"{mode}_{variant}"
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        outs = run_case(case, R, d)
        check_schedule_weights(d, case, mode, R, outs)


def test_p2p_split_pulls_bit_exact(two_gpus, tmp_path):
    """Same, but one pull_update per key: the first pull of a bucket fuses only
    its own key's update, so the kernel keeps the whole sum in every bucket
    (shard_only off) and the later pulls read it."""
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        outs = run_case("depcha_p2psplit", R, d)
        check_schedule_weights(d, "depcha_p2psplit", "depcha", R, outs)


def test_p2p_c_abi_reduce_and_shard_only(two_gpus, tmp_path):
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("p2p_api", R, d)
        check_p2p_api(d, R)


@pytest.mark.parametrize("case", ["torch_dp", "torch_dp_zero"])
def test_torch_producer_over_nvlink_bit_exact(two_gpus, tmp_path, case):
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case(case, R, d)
        check_torch_dp(d, case, R)


def test_stress_random_completion_order_is_deadlock_free_and_order_independent(two_gpus, tmp_path):
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        check_stress_order(R, run_case("stress_order", R, d))


def test_zero_equals_replicated_update_fp32_and_bf16(two_gpus, tmp_path):
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("zero_vs_replicated", R, d)
        check_zero_vs_replicated(d, R)
        check_zero_vs_oracle(d, R)


def test_direct_gradient_reads_over_ipc_equal_staged(two_gpus, tmp_path):
    """register_grads over CUDA IPC (an interior pointer of a torch
    allocation: the handle names the allocation, the offset travels with
    it): in-place peer reads of every rank's gradients == the staged run."""
    for R in world_sizes(two_gpus):
        d = tmp_path / f"R{R}"
        d.mkdir()
        run_case("direct", R, d)
        check_direct(d, R)
    check_direct_mismatch(run_case("direct_mismatch", 2, tmp_path), 2)


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
