"""Checks of the peer-memory / multi-rank cases of tests/mp_worker.py, shared
by the one-process-per-GPU tests (test_nccl_multigpu.py, torchrun over NCCL)
and the one-GPU colocated tests (test_peer_local_gpu.py, rank threads over a
local peer transport).  Each takes the case's output directory, the world
size R and the per-rank JSON records.

Pins: reference golden weights (tests/golden/train_steps.npz, produced by
the unmodified reference KvStore, test_kvstore.cpp:290-330 seeds, loop shape
trainer.cpp:112-141), the rank-order sum collective.cpp:228-236 and the
sgd_update arithmetic model.cpp:17-27 through the C oracle.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

import _oracle as O

HERE = Path(__file__).resolve().parent


def golden():
    return np.load(HERE / "golden" / "train_steps.npz")


def check_schedule_weights(d: Path, case: str, mode: str, R: int, outs, exact: bool = True):
    """Every rank's weights after 3 push/pull/sgd iterations equal the
    reference KvStore's (bit-exact for rank-order sums; 1e-12 for NCCL's own
    reduction order at R > 2), and every rank issued identical per-comm
    collective sequences."""
    gold = golden()
    K = len(gold["sizes"])
    for r in range(R):
        w = np.load(d / f"{case}_r{r}.npz")
        for k in range(K):
            exp = gold[f"{mode}_R{R}_r{r}_k{k}"]
            if exact:
                np.testing.assert_array_equal(w[f"arr_{k}"], exp, err_msg=f"{case} R={R} rank {r} key {k}")
            else:
                np.testing.assert_allclose(w[f"arr_{k}"], exp, rtol=0, atol=1e-12)
    for r in range(1, R):
        for comm in {s.split(":")[1] for s in outs[0]["trace"]}:
            assert [s for s in outs[r]["trace"] if s.split(":")[1] == comm] == \
                [s for s in outs[0]["trace"] if s.split(":")[1] == comm]


def check_p2p_api(d: Path, R: int, n: int = 4 << 20):
    """cs_allreduce_p2p on a 16 MiB fp32 bucket: the reduce-only sum is the
    fp32 rank-order sum bit for bit; the fused update gives identical weights
    and momentum with shard_only 0 and 1; shard_only 0 leaves the whole sum in
    the bucket, shard_only 1 exactly the own shard; weights and momentum match
    the f32 oracle update bit for bit."""
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


def check_torch_dp(d: Path, case: str, R: int):
    """PyTorch autograd as the producer: every rank's weights after each step
    are the f32 oracle update with the rank-order sum of the ranks' gradients."""
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


def check_stress_order(R: int, outs):
    """Every schedule finished with per-rank random completion orders, every
    rank holds the same weights, and they equal the in-order run's."""
    sums = [o["sums"] for o in outs]
    for name in sums[0]:
        for r in range(R):
            assert sums[r][name] == sums[0][name], (R, name)
        if name.endswith("_s11"):
            assert sums[0][name] == sums[0][name[:-3] + "s0"], (R, name)


def check_zero_vs_replicated(d: Path, R: int):
    """ZeRO-1 weights == replicated fused update weights, fp32 and bf16
    buckets, momentum 0.9, 3 steps; identical on every rank."""
    outs = [np.load(d / f"zero_vs_replicated_r{r}.npz") for r in range(R)]
    for r in range(R):
        for name in outs[r].files:
            if name.startswith("z1_"):
                np.testing.assert_array_equal(outs[r][name], outs[r]["z0_" + name[3:]], err_msg=f"R={R} {name}")
            np.testing.assert_array_equal(outs[r][name], outs[0][name])


def check_zero_vs_oracle(d: Path, R: int):
    """...and the fp32-bucket run equals the f32 oracle: rank-order sum of
    the ranks' fp32 gradients, then the momentum update, 3 steps."""
    sizes = [1, 7, 64, 300, 4097, 70000, 1 << 18]
    K = len(sizes)
    o = np.load(d / "zero_vs_replicated_r0.npz")
    for k, n in enumerate(sizes):
        w = O.random_uniform(n, O.mix_seed(7, k)).astype(np.float32)
        g = O.rank_order_sum([O.random_uniform(n, 1000 + r * K + k).astype(np.float32) for r in range(R)], "f32")
        m = np.zeros(n, np.float32)
        for _ in range(3):
            w, m = O.sgd_update(w, g, 0.1, 1.0 / 64, 0.9, m, kind="f32")
        np.testing.assert_array_equal(o[f"z1_c1_k{k}"], w, err_msg=f"R={R} key {k}")


def check_direct(d: Path, R: int):
    """Direct gradient reads (registered region, nothing staged) give the
    staged run's weights bit for bit -- DepCha's fused ZeRO-1 and replicated
    kernels and Funnel's plain allreduce, fp32 and bf16 gradients -- on every
    rank, and the fp32 ZeRO-1 run equals the f32 oracle."""
    outs = [np.load(d / f"direct_r{r}.npz") for r in range(R)]
    for r in range(R):
        names = [n for n in outs[r].files if "_d1_" in n]
        assert len(names) == 6 * 7, names  # DepCha: ZeRO-1 / replicated x fp32 / bf16; Funnel: fp32 / bf16
        for name in names:
            np.testing.assert_array_equal(outs[r][name], outs[r][name.replace("_d1_", "_d0_")],
                                          err_msg=f"R={R} rank {r} {name}")
            np.testing.assert_array_equal(outs[r][name], outs[0][name])
    sizes = [1, 7, 64, 300, 4097, 70000, 1 << 18]
    K = len(sizes)
    for k, n in enumerate(sizes):
        w = O.random_uniform(n, O.mix_seed(7, k)).astype(np.float32)
        g = O.rank_order_sum([O.random_uniform(n, 1000 + r * K + k).astype(np.float32) for r in range(R)], "f32")
        m = np.zeros(n, np.float32)
        for _ in range(3):
            w, m = O.sgd_update(w, g, 0.1, 1.0 / 64, 0.9, m, kind="f32")
        np.testing.assert_array_equal(outs[0][f"z1_g1_d1_k{k}"], w, err_msg=f"R={R} key {k}")


def check_direct_mismatch(outs, R: int):
    """Rank-dependent gradient layouts are caught by the ledger (layout hash
    in the call signature) before any peer kernel reads a wrong address."""
    for r in range(R):
        assert outs[r]["error"] and outs[r]["error"].startswith("MismatchError"), outs[r]
        assert "direct" in outs[r]["error"], outs[r]["error"]
