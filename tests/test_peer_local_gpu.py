"""The cross-GPU peer-memory path on ONE GPU: R rank threads on cuda:0 over a
local peer transport (Transport.local(R, peer=True)).  Every rank runs the
same fused kernels as across GPUs -- p2p_allreduce_kernel (whole-bucket and
split pulls, shard_only 0/1), p2p_zero_kernel (ZeRO-1) -- with the same pair
barriers, epochs and M = 2 / 4 / 8 instantiations; only the peer addresses
are plain device pointers and each grid is capped to 1/R of the device so
all R grids are co-resident.  This is what the driver's 1-GPU box runs, so
the cross-GPU kernels are checked there, not only on multi-GPU boxes.

Pins: the unmodified reference KvStore's final weights at R = 2, 4, 8
(tests/golden/train_steps.npz; test_kvstore.cpp:290-330 seeds, trainer.cpp
:112-141 loop shape), collective.cpp:228-236 rank-order sums and model.cpp
:17-27 through the C oracle.  Bit-exact everywhere (rank-order sums)."""
import threading
import time

import numpy as np
import pytest
import torch

from mp_worker import run_colocated
from peer_cases import (check_direct, check_direct_mismatch, check_p2p_api, check_schedule_weights,
                        check_stress_order, check_torch_dp, check_zero_vs_oracle, check_zero_vs_replicated)

pytestmark = pytest.mark.gpu
RANKS = [2, 4, 8]


@pytest.mark.parametrize("R", RANKS)
@pytest.mark.parametrize("mode,variant", [("depcha", "p2p"), ("funnel", "p2p"), ("depcha", "p2pzero"),
                                          ("depcha", "p2psplit"), ("concom", "p2p")])
def test_colocated_fused_kernel_matches_reference_weights(gpu, tmp_path, R, mode, variant):
    case = f"{mode}_{variant}"
    outs = run_colocated(case, R, tmp_path)
    check_schedule_weights(tmp_path, case, mode, R, outs)


@pytest.mark.parametrize("R", RANKS)
@pytest.mark.parametrize("mode", ["funnel", "depcha", "concom"])
def test_colocated_three_schedules_match_reference_weights(gpu, tmp_path, R, mode):
    """The paper's three schedules with R rank threads (R = 8: the north
    star's 8-rank case) over the in-process transport -- kernel (b)'s
    rank-order sum as the collective, ConCom on 2 extra communicators --
    deadlock-free, every rank's weights equal to the unmodified reference
    KvStore's (golden, trainer.cpp:112-141 loop), identical per-comm issue
    sequences on every rank."""
    outs = run_colocated(mode, R, tmp_path)
    check_schedule_weights(tmp_path, mode, mode, R, outs)


@pytest.mark.parametrize("R", RANKS)
def test_colocated_c_abi_reduce_and_shard_only(gpu, tmp_path, R):
    run_colocated("p2p_api", R, tmp_path)
    check_p2p_api(tmp_path, R)


@pytest.mark.parametrize("R", RANKS)
def test_colocated_zero_equals_replicated_and_oracle(gpu, tmp_path, R):
    run_colocated("zero_vs_replicated", R, tmp_path)
    check_zero_vs_replicated(tmp_path, R)
    check_zero_vs_oracle(tmp_path, R)


@pytest.mark.parametrize("R", RANKS)
def test_colocated_direct_gradient_reads_equal_staged(gpu, tmp_path, R):
    run_colocated("direct", R, tmp_path)
    check_direct(tmp_path, R)


def test_colocated_direct_layout_mismatch_raises(gpu, tmp_path):
    check_direct_mismatch(run_colocated("direct_mismatch", 2, tmp_path, watchdog_ms=5000), 2)


@pytest.mark.parametrize("R", [2, 4, 8])
def test_colocated_stress_random_completion_order(gpu, tmp_path, R):
    check_stress_order(R, run_colocated("stress_order", R, tmp_path))


@pytest.mark.parametrize("case", ["torch_dp", "torch_dp_zero"])
def test_colocated_torch_producer_bit_exact(gpu, tmp_path, case):
    run_colocated(case, 2, tmp_path)
    check_torch_dp(tmp_path, case, 2)


def test_mismatched_barrier_protocol_raises_before_launch(gpu):
    """ranks choosing different fused-kernel variants (shard_only
    on one rank, a plain reduce on the other) would wait at barriers their
    peers never reach.  The ledger signature carries the variant, so both
    ranks get MismatchError before anything is launched."""
    from paper_1802_06949_b200 import Engine, MismatchError, Transport, api
    R, n = 2, 1 << 12
    tr = Transport.local(R, 3000, None, peer=True)
    errs = [None] * R

    def body(r):
        eng = Engine(1, r, None, 0)
        buf = torch.zeros(n, dtype=torch.float32, device="cuda")
        w = torch.zeros(n, dtype=torch.float32, device="cuda")
        peers = tr.share_buffer(buf.data_ptr(), r)
        upd = ([(w.data_ptr(), buf.data_ptr(), 0, n)], api.F32, 0.1, 1.0, 0.0, 1) if r == 0 else None
        try:
            tr.allreduce_p2p(0, r, peers, n, api.F32, 0, upd, eng.lane_stream(0))
        except MismatchError as e:
            errs[r] = str(e)
        eng.wait_all()
        eng.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    tr.close()
    assert all(e is not None for e in errs), errs
    assert "p2p+update+shard_only" in errs[0] and "allreduce(count=4096, p2p)" in errs[0]


def test_missing_peer_kernel_times_out_without_a_gpu_fault(gpu):
    """collective.cpp:249-264 (watchdog -> DeadlockTimeout -> latch) for a
    device-side hang: rank 1 passes the matching ledger but its kernel is
    held behind a 5 s device-side spin on its stream, so rank 0's pair
    barrier waits far past rank 0's 1.5 s engine watchdog.  The engine watchdog
    sets the transport's abort word; the kernel leaves its barrier and
    returns (no __trap), wait_all raises DeadlockTimeout, the transport is
    latched, and the GPU keeps working afterwards."""
    from paper_1802_06949_b200 import DeadlockTimeout, Engine, Transport, api
    R, n = 2, 1 << 16
    tr = Transport.local(R, 20000, None, peer=True)
    e0, e1 = Engine(1, 0, None, 0), Engine(1, 1, None, 0)
    e0.set_watchdog(1500)
    bufs = [torch.ones(n, dtype=torch.float32, device="cuda") for _ in range(R)]
    peers = [None, None]

    def share(r):
        peers[r] = tr.share_buffer(bufs[r].data_ptr(), r)

    th = [threading.Thread(target=share, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    # rank 1's lane is blocked by a long device-side spin (its kernel stays
    # queued behind it for much longer than rank 0's watchdog)
    s1 = e1.lane_stream(0)
    api.synth_backward(0, 0, 0, api.F32, int(5e9), 1, s1)
    errs = {}

    def call(r, eng, stream):
        try:
            tr.allreduce_p2p(0, r, peers[r], n, api.F32, 0, None, stream)
        except DeadlockTimeout as e:
            errs[r] = str(e)

    # a colocated rank returns from the call once its kernel completed
    th = [threading.Thread(target=call, args=(1, e1, s1)),
          threading.Thread(target=call, args=(0, e0, e0.lane_stream(0)))]
    for t in th:
        t.start()
    time.sleep(0.5)
    t0 = time.time()
    with pytest.raises(DeadlockTimeout):
        e0.wait_all()  # rank 0's lane holds the waiting kernel: the watchdog aborts it
    assert time.time() - t0 < 10
    th[1].join(timeout=10)
    assert not th[1].is_alive() and 0 in errs  # rank 0's kernel left its barrier
    th[0].join(timeout=30)  # rank 1's kernel runs after the spin and sees the abort word
    assert not th[0].is_alive()
    torch.cuda.synchronize()
    with pytest.raises(DeadlockTimeout):  # latched
        tr.allreduce_p2p(0, 0, peers[0], n, api.F32, 0, None, e0.lane_stream(0))
    x = torch.arange(1000, device="cuda", dtype=torch.float32)
    assert float(x.sum()) == 499500.0  # the context is healthy
    e0.close()
    e1.close()
    tr.close()
