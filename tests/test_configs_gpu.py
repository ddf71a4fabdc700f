"""BASELINE.json configs C2-C5 at full key-set size on ONE GPU, parity against
the oracle (or_synth_expect, pinned to the reference's golden weights):

  C2 ResNet-50 (161 keys, 25.6 M fp32)      DepCha, 100 MiB bucket, fused peer kernel (ZeRO-1)
  C3 AlexNet (16 keys, 61.1 M fp32)          ConCom, 4 communicators, 25 MiB buckets
  C4 ResNet-152 (467 keys, 60.2 M bf16)      DepCha / Funnel / ConCom, 128 MiB / 25 MiB buckets
     Inception-v3 (292 keys, 27.2 M bf16)    DepCha, fused peer kernel
  C5 deadlock stress (2048 keys, 1 KiB-64 MiB log-uniform; each key capped at
     64 Ki elements so one GPU holds every rank) with per-rank random
     completion order, DepCha over the fused peer kernel

Each runs R rank threads on cuda:0 (a local transport; `peer` = the fused
peer-memory kernels colocated, else the last arriver's rank-order sum), the
config's real loop shape (trainer.cpp:112-141 via the synthetic model), 3
steps with the synthetic backward, momentum 0.9 (fp32) as in the bench.
Weights of every rank are read back: rank 0 against the oracle, every other
rank bit-identical to rank 0.  Bars (north star): fp32 bit-exact against the
fp32 restatement and <= 1e-6 relative to fp64; bf16 sums bit-exact against
the bf16 restatement and <= 1e-2 relative to fp64."""
import threading

import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu


def run_config(keys, R, *, mode, dtype, bucket_mb, peer, outstanding=1, zero=False, order_seed=0, momentum=0.9):
    from paper_1802_06949_b200 import Engine, Transport, api, create_communicators
    D = {"fp32": api.F32, "bf16": api.BF16}
    tr = Transport.local(R, 120000, None, peer=peer)
    comms = create_communicators(tr, outstanding) if mode == "concom" else []
    out, errs = [None] * R, []

    def rank(r):
        try:
            eng = Engine(4, r, None, 0)
            m = api.SynthModel(eng, tr, r, R, keys, mode=mode, w_dtype=api.F32, g_dtype=D[dtype],
                               comm_dtype=D[dtype], bucket_bytes=int(bucket_mb * 2**20), issue_order=1,
                               outstanding=outstanding, lr=0.1, rescale=1.0 / (64 * R), momentum=momentum,
                               p2p=1 if peer else 0, zero=zero, order_seed=order_seed,
                               direct_grads=mode != "concom",  # the bench default: registered gradients
                               concom_comms=comms)
            m.init()
            m.run(3, m.BACKWARD | m.COMM)
            out[r] = m.read_weights()
            m.close()
            eng.close()
        except BaseException as e:
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    tr.close()
    if errs:
        raise errs[0]
    exp, r64, sc = O.synth_expect(keys, R, 3, wdt="f32", gdt={"fp32": "f32", "bf16": "bf16"}[dtype], lr=0.1,
                                  rescale=1.0 / (64 * R),
                                  momentum=momentum)
    np.testing.assert_array_equal(out[0], exp)
    err = float(np.max(np.abs(out[0].astype(np.float64) - r64) / sc))
    assert err <= (1e-2 if dtype == "bf16" else 1e-6), err
    for r in range(1, R):
        np.testing.assert_array_equal(out[r], out[0])
    return err


def keys_of(name):
    from paper_1802_06949_b200 import keysets
    return keysets.load(name)


def test_c2_resnet50_depcha_zero_fused_kernel(gpu):
    run_config(keys_of("resnet50"), 2, mode="depcha", dtype="fp32", bucket_mb=100, peer=True, zero=True)


@pytest.mark.parametrize("peer", [False, True])
def test_c3_alexnet_concom_4_communicators(gpu, peer):
    """ConCom x 4 over the in-process transport (kernel (b)) and over the
    peer-memory kernel (four communicators' grids concurrently, each capped
    to a quarter of the device's share)."""
    run_config(keys_of("alexnet"), 2, mode="concom", dtype="fp32", bucket_mb=25, peer=peer, outstanding=4)


@pytest.mark.parametrize("mode,bucket_mb,peer", [("depcha", 128, True), ("funnel", 128, True),
                                                 ("concom", 25, True)])
def test_c4_resnet152_bf16_all_schedules(gpu, mode, bucket_mb, peer):
    run_config(keys_of("resnet152"), 2, mode=mode, dtype="bf16", bucket_mb=bucket_mb, peer=peer,
               outstanding=4 if mode == "concom" else 1)


def test_c4_inception_v3_bf16_depcha(gpu):
    run_config(keys_of("inception_v3"), 4, mode="depcha", dtype="bf16", bucket_mb=128, peer=True)


def test_c5_stress_2048_keys_random_order(gpu):
    keys = [min(n, 1 << 16) for n in keys_of("stress")]
    run_config(keys, 4, mode="depcha", dtype="fp32", bucket_mb=64, peer=True, order_seed=1)
