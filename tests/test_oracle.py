"""Pins the CPU oracle (oracle/oracle.c, oracle/schedule.py) to the reference:
its own golden vectors (test_tensor.cpp:49-71), fixtures frozen from the
reference (tests/golden/), and -- when oracle/_ref was built in this container
-- the reference library itself.  CPU only."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import _oracle as O
from schedule import bucket_map, issue_sequence

GOLD = Path(__file__).resolve().parent / "golden"


def test_random_uniform_reference_golden_vectors():
    # R/tests/test_tensor.cpp:49-52 (seed 7) and 58-63 (seeds 1, 2), bit-exact
    exp7 = [0.50877060830571597, 0.89860240578528838, -0.76517143793096398, 0.78382635342495255,
            -0.71745687359242649, -0.88981368299211394, 0.6650459610628916, 0.80142095291941651]
    exp1 = [-0.73224671197493474, -0.72718592726760556, -0.097570192310923787, -0.95795154316654596]
    exp2 = [0.80720805238798854, 0.7004722791516198, 0.56764093080429623, 0.8506342002308156]
    assert O.random_uniform(8, 7).tolist() == exp7
    assert O.random_uniform(4, 1).tolist() == exp1
    assert O.random_uniform(4, 2).tolist() == exp2


def test_random_uniform_and_mix_seed_match_reference_fixture():
    g = json.loads((GOLD / "random_uniform.json").read_text())
    assert O.random_uniform(8, 7).tolist() == g["seed7_n8"]
    assert O.random_uniform(6, 1000).tolist() == g["seed1000_n6"]
    assert O.mix_seed(2000, 3) == g["mix_seed_2000_3"]
    assert O.mix_seed(7, 0) == g["mix_seed_7_0"]


def test_random_uniform_range_and_long_stream():
    x = O.random_uniform(100000, 0)
    assert x.min() >= -1.0 and x.max() < 1.0
    # 312-word mt19937_64 state: streams longer than one twist stay exact
    ref = O.ref_lib()
    if ref is not None:
        y = np.empty(1000, dtype=np.float64)
        ref.ref_random_uniform(C.c_void_p(y.ctypes.data), 1000, 12345)
        np.testing.assert_array_equal(O.random_uniform(1000, 12345), y)


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_rank_order_sum_matches_reference_transport(R):
    """acceptance.cpp criterion-1 inputs through Transport::allreduce_sum of the
    reference itself (oracle/_ref) vs the oracle restatement: bit-exact."""
    ref = O.ref_lib()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    for i in range(0, 100, 7):
        n = 1 + (i * 7) % 64
        ins = [O.random_uniform(n, O.mix_seed(R * 1000 + i, r)) for r in range(R)]
        bufs = np.concatenate(ins).copy()
        assert ref.ref_allreduce(R, n, C.c_void_p(bufs.ctypes.data)) == 0
        exp = O.rank_order_sum(ins, "f64")
        for r in range(R):
            np.testing.assert_array_equal(bufs[r * n:(r + 1) * n], exp)


def test_sgd_restatement_matches_reference_train_steps_fixture():
    """The fp64 rank-order sum + sgd_update restatement reproduces the
    reference KvStore's final weights (train_steps.npz) bit-for-bit."""
    gold = np.load(GOLD / "train_steps.npz")
    sizes = [int(s) for s in gold["sizes"]]
    K, lr = len(sizes), float(gold["lr"])
    for R in (2, 4):
        rescale = 1.0 / (64 * R)
        for k, n in enumerate(sizes):
            w = O.random_uniform(n, O.mix_seed(7, k))
            grads = [O.random_uniform(n, 1000 + r * K + k) for r in range(R)]
            s = O.rank_order_sum(grads, "f64")
            for _ in range(3):
                w, _ = O.sgd_update(w, s, lr, rescale)
            for mode in ("funnel", "depcha", "concom"):
                for r in range(R):
                    np.testing.assert_array_equal(w, gold[f"{mode}_R{R}_r{r}_k{k}"])


def test_sgd_update_arithmetic_reference_case():
    # R/tests/test_trainer.cpp:182-198
    w, _ = O.sgd_update(np.array([1.0]), np.array([2.0]), 0.5, 1.0)
    assert w[0] == 0.0
    w2 = O.random_uniform(5, 8)
    np.testing.assert_array_equal(O.sgd_update(w2, np.zeros(5), 0.3, 1.0)[0], w2)
    w3, _ = O.sgd_update(np.zeros(3), np.full(3, 128.0 * 0.25), 1.0, 1.0 / 128.0)
    np.testing.assert_allclose(w3, -0.25, atol=1e-15)


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5, 3.0e38, 1e-40], dtype=np.float32)
    h = O.f32_to_bf16_bits(x)
    back = O.bf16_bits_to_f32(h)
    # ties to even: 1 + 2^-8 is halfway between 1 and 1 + 2^-7 -> 1.0
    assert back[0] == 1.0 and back[1] == 1.0 and back[2] == np.float32(1.0 + 2 ** -7)
    assert back[3] == -2.5


def test_issue_sequence_restatement_matches_reference_golden():
    gold = json.loads((GOLD / "issue_kv.json").read_text())
    for mode, g in gold.items():
        mine = issue_sequence(mode, g["K"], g["iters"], g["outstanding"])
        for r in ("0", "1"):
            ref = g["per_rank"][r]
            if mode == "concom":
                for comm in {s.split(":")[1] for s in ref}:
                    assert [s for s in mine if s.split(":")[1] == comm] == \
                        [s for s in ref if s.split(":")[1] == comm]
            else:
                assert mine == ref


def test_appendix_a_scenario_fixture():
    """funnel == depcha sequences, concom per-comm, loss."""
    g = json.loads((GOLD / "issue_scenario.json").read_text())
    assert g["funnel"]["per_rank"] == g["depcha"]["per_rank"]
    for mode in g:
        assert g[mode]["per_rank"]["0"] == g[mode]["per_rank"]["1"] or mode == "concom"
        assert g[mode]["loss"] == 1.3429355172450554
        assert g[mode]["accuracy"] == 0.5625
    assert issue_sequence("funnel", 8, 2) == g["funnel"]["per_rank"]["0"]


def test_bucket_map_spec():
    sizes = [3, 1000, 5, 70000, 64]
    b, off, groups = bucket_map(sizes, 4, 0)
    assert b == [0, 1, 2, 3, 4] and off == [0] * 5 and groups == [[0], [1], [2], [3], [4]]
    b, off, groups = bucket_map(sizes, 4, 4096, issue_order=0)
    # 3 -> 64-elem slot, 1000 -> rounds to 1024; 3+1000 elems = 4012 B <= 4096; +5 -> 4032 B
    assert groups[0] == [0, 1, 2] and off[:3] == [0, 64, 1088]
    assert groups[1] == [3] and groups[2] == [4]
    b2, off2, groups2 = bucket_map(sizes, 4, 4096, issue_order=1)
    assert groups2[0] == [4] and groups2[1] == [3] and groups2[2] == [2, 1, 0]


def test_synth_expect_pinned_to_reference_golden_weights():
    """or_synth_expect (the bench / large-config parity oracle) in fp64 with
    momentum 0 IS the reference trainer's 3-step result: equal, bit for bit,
    to the weights the unmodified reference KvStore produced
    (tests/golden/train_steps.npz, seeds of test_kvstore.cpp:304) at R = 2, 4, 8."""
    gold = np.load(GOLD / "train_steps.npz")
    sizes = [int(x) for x in gold["sizes"]]
    for R in (2, 4, 8):
        w, r64, _ = O.synth_expect(sizes, R, 3, wdt="f64", gdt="f64", lr=float(gold["lr"]), rescale=1.0 / (64 * R))
        off = 0
        for k, n in enumerate(sizes):
            np.testing.assert_array_equal(w[off:off + n], gold[f"depcha_R{R}_r0_k{k}"])
            np.testing.assert_array_equal(r64[off:off + n], gold[f"depcha_R{R}_r0_k{k}"])
            off += n


def test_synth_expect_matches_elementwise_oracle_f32_bf16():
    """The fused fp32 / bf16 expectation equals the element-wise restatement
    (rank_order_sum + sgd_update with momentum), and stays within the
    north-star tolerance of its fp64 restatement (1e-6 fp32, 1e-2 bf16)."""
    sizes, R, steps, mu = [3, 64, 1000], 4, 3, 0.9
    K = len(sizes)
    for gdt, tol in (("f32", 1e-6), ("bf16", 1e-2)):
        w, r64, sc = O.synth_expect(sizes, R, steps, wdt="f32", gdt=gdt, momentum=mu, rescale=1.0 / 256)
        off = 0
        for k, n in enumerate(sizes):
            gs = [O.random_uniform(n, 1000 + r * K + k).astype(np.float32) for r in range(R)]
            if gdt == "bf16":
                g = O.bf16_bits_to_f32(O.rank_order_sum([O.f32_to_bf16_bits(x) for x in gs], "bf16"))
            else:
                g = O.rank_order_sum(gs, "f32")
            wk = O.random_uniform(n, O.mix_seed(7, k)).astype(np.float32)
            m = np.zeros(n, np.float32)
            for _ in range(steps):
                wk, m = O.sgd_update(wk, g, 0.1, 1.0 / 256, mu, m, kind="f32")
            np.testing.assert_array_equal(w[off:off + n], wk)
            off += n
        assert np.max(np.abs(w - r64) / sc) <= tol
