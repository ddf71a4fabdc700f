"""Freeze golden fixtures from the UNMODIFIED reference (collsim), compiled from
/root/reference by oracle/Makefile into oracle/_ref/libcollsim_ref.so.

Run here (the reference sources exist only in this container):
    make -C oracle all ref && python tests/golden/make_golden.py

Outputs (committed, small):
  random_uniform.json   reference generator values (test_tensor.cpp:49-71 seeds + extra)
  issue_scenario.json   Appendix-A per-rank collective sequences from run_scenario
                        (diamond, workers 2, engine threads 4, outstanding 2, batch 64,
                        samples 160, seed 1) for funnel / depcha / concom
  issue_kv.json         per-rank per-comm collective sequences of the trainer loop
                        shape (trainer.cpp:112-141) over K=8 synthetic keys, 2 iterations
  train_steps.npz       final fp64 weights of every rank after 3 push/pull/sgd
                        iterations through the reference KvStore, per mode and R in {2, 4, 8}
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import _oracle as O  # noqa: E402

R = O.ref_lib()
assert R is not None, "build oracle/_ref first: make -C oracle ref"

TRAIN_SIZES = [1, 7, 64, 300, 4097]
LR = 0.1


def ref_random_uniform(n, seed):
    out = np.empty(n, dtype=np.float64)
    R.ref_random_uniform(C.c_void_p(out.ctypes.data), n, seed)
    return out


def read_trace(path):
    with open(path) as f:
        return [json.loads(line) for line in f if line.strip()]


def seqs_from_trace(events, nranks):
    """per rank: list of 'kind:comm:seq:key' from coll_enqueued, in emission order."""
    out = {r: [] for r in range(nranks)}
    for ev in events:
        if ev["event"] == "coll_enqueued":
            out[ev["rank"]].append(f"{ev['kind']}:{ev['comm']}:{ev['seq']}:{ev.get('key', -1)}")
    return out


def main():
    rnd = {
        "seed7_n8": ref_random_uniform(8, 7).tolist(),
        "seed1_n4": ref_random_uniform(4, 1).tolist(),
        "seed2_n4": ref_random_uniform(4, 2).tolist(),
        "seed1000_n6": ref_random_uniform(6, 1000).tolist(),
        "mix_seed_2000_3": int(R.ref_mix_seed(2000, 3)),
        "mix_seed_7_0": int(R.ref_mix_seed(7, 0)),
    }
    (HERE / "random_uniform.json").write_text(json.dumps(rnd, indent=1))

    scen = {}
    for mode in ("funnel", "depcha", "concom"):
        with tempfile.TemporaryDirectory() as d:
            p = Path(d) / "t.jsonl"
            loss, acc = C.c_double(), C.c_double()
            rc = R.ref_run_scenario(mode.encode(), 2, 4, 2, 1, 64, 160, 1, str(p).encode(),
                                    C.byref(loss), C.byref(acc))
            assert rc == 0, R.ref_last_error()
            scen[mode] = {"per_rank": seqs_from_trace(read_trace(p), 2), "loss": loss.value,
                          "accuracy": acc.value}
    (HERE / "issue_scenario.json").write_text(json.dumps(scen, indent=1))

    kvseq = {}
    K, iters = 8, 2
    for mode, outstanding in (("funnel", 1), ("depcha", 1), ("concom", 2)):
        sizes = np.array([5] * K, dtype=np.int64)
        g = [np.full(5, float(r + 1)) for r in range(2) for _ in range(K)]
        w0 = [np.zeros(5) for _ in range(K)]
        wout = [np.zeros(5) for _ in range(2 * K)]
        with tempfile.TemporaryDirectory() as d:
            p = Path(d) / "t.jsonl"
            rc = R.ref_train_steps(mode.encode(), 2, K, C.c_void_p(sizes.ctypes.data),
                                   (C.c_void_p * len(g))(*[x.ctypes.data for x in g]),
                                   (C.c_void_p * K)(*[x.ctypes.data for x in w0]),
                                   (C.c_void_p * len(wout))(*[x.ctypes.data for x in wout]),
                                   iters, LR, 1.0 / 128, 4, outstanding, str(p).encode())
            assert rc == 0, R.ref_last_error()
            kvseq[mode] = {"outstanding": outstanding, "K": K, "iters": iters,
                           "per_rank": seqs_from_trace(read_trace(p), 2)}
    (HERE / "issue_kv.json").write_text(json.dumps(kvseq, indent=1))

    arrays = {}
    sizes = np.array(TRAIN_SIZES, dtype=np.int64)
    K = len(TRAIN_SIZES)
    for nranks in (2, 4, 8):
        rescale = 1.0 / (64 * nranks)
        grads = [O.random_uniform(int(sizes[k]), 1000 + r * K + k) for r in range(nranks) for k in range(K)]
        w0 = [O.random_uniform(int(sizes[k]), O.mix_seed(7, k)) for k in range(K)]
        for mode, outstanding in (("funnel", 1), ("depcha", 1), ("concom", 2)):
            wout = [np.zeros(int(sizes[k])) for _ in range(nranks) for k in range(K)]
            rc = R.ref_train_steps(mode.encode(), nranks, K, C.c_void_p(sizes.ctypes.data),
                                   (C.c_void_p * len(grads))(*[x.ctypes.data for x in grads]),
                                   (C.c_void_p * K)(*[x.ctypes.data for x in w0]),
                                   (C.c_void_p * len(wout))(*[x.ctypes.data for x in wout]),
                                   3, LR, rescale, 4, outstanding, b"")
            assert rc == 0, R.ref_last_error()
            for r in range(nranks):
                for k in range(K):
                    arrays[f"{mode}_R{nranks}_r{r}_k{k}"] = wout[r * K + k]
    np.savez_compressed(HERE / "train_steps.npz", sizes=sizes, lr=LR, **arrays)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
