#!/usr/bin/env python
"""Kernel microbenchmark: (a) pack, (b) sum, (c) sgd at bucket-like sizes.
Times N back-to-back launches with CUDA events (L2 defeated by a working set
> 126 MB) and prints algorithmic GB/s per kernel.  Used for ncu captures:
  python tools/kbench.py --only sgd --iters 3
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1802_06949_b200 import api  # noqa: E402


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=25557032)  # ResNet-50 params
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--only", default="")
    p.add_argument("--keys", type=int, default=1)
    a = p.parse_args()
    s = torch.cuda.current_stream().cuda_stream
    n = a.n
    res = {}
    f32 = torch.float32
    if a.only in ("", "pack"):
        src = torch.randn(n, device="cuda", dtype=f32)
        dst = torch.empty(n, device="cuda", dtype=f32)
        per = n // a.keys
        ent = [(src.data_ptr() + 4 * i * per, dst.data_ptr() + 4 * i * per, per) for i in range(a.keys)]
        ms = timeit(lambda: api.pack(ent, api.F32, api.F32, s), a.iters)
        res["pack_f32"] = {"ms": ms, "GBps": 8 * per * a.keys / ms / 1e6}
        dstb = torch.empty(n, device="cuda", dtype=torch.bfloat16)
        entb = [(src.data_ptr(), dstb.data_ptr(), n)]
        ms = timeit(lambda: api.pack(entb, api.F32, api.BF16, s), a.iters)
        res["pack_f32_bf16"] = {"ms": ms, "GBps": 6 * n / ms / 1e6}
        ms = timeit(lambda: dst.copy_(src), a.iters)
        res["torch_copy_f32"] = {"ms": ms, "GBps": 8 * n / ms / 1e6}
        del src, dst, dstb
    if a.only in ("", "sgd"):
        w = torch.randn(n, device="cuda", dtype=f32)
        g = torch.randn(n, device="cuda", dtype=f32)
        m = torch.zeros(n, device="cuda", dtype=f32)
        per = n // a.keys
        ent = [(w.data_ptr() + 4 * i * per, g.data_ptr() + 4 * i * per, m.data_ptr() + 4 * i * per, per)
               for i in range(a.keys)]
        ms = timeit(lambda: api.sgd_update(ent, api.F32, api.F32, 0.1, 0.01, 0.9, s), a.iters)
        res["sgd_mom_f32"] = {"ms": ms, "GBps": 20 * per * a.keys / ms / 1e6}
        ent0 = [(w.data_ptr(), g.data_ptr(), 0, n)]
        ms = timeit(lambda: api.sgd_update(ent0, api.F32, api.F32, 0.1, 0.01, 0.0, s), a.iters)
        res["sgd_f32"] = {"ms": ms, "GBps": 12 * n / ms / 1e6}
        del w, g, m
    if a.only in ("", "sum"):
        R = 8
        nn = n // 2
        bufs = [torch.randn(nn, device="cuda", dtype=f32) for _ in range(R)]
        out = torch.empty(nn, device="cuda", dtype=f32)
        ms = timeit(lambda: api.sum_buffers([b.data_ptr() for b in bufs], [out.data_ptr()], nn, api.F32, s),
                    a.iters)
        res["sum8_f32"] = {"ms": ms, "GBps": 4 * nn * (R + 1) / ms / 1e6}
    print(json.dumps({k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in res.items()}))


if __name__ == "__main__":
    main()
