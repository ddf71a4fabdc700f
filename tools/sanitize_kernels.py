#!/usr/bin/env python
"""Every single-GPU kernel of the hot path on small, awkward shapes, meant to
run under compute-sanitizer:

    compute-sanitizer --tool memcheck python tools/sanitize_kernels.py
    compute-sanitizer --tool racecheck python tools/sanitize_kernels.py

Shapes: tails that are not a multiple of the 8-element group, keys whose
pointers are not 16-byte aligned (the scalar paths), fp64 / fp32 / bf16, with
and without momentum; plus a KvStore round (resident tables: pack_tab /
sgd_tab) over fusion buckets.  Prints "sanitize ok" when every call returned.

(compute-sanitizer is closed on the round's GPU pool; the script runs plain
there, and the parity tests cover the same shapes against the CPU oracle.)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1802_06949_b200 import Engine, KvConfig, KvStore, Slot, Transport, api  # noqa: E402

DT = {api.F64: torch.float64, api.F32: torch.float32, api.BF16: torch.bfloat16}


def main():
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream().cuda_stream
    sizes = [1, 7, 8, 9, 63, 1000, 4097]
    for sdt, ddt in ((api.F64, api.F64), (api.F32, api.F32), (api.F32, api.BF16), (api.BF16, api.BF16),
                     (api.BF16, api.F32)):
        for off in (0, 1):  # element offset 1: unaligned -> scalar path
            src = [torch.randn(n + off, device=dev).to(DT[sdt]) for n in sizes]
            dst = [torch.zeros(n + off, device=dev).to(DT[ddt]) for n in sizes]
            ents = [(a[off:].data_ptr(), b[off:].data_ptr(), n) for a, b, n in zip(src, dst, sizes)]
            api.pack(ents, sdt, ddt, s)
    for dt in (api.F64, api.F32, api.BF16):
        for m in (1, 2, 3, 8):
            n = 4097
            ins = [torch.randn(n, device=dev).to(DT[dt]) for _ in range(m)]
            outs = [torch.zeros(n, device=dev).to(DT[dt]) for _ in range(2)]
            api.sum_buffers([x.data_ptr() for x in ins], [y.data_ptr() for y in outs], n, dt, s)
    for wdt, gdt in ((api.F64, api.F64), (api.F32, api.F32), (api.F32, api.BF16)):
        for mom in (0.0, 0.9):
            for off in (0, 1):
                mdt = torch.float64 if wdt == api.F64 else torch.float32
                w = [torch.randn(n + off, device=dev).to(DT[wdt]) for n in sizes]
                g = [torch.randn(n + off, device=dev).to(DT[gdt]) for n in sizes]
                v = [torch.zeros(n + off, device=dev, dtype=mdt) for n in sizes]
                ents = [(a[off:].data_ptr(), b[off:].data_ptr(), c[off:].data_ptr() if mom else 0, n)
                        for a, b, c, n in zip(w, g, v, sizes)]
                api.sgd_update(ents, wdt, gdt, 0.1, 0.01, mom, s)
    x = torch.randn(4097, device=dev)
    out = torch.zeros(1, device=dev, dtype=torch.float64)
    api.checksum(x.data_ptr(), x.numel(), api.F32, out.data_ptr(), s)
    y = torch.zeros_like(x)
    api.synth_backward(x.data_ptr(), y.data_ptr(), x.numel(), api.F32, 1000, 4, s)
    torch.cuda.synchronize()

    # a KvStore round: resident kernel tables over fusion buckets, 1 rank
    eng = Engine(2, 0, None, 0)
    tr = Transport.local(1, 10000)
    K = len(sizes)
    store = KvStore(eng, tr, 0, KvConfig("depcha", 1, K, bucket_bytes=16 * 1024, issue_order=1))
    ws = [Slot(torch.randn(n, device=dev), eng.new_variable()) for n in sizes]
    gs = [Slot(torch.randn(n, device=dev), eng.new_variable()) for n in sizes]
    for k in range(K):
        store.init(k, ws[k])
    eng.wait_all()
    for _ in range(2):
        store.push(list(range(K)), gs)
        store.pull_update(list(range(K)), ws, 0.1, 0.01, 0.9)
    eng.wait_all()
    store.close()
    eng.close()
    tr.close()
    torch.cuda.synchronize()
    print("sanitize ok")


if __name__ == "__main__":
    main()
