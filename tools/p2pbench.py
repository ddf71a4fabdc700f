#!/usr/bin/env python
"""Per-bucket cost of the collective engines at N ranks (torchrun, 1 process/GPU):
NCCL allreduce, NCCL allreduce + separate SGD kernel, peer-memory allreduce,
and the fused peer-memory allreduce+SGD kernel.  Device time with CUDA events
on the launching stream, max over ranks.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2pbench.py
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1802_06949_b200 import api  # noqa: E402


def busbw_of(n, world, us):
    """nccl-tests bus bandwidth of an allreduce of n fp32 elements, GB/s."""
    return round(4 * n * 2 * (world - 1) / world / (us * 1e3), 1)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--mb", type=float, nargs="+", default=[1, 4, 25, 100])
    p.add_argument("--iters", type=int, default=20)
    a = p.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    name = [f"p2pb_{os.getpid()}_{time.time_ns() % 10**9}"]
    dist.broadcast_object_list(name, src=0)
    tr = api.Transport.nccl(name[0], world, rank, local, 60000)
    assert tr.p2p_capable()
    s = torch.cuda.Stream()
    sh = s.cuda_stream
    res = {}
    for mb in a.mb:
        n = int(mb * 2**20 / 4) // 64 * 64
        buf = torch.randn(n, device="cuda")
        w = torch.randn(n, device="cuda")
        m = torch.zeros(n, device="cuda")
        peers = tr.share_buffer(buf.data_ptr())
        ent = [(w.data_ptr(), buf.data_ptr(), m.data_ptr(), n)]

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.iters):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.iters])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return round(t.item() * 1000, 2)  # us

        r = {}
        r["nccl_us"] = timed(lambda: tr.allreduce_sum(0, rank, buf, 0, sh))
        r["nccl_plus_sgd_us"] = timed(lambda: (tr.allreduce_sum(0, rank, buf, 0, sh),
                                               api.sgd_update(ent, api.F32, api.F32, 0.1, 1e-3, 0.9, sh)))
        r["p2p_us"] = timed(lambda: tr.allreduce_p2p(0, rank, peers, n, api.F32, 0, None, sh))
        r["p2p_fused_sgd_us"] = timed(lambda: tr.allreduce_p2p(0, rank, peers, n, api.F32, 0,
                                                               (ent, api.F32, 0.1, 1e-3, 0.9), sh))
        r["p2p_fused_sgd_shard_us"] = timed(lambda: tr.allreduce_p2p(0, rank, peers, n, api.F32, 0,
                                                                     (ent, api.F32, 0.1, 1e-3, 0.9, 1), sh))
        r["sgd_only_us"] = timed(lambda: api.sgd_update(ent, api.F32, api.F32, 0.1, 1e-3, 0.9, sh))
        if tr.nvls_capable():
            uc, mc = tr.alloc_nvls(4 * n)
            api.pack([(buf.data_ptr(), uc, n)], api.F32, api.F32, sh)
            torch.cuda.synchronize()
            entv = [(w.data_ptr(), uc, m.data_ptr(), n)]
            r["nvls_us"] = timed(lambda: tr.allreduce_nvls(0, rank, uc, mc, n, api.F32, 0, None, sh))
            r["nvls_fused_sgd_us"] = timed(lambda: tr.allreduce_nvls(0, rank, uc, mc, n, api.F32, 0,
                                                                     (entv, api.F32, 0.1, 1e-3, 0.9), sh))
            r["nvls_busbw"] = busbw_of(n, world, r["nvls_us"])
        r["nccl_busbw"] = busbw_of(n, world, r["nccl_us"])
        r["p2p_busbw"] = busbw_of(n, world, r["p2p_us"])
        res[f"{mb}MB"] = r
    if rank == 0:
        print(json.dumps({"world": world, "results": res}))
    dist.barrier()
    tr.close()


if __name__ == "__main__":
    main()
