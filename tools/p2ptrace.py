#!/usr/bin/env python
"""Phase timeline of the fused peer kernel (the N>1 hot kernel), which ncu
cannot replay: its CTAs wait on CTAs of other GPUs.  Every CTA stamps
%globaltimer at 5 points (CSB_P2P_TRACE=1): start, past the arrival
barrier, own shard done (reduce + update [+ own-shard gather]), past
barrier 1, end.  The bench workload (ResNet-50 set, DepCha, one 100 MiB
bucket, momentum 0.9, ZeRO-1, direct gradient reads unless --staged) runs
--steps steps; the last launch's stamps are summarised per rank.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/p2ptrace.py [--staged] [--replicated]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

os.environ["CSB_P2P_TRACE"] = "1"  # before the transport exists
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1802_06949_b200 import api, keysets  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--staged", action="store_true", help="stage the gradients (no register_grads)")
    ap.add_argument("--replicated", action="store_true", help="replicated update instead of ZeRO-1")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--keyset", default="resnet50")
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"])
    ap.add_argument("--bucket-mb", type=float, default=100)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    name = [f"p2ptrace_{os.getpid()}_{time.time_ns() % 10**9}"]
    dist.broadcast_object_list(name, src=0)
    tr = api.Transport.nccl(name[0], world, rank, local, 60000)
    eng = api.Engine(4, rank, None, local)
    keys = keysets.load(a.keyset)
    dt = {"fp32": api.F32, "bf16": api.BF16}[a.dtype]
    m = api.SynthModel(eng, tr, rank, world, keys, mode="depcha", g_dtype=dt, comm_dtype=dt,
                       bucket_bytes=int(a.bucket_mb * 2**20), issue_order=1, lr=0.1,
                       rescale=1.0 / (64 * world), momentum=0.9, p2p=1, zero=not a.replicated,
                       direct_grads=not a.staged)
    m.init()
    m.run(1, m.BACKWARD | m.COMM)
    m.run(3, m.COMM)
    dist.barrier()
    ms = m.run(a.steps, m.COMM) / a.steps
    st = tr.p2p_stamps(rank).astype(np.int64)
    st = st[st[:, 0] != 0]
    t0 = st[:, 0].min()
    d = {"arrive": st[:, 1] - st[:, 0], "own_shard": st[:, 2] - st[:, 1], "barrier1": st[:, 3] - st[:, 2],
         "other_shards": st[:, 4] - st[:, 3]}
    summary = {"rank": rank, "ctas": int(len(st)), "step_ms": round(ms, 4),
               "launch_us": round(float(st[:, 4].max() - t0) / 1e3, 2),
               "first_cta_start_to_last_start_us": round(float(st[:, 0].max() - t0) / 1e3, 2)}
    for k, v in d.items():
        summary[k + "_us"] = {"median": round(float(np.median(v)) / 1e3, 2), "max": round(float(v.max()) / 1e3, 2)}
    # when the phases END across the grid (relative to the first CTA's start)
    for i, k in enumerate(["past_barrier0", "own_shard_done", "past_barrier1", "end"], start=1):
        summary[k + "_at_us"] = {"median": round(float(np.median(st[:, i] - t0)) / 1e3, 2),
                                 "max": round(float((st[:, i] - t0).max()) / 1e3, 2)}
    out = [None] * world
    dist.all_gather_object(out, summary)
    if rank == 0:
        print(json.dumps({"tool": "p2ptrace", "world": world, "keyset": a.keyset, "dtype": a.dtype,
                          "gradients": "staged" if a.staged else "direct",
                          "update": "replicated" if a.replicated else "zero1", "ranks": out}))
    m.close()
    eng.close()
    dist.barrier()
    tr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
