#!/usr/bin/env python
"""Real ResNet-50 training steps with the KvStore as the gradient path
(SURVEY.md §8 f2), against torch DDP and a no-communication control.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/train_resnet50.py --impl kv|local|ddp [--steps 30 --warmup 10 --batch 64]

impl:
  kv     torch_dp.TorchKvStoreDP: gradients pushed from autograd hooks per
         fusion bucket (DepCha), fused NVLink allreduce + SGD momentum kernel
         (NCCL with --comm nccl), framework stream ordered by engine events
  local  the same KvStore machinery over a 1-rank transport on every GPU
         (pack + update, no communication): the compute-only control, so
         kv - local = exposed communication
  ddp    torch DistributedDataParallel (NCCL, 25 MiB buckets, gradient views)
         + torch.optim.SGD(momentum) -- the library baseline

Synthetic ImageNet-shaped batches (random, fixed per rank), random-init
weights, fp32 with TF32 convolutions/matmuls (the calibration setting of
paper_1802_06949_b200/calibration/resnet50_b64.json).  Device time with CUDA
events on the training stream over --steps steps, max over ranks.  One JSON
line on rank 0.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="kv", choices=["kv", "local", "ddp"])
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--bucket-mb", type=float, default=50.0)
    ap.add_argument("--comm", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--momentum", type=float, default=0.9)
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--channels-last", action="store_true")
    ap.add_argument("--metrics-out", default=None, help="write collsim-metrics-v1 (rank 0)")
    ap.add_argument("--bucket-views", action="store_true", help="gradients accumulate in the comm buckets")
    ap.add_argument("--zero", action="store_true", help="ZeRO-1 sharded optimizer state (kv, N>1)")
    a = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    torch.backends.cudnn.benchmark = True

    import torchvision
    torch.manual_seed(0)
    model = torchvision.models.resnet50().to(dev)
    fmt = torch.channels_last if a.channels_last else torch.contiguous_format
    model = model.to(memory_format=fmt)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn(a.batch, 3, 224, 224, device=dev, generator=gen).to(memory_format=fmt)
    y = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)
    lossf = torch.nn.CrossEntropyLoss()

    engine = transport = dp = None
    if a.impl in ("kv", "local"):
        from paper_1802_06949_b200 import api
        from paper_1802_06949_b200.torch_dp import TorchKvStoreDP
        engine = api.Engine(4, rank if a.impl == "kv" else 0, None, local)
        if a.impl == "kv" and world > 1:
            name = [f"trainr50_{os.getpid()}_{time.time_ns() % 10**9}"]
            dist.broadcast_object_list(name, src=0)
            transport = api.Transport.nccl(name[0], world, rank, local, 120000)
            dp = TorchKvStoreDP(model, engine, transport, rank, world, lr=a.lr, momentum=a.momentum,
                                bucket_mb=a.bucket_mb, p2p=1 if a.comm == "p2p" else 0,
                                bucket_views=a.bucket_views, zero=a.zero)
        else:
            transport = api.Transport.local(1, 120000)
            dp = TorchKvStoreDP(model, engine, transport, 0, 1, lr=a.lr, momentum=a.momentum,
                                rescale=1.0 / world, bucket_mb=a.bucket_mb, bucket_views=a.bucket_views)

        def step():
            dp.zero_grad()
            loss = lossf(model(x), y)
            loss.backward()
            dp.step()
            return loss
    else:
        from torch.nn.parallel import DistributedDataParallel as DDP
        net = DDP(model, device_ids=[local], bucket_cap_mb=a.bucket_mb, gradient_as_bucket_view=True) \
            if world > 1 else model
        opt = torch.optim.SGD(model.parameters(), lr=a.lr, momentum=a.momentum)

        def step():
            opt.zero_grad(set_to_none=False)
            loss = lossf(net(x), y)
            loss.backward()
            opt.step()
            return loss

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    last_loss = loss.detach().float()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.all_reduce(last_loss, op=dist.ReduceOp.SUM)
        last_loss /= world
    if a.metrics_out and rank == 0:
        from paper_1802_06949_b200.metrics import Metrics, write_metrics
        write_metrics(Metrics(mode="depcha" if a.impl != "ddp" else "ddp", model="torchvision-resnet50",
                              workers=world, engine_threads=4, outstanding=1, epochs=1,
                              global_batch=a.batch * world, seed=1000, epoch_times_s=[ms * a.steps / 1e3],
                              final_train_loss=float(last_loss.item()), test_accuracy=0.0,
                              max_concurrent_collectives=1, compute_overlap_observed=True,
                              b200={"impl": a.impl, "comm": a.comm, "steps": a.steps, "ms_per_step": ms,
                                    "test_accuracy": "n/a (synthetic data)"}), a.metrics_out)
    if rank == 0:
        print(json.dumps({"tool": "train_resnet50", "impl": a.impl, "comm": a.comm if a.impl == "kv" else None,
                          "n_gpus": world, "batch_per_gpu": a.batch, "ms_per_step": round(ms, 3),
                          "images_per_s": round(world * a.batch / ms * 1e3, 1), "bucket_mb": a.bucket_mb,
                          "momentum": a.momentum, "channels_last": a.channels_last,
                          "bucket_views": a.bucket_views, "zero": a.zero,
                          "buckets": len(dp.groups) if dp else None, "steps": a.steps, "warmup": a.warmup,
                          "data": "synthetic random images, random-init torchvision resnet50, fp32/TF32"}),
              flush=True)
    if dp:
        dp.close()
        engine.close()
        transport.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
