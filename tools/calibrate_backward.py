#!/usr/bin/env python
"""Calibrates the synthetic backward from a real torchvision backward on the
B200: per-parameter gradient-ready times (CUDA events recorded by
post-accumulate-grad hooks) relative to the start of backward.

    python tools/calibrate_backward.py --model resnet50 --batch 64 [--amp]

Writes paper_1802_06949_b200/calibration/<model>_b<batch>[_amp].json with the
ready time of every key (parameter order = KVStore key order); the bench's
synthetic producer holds key k for ready[k] - ready[k+1] (keys become ready in
descending order)."""
import argparse
import json
import sys
from pathlib import Path

import torch
import torchvision.models as tvm

ROOT = Path(__file__).resolve().parent.parent


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="resnet50")
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--amp", action="store_true")
    p.add_argument("--iters", type=int, default=10)
    a = p.parse_args()
    torch.backends.cudnn.benchmark = True
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    ctor = {"resnet50": tvm.resnet50, "alexnet": tvm.alexnet, "resnet152": tvm.resnet152,
            "inception_v3": lambda: tvm.inception_v3(aux_logits=True, init_weights=False)}[a.model]
    model = ctor().cuda().to(memory_format=torch.channels_last)
    params = list(model.parameters())
    size = 299 if a.model == "inception_v3" else 224
    x = torch.randn(a.batch, 3, size, size, device="cuda").to(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (a.batch,), device="cuda")
    events = [None] * len(params)

    def hook(i):
        def h(_p):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            events[i] = e
        return h

    for i, prm in enumerate(params):
        prm.register_post_accumulate_grad_hook(hook(i))
    crit = torch.nn.CrossEntropyLoss()
    readies, bwd, fwd = [], [], []
    for it in range(a.iters + 3):
        model.zero_grad(set_to_none=True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=a.amp):
            out = model(x)
            if isinstance(out, tuple) or hasattr(out, "logits"):
                out = out[0] if isinstance(out, tuple) else out.logits
            loss = crit(out.float(), y)
        e1.record()
        loss.backward()
        e2.record()
        torch.cuda.synchronize()
        if it >= 3:
            fwd.append(e0.elapsed_time(e1))
            bwd.append(e1.elapsed_time(e2))
            readies.append([e1.elapsed_time(ev) for ev in events])
    ready = [sorted(r[i] for r in readies)[len(readies) // 2] for i in range(len(params))]
    res = {"model": a.model, "batch": a.batch, "amp": a.amp, "gpu": torch.cuda.get_device_name(),
           "forward_ms": sorted(fwd)[len(fwd) // 2], "backward_ms": sorted(bwd)[len(bwd) // 2],
           "sizes": [int(p.numel()) for p in params], "ready_ms": ready}
    out_dir = ROOT / "paper_1802_06949_b200" / "calibration"
    out_dir.mkdir(exist_ok=True)
    name = f"{a.model}_b{a.batch}{'_amp' if a.amp else ''}.json"
    (out_dir / name).write_text(json.dumps(res))
    print(json.dumps({k: v for k, v in res.items() if k not in ("sizes", "ready_ms")}))


if __name__ == "__main__":
    sys.exit(main())
