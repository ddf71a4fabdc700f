#!/usr/bin/env python
"""Host cost of one cs_pack / cs_sgd_update launch vs table size (param-block CAP)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1802_06949_b200 import api  # noqa: E402

s = torch.cuda.current_stream().cuda_stream
buf = torch.zeros(1 << 20, device="cuda")
out = {}
for n in (1, 4, 5, 32, 33, 64, 161, 512):
    ent = [(buf.data_ptr() + 1024 * i, buf.data_ptr() + 1024 * i + 512 * 1024, 64) for i in range(n)]
    for _ in range(20):
        api.pack(ent, api.F32, api.F32, s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        api.pack(ent, api.F32, api.F32, s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out[n] = {"host_us": round((t1 - t0) / 200 * 1e6, 2), "total_us": round((t2 - t0) / 200 * 1e6, 2)}
print(json.dumps(out))
