#!/usr/bin/env python
"""bench.py -- aggregated gradient GB/s/GPU & exposed comm ms/iter (BASELINE.json).

Workload (N=1 default, BASELINE.json configs[1]): the ResNet-50 gradient set
(161 keys, 25,557,032 fp32 params, torchvision parameter order) under DepCha,
one 100 MiB fusion bucket in gradient-ready (descending) order, SGD with
momentum 0.9.  One "step" = one pass of the hot path over every key: push
(kernel (a) packs the gradients into the bucket) -> allreduce (the identity
at N=1; at N>1 the fused peer-memory kernel: rank-order reduce-scatter over
NVLink + SGD/momentum update + all-gather, ZeRO-1 for fp32 sets) -> fused
pull+update (kernel (c)).

  value          aggregated gradient GB/s PER GPU (the metric's unit) =
                 gradient bytes per rank / device step time (max over ranks);
                 gradients resident in HBM, working set (~409 MB/rank) > the
                 126 MB L2, so no flush is needed.  `whole_job_gbs` = N x value.
  e2e            the same metric through the C ABI with HOST buffers: every
                 step copies the gradients H2D from pinned memory, runs the
                 path and reads the weight checksum back D2H (wall clock).
  exposed_comm   T(synthetic backward + aggregation) - T(synthetic backward +
                 local update), per iteration, CUDA events, max over ranks.
  roofline       dominant kernel, CUDA-event timed per launch on its stream,
                 algorithmic bytes / duration vs measured HBM (N=1) or NVLink.
  parity         a fresh model of the same config, 3 steps, weights read back
                 and checked against the CPU oracle (the checker, oracle.c
                 or_synth_expect, pinned to the reference's golden weights):
                 bit-exact vs the fp32 restatement, max relative error vs fp64.
  f64            the same step in the reference's own arithmetic (fp64
                 weights and gradients, plain SGD), bit-exact vs the reference.
  cpu_baseline   the reference (oracle/_ref, compiled from /root/reference)
                 timed on this host's cores on a bounded sample (rank 0, N=1).

`--gpus N` without torchrun re-launches itself under torch.distributed.run
(one process per GPU, NCCL between them) and fails if fewer than N GPUs are
visible.  `--impl reference` times the reference's own CPU path instead
(rank 0 only; R = N rank threads), with the identical `config`.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
import zlib
from pathlib import Path

ROOT = Path(__file__).resolve().parent

METRIC = "aggregated gradient GB/s/GPU & exposed comm ms/iter at 1/2/4/8 B200"
CONFIGS = {
    # name: (keyset, mode, outstanding, dtype, bucket_mb, backward calibration or fixed ms)
    "resnet50": ("resnet50", "depcha", 1, "fp32", 100, "resnet50_b64.json"),
    "alexnet": ("alexnet", "concom", 4, "fp32", 25, "alexnet_b64_amp.json"),
    "resnet152": ("resnet152", "depcha", 1, "bf16", 128, "resnet152_b64_amp.json"),
    "inception_v3": ("inception_v3", "depcha", 1, "bf16", 128, 30.0),
    # 256 MiB buckets: 51 launches per step instead of 236 (64 MiB measured
    # slower and, at 2 GPUs, multimodal: profiles/r2_stress_buckets.log)
    "stress": ("stress", "depcha", 1, "fp32", 256, 0.0),
    "uniform16": ("uniform16x1048576", "funnel", 1, "fp32", 0, 0.0),
}
CALIB = ROOT / "paper_1802_06949_b200" / "calibration"
ELEM = {"fp32": 4, "bf16": 2, "fp64": 8}


def load_keys(keyset: str) -> list[int]:
    """Key sizes from paper_1802_06949_b200/keysets.py, loaded as a plain
    module file: the reference arm must not import the package (which maps
    libcollsim_b200.so)."""
    spec = importlib.util.spec_from_file_location("_csb_keysets", ROOT / "paper_1802_06949_b200" / "keysets.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.load(keyset)


def backward_profile(spec, keys):
    """-> (ready_ms per key or None, backward ms, description).  Calibration
    files hold per-parameter gradient-ready times measured on a B200 with a
    real torchvision backward (tools/calibrate_backward.py, batch 64)."""
    if isinstance(spec, str):
        d = json.loads((CALIB / spec).read_text())
        if d["sizes"] != keys:
            raise SystemExit(f"calibration {spec} does not match the key set")
        return d["ready_ms"], d["backward_ms"], f"measured {d['model']} batch {d['batch']} " \
            f"{'bf16 AMP' if d['amp'] else 'fp32/TF32'} backward on {d['gpu']} ({spec})"
    return None, float(spec), f"fixed {spec} ms split in proportion to key size"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="resnet50", choices=sorted(CONFIGS))
    p.add_argument("--mode", default=None, choices=["funnel", "depcha", "concom"])
    p.add_argument("--outstanding", type=int, default=None)
    p.add_argument("--bucket-mb", type=float, default=None)
    p.add_argument("--issue-order", default="descending", choices=["ascending", "descending"])
    p.add_argument("--momentum", type=float, default=0.9)
    p.add_argument("--backward-ms", type=float, default=None)
    p.add_argument("--engine-threads", type=int, default=4)
    p.add_argument("--no-extras", action="store_true", help="headline only (no e2e/exposed/roofline/cpu)")
    p.add_argument("--no-parity", dest="parity", action="store_false")
    p.add_argument("--parity-steps", type=int, default=3)
    p.add_argument("--cpu-steps", type=int, default=2)
    p.add_argument("--no-zero", dest="zero", action="store_false",
                   help="replicated optimizer state instead of ZeRO-1 (the fused kernel's default at N>1 for "
                        "fp32 gradients: sharded master weights + momentum, weight all-gather, bit-identical "
                        "results; bf16 gradient sets keep the replicated update, whose all-gather moves bf16 "
                        "sums instead of fp32 weights)")
    p.add_argument("--no-direct", dest="direct", action="store_false",
                   help="stage the gradients into the comm buckets (kvstore.cpp:109) instead of registering the "
                        "gradient arena and reading the gradients in place (every rank's over NVLink at N>1)")
    p.add_argument("--grad-views", action="store_true",
                   help="gradients produced in place in the comm buckets (gradient-as-bucket-view): "
                        "push copies nothing")
    p.add_argument("--comm", default=None, choices=["nccl", "p2p", "nvls"],
                   help="collective engine for N>1: the fused NVLink peer-memory kernel (default; "
                        "NCCL for ConCom, whose extra communicators run concurrently), NCCL, or NVLS")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: one process per GPU through
    torch.distributed.run (rendezvous on 127.0.0.1).  Returns the child's exit
    code, or None when this process is already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {n} CUDA device(s) visible"}),
              flush=True)
        return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks
    line).  Each query briefly stalls the driver: at 4 GPUs a query landing
    inside the ~12 ms timed region was measured to add ~1 ms/step, and an
    in-process NVML sampler at 10 ms slowed every run.  So the period is
    200 ms and the timed region starts right after a sample arrives
    (wait_first); the soak that follows keeps the same steps running so the
    next samples see this load."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, devices: str, enabled: bool = True):
        self.device = devices  # "0" or "0,1,2,3": one process samples every GPU of the job
        self.ndev = len(devices.split(","))
        self.rows = []
        self.proc = None
        self.enabled = enabled

    def __enter__(self):
        if os.environ.get("CSB_CLOCKS") == "off" or not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def wait_first(self, timeout: float = 5.0):
        """Returns right after a fresh sample arrived (the next query is
        ~200 ms away)."""
        t0 = time.time()
        n0 = len(self.rows)
        while self.proc and len(self.rows) < n0 + self.ndev and time.time() - t0 < timeout:
            time.sleep(0.001)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# committed `ncu --set full` captures of the N=1 headline workload, newest first
NCU_CAPTURES = ("r2g", "r2f", "r2", "r1b")  # newest first


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture of this exact workload
    (profiles/<round>_<kernel>_raw.csv, ResNet-50 DepCha 100 MiB, N=1), or None."""
    import csv
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for tag in NCU_CAPTURES:
        path = ROOT / "profiles" / f"{tag}_{kernel}_raw.csv"
        if not path.exists():
            continue
        try:
            rows = list(csv.reader(path.open()))
            head, units, vals = rows[0], rows[1], rows[2]
            total = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = head.index(k)
                total += float(vals[i].replace(",", "")) * scale[units[i]]
            return {"bytes": int(total), "source": f"profiles/{path.name} (ncu --set full, one launch)"}
        except Exception:
            continue
    return None


def peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def workload(args):
    keyset, mode, outstanding, dtype, bucket_mb, bwd_spec = CONFIGS[args.config]
    mode = args.mode or mode
    outstanding = args.outstanding or outstanding
    bucket_mb = args.bucket_mb if args.bucket_mb is not None else bucket_mb
    return keyset, mode, outstanding, dtype, bucket_mb, bwd_spec


def direct_active(args, mode, bucket_mb, world) -> bool:
    """Registered gradients read in place (KvStore.register_grads), nothing
    staged: at N>1 by the fused peer kernel over NVLink, at N=1 by the fused
    pack + update kernel (DepCha / Funnel over fusion buckets)."""
    return (args.direct and not args.grad_views and mode != "concom" and bool(bucket_mb)
            and args.comm in (None, "p2p"))


def config_dict(args, keys, mode, outstanding, dtype, bucket_mb, world) -> dict:
    """The workload, identical in both arms (the driver compares them)."""
    return {"workload": f"{args.config}-{mode}", "keys": len(keys), "params": sum(keys), "mode": mode,
            "outstanding": outstanding, "grad_dtype": dtype, "bucket_mb": bucket_mb,
            "issue_order": args.issue_order, "momentum": args.momentum, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (no flush)",
            "producer_order": "per-rank random (seeded)" if args.config == "stress" else "reverse key order",
            "grad_layout": "bucket views (produced in place; push copies nothing)" if args.grad_views
            else ("separate gradient tensors in one registered region (KvStore.register_grads): the fused "
                  "kernel reads the gradients in place (every rank's over NVLink at N>1), nothing staged "
                  "into the comm buckets"
                  if direct_active(args, mode, bucket_mb, world) else
                  "separate gradient tensors (push packs them into the comm buckets, kvstore.cpp:109)"),
            "step": "push + allreduce + pull/SGD update over every key (trainer.cpp:112-141), no backward",
            "value_basis": f"gradient bytes per rank = params x {ELEM[dtype]} B ({dtype}) per step time, per GPU"}


# ------------------------------------------------------------- reference

def ref_lib():
    """The unmodified reference (oracle/_ref/libcollsim_ref.so, compiled from
    /root/reference by oracle/Makefile), loaded on its own: nothing of this
    package and not the oracle restatement."""
    import ctypes as C
    so = ROOT / "oracle" / "_ref" / "libcollsim_ref.so"
    if not so.exists():
        return None
    lib = C.CDLL(str(so))
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_bench.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                              C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p]
    return lib


def run_reference(keys, mode, outstanding, ranks, warmup, iters, elem_bytes):
    """The reference's own CPU path (Engine + KvStore + Transport) on the host
    cores: R rank threads x T engine threads, fp64 (its only dtype), the same
    push / pull / sgd loop as the GPU step (ref_driver.cpp ref_bench)."""
    import ctypes as C
    R = ref_lib()
    if R is None:
        return None
    ncores = os.cpu_count() or 1
    threads = max(2, ncores // ranks)
    sizes = (C.c_int64 * len(keys))(*keys)
    stats = (C.c_double * 2)()
    rescale = 1.0 / (64 * ranks)
    rc = R.ref_bench(mode.encode(), ranks, threads, outstanding, len(keys), sizes, warmup, iters, 0,
                     0.1, rescale, stats)
    if rc != 0:
        raise RuntimeError(R.ref_last_error().decode())
    ms = stats[0]
    gbytes = sum(keys) * elem_bytes
    return {"ms_per_step": ms, "per_gpu": gbytes / (ms * 1e6), "cores": min(ncores, ranks * (threads + 1)),
            "ranks": ranks, "threads": threads, "fp64_bytes_per_rank": stats[1]}


def reference_main(args, keys, mode, outstanding, dtype, bucket_mb):
    rank, _, world = dist_env()
    ranks = world if "WORLD_SIZE" in os.environ else args.gpus
    if rank != 0:
        return 0  # rank 0 runs all R rank threads of the reference on the host
    config = config_dict(args, keys, mode, outstanding, dtype, bucket_mb, ranks)
    ref = run_reference(keys, mode, outstanding, ranks, args.warmup, args.steps, ELEM[dtype])
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcollsim_ref.so not built"}))
        return 0
    v = round(ref["per_gpu"], 4)
    sample = (f"{len(keys)} keys, {ranks} rank thread(s) x {ref['threads']} engine threads, fp64 arithmetic, "
              f"{args.steps} steps after {args.warmup} warm-up (the driver's --steps/--warmup)")
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "GB/s", "n_gpus": ranks, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ref["ms_per_step"], 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random_uniform seeds 1000+r*K+k)", "config": config,
        "whole_job_gbs": round(v * ranks, 4),
        "reference_arithmetic": "fp64 plain SGD (model.cpp:17-27 has no momentum); value counts the config's "
                                f"gradient bytes ({ELEM[dtype]} B/param) so both arms' GB/s measure the same "
                                "work -- the reference moves fp64 (8 B/param)",
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": ref["cores"], "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- parity

def parity_check(api, engine, transport, rank, world, keys, kw, comms, gdt, steps, barrier, dist):
    """A fresh model of the benchmarked config runs `steps` steps (synthetic
    backward + aggregation), its weights are read back and compared with the
    CPU oracle -- the checker, oracle.c or_synth_expect, itself pinned to the
    reference's golden weights (tests/test_oracle.py).  Rank 0 compares; every
    rank's weight CRC must equal rank 0's.  Outside every timed region."""
    import numpy as np
    import torch
    sys.path.insert(0, str(ROOT / "tests"))
    m = api.SynthModel(engine, transport, rank, world, keys, concom_comms=comms,
                       **{**kw, "backward_ns": 0, "grad_views": False})
    m.init()
    m.run(steps, api.SynthModel.BACKWARD | api.SynthModel.COMM)
    barrier()
    K = len(keys)
    # bounded check for huge key sets (C5): every 16th key
    sel = list(range(K)) if sum(keys) <= 2**28 else list(range(0, K, 16))
    w_all = m.read_weights()
    m.close()
    offs = np.concatenate([[0], np.cumsum(keys)])
    w = np.concatenate([w_all[offs[k]:offs[k + 1]] for k in sel]) if len(sel) < K else w_all
    crc = zlib.crc32(w.tobytes())
    agree = True
    if world > 1:
        t = torch.tensor([crc, -crc], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        agree = int(t[0]) == crc and int(t[1]) == -crc
    out = None
    if rank == 0:
        import _oracle as O  # the checker (test infrastructure), never on the measured path
        wname = {api.F64: "f64", api.F32: "f32"}[kw["w_dtype"]]
        gname = {api.F64: "f64", api.F32: "f32", api.BF16: "bf16"}[kw["g_dtype"]]
        cname = {api.F64: "f64", api.F32: "f32", api.BF16: "bf16"}[kw["comm_dtype"]]
        t0 = time.time()
        exp, r64, scale = O.synth_expect(keys, world, steps, wdt=wname, gdt=gname, cdt=cname, lr=kw["lr"],
                                         rescale=kw["rescale"], momentum=kw["momentum"],
                                         keys=None if len(sel) == K else sel)
        err = float(np.max(np.abs(w.astype(np.float64) - r64) / np.maximum(scale, 1e-30)))
        tol = 1e-2 if gname == "bf16" else 1e-6
        out = {"steps": steps, "ranks": world, "keys_checked": len(sel), "elems_checked": int(w.size),
               "bit_exact_vs_restatement": bool(np.array_equal(w, exp)),
               "max_rel_err_vs_f64": err, "tolerance": tol, "within_tolerance": err <= tol,
               "rel_err_scale": "|w0| + lr*rescale*C*sum_r|g_r| per element, C = the gradient's total "
                                "coefficient over the steps (SURVEY 8(c)'s update scale, over T momentum steps)",
               "ranks_agree": agree,
               "oracle": f"oracle/oracle.c or_synth_expect ({wname} weights, {cname} sums in rank order; "
                         f"pinned to the reference's golden weights), {time.time() - t0:.1f} s on the host"}
    barrier()
    return out


# ------------------------------------------------------------------ busbw

def busbw_sweep(api, transport, rank, world, max_over_ranks, sizes_mb=(16, 64, 256), iters=20):
    """Bus bandwidth (nccl-tests convention: algbw x 2(N-1)/N) of one fp32
    bucket allreduce per size: the peer-memory kernel alone (rank-order
    sums, no update), the same fused with the SGD / momentum update of the
    whole bucket, and NCCL's allreduce.  CUDA events on the launch stream,
    max over ranks.  Peak: the measured peer copy (770 GB/s per direction);
    `ceiling_gbs` is the all-to-all NVLink ceiling tools/nvlink_probe.cu
    measures with every GPU sending and receiving at once."""
    import torch
    out = {"unit": "GB/s", "peak": peaks().get("nvlink_gbs_per_dir", 770.0),
           "ceiling_gbs": {2: 692.5, 4: 581.2}.get(world),
           "ceiling_source": "profiles/r2_nvlink_probe_n%d.txt best all-to-all pattern" % world,
           "sizes": {}}
    s = torch.cuda.Stream()
    sh = s.cuda_stream
    for mb in sizes_mb:
        n = int(mb * 2**20 / 4) // 64 * 64
        buf = torch.randn(n, device="cuda")
        w = torch.randn(n, device="cuda")
        m = torch.zeros(n, device="cuda")
        peers = transport.share_buffer(buf.data_ptr())
        upd = ([(w.data_ptr(), buf.data_ptr(), m.data_ptr(), n)], api.F32, 0.1, 1e-3, 0.9)

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(iters):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            return max_over_ranks(e0.elapsed_time(e1) / iters) * 1000.0  # us

        r = {}
        for name, fn in (("p2p", lambda: transport.allreduce_p2p(0, rank, peers, n, api.F32, 0, None, sh)),
                         ("p2p_fused_sgd", lambda: transport.allreduce_p2p(0, rank, peers, n, api.F32, 0, upd, sh)),
                         ("nccl", lambda: transport.allreduce_sum(0, rank, buf, 0, sh))):
            us = timed(fn)
            bw = 4 * n * 2 * (world - 1) / world / (us * 1e3)
            r[name] = {"us": round(us, 2), "busbw": round(bw, 1), "frac": round(bw / out["peak"], 4)}
        out["sizes"][f"{mb}MiB"] = r
        del buf, w, m
    return out


# ------------------------------------------------------------------ ours

def main():
    args = parse()
    keyset, mode, outstanding, dtype, bucket_mb, bwd_spec = workload(args)
    keys = load_keys(keyset)
    if args.impl == "reference":
        return reference_main(args, keys, mode, outstanding, dtype, bucket_mb)
    rc = self_launch(args)
    if rc is not None:
        return rc
    rank, local_rank, world = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    ready_ms, bwd_ms, bwd_desc = backward_profile(
        args.backward_ms if args.backward_ms is not None else bwd_spec, keys)
    config = config_dict(args, keys, mode, outstanding, dtype, bucket_mb, world)
    if args.comm is None:  # the fused kernel needs fusion buckets and one communicator stream
        # ConCom keeps NCCL: its concurrent peer-memory kernels (grids capped to
        # co-reside) measured faster at 2 GPUs but slower at 4
        args.comm = "nccl" if (mode == "concom" or not bucket_mb) else "p2p"
    zero_on = args.zero and args.comm == "p2p" and mode == "depcha" and dtype == "fp32" and world > 1

    import torch
    import torch.distributed as dist
    from paper_1802_06949_b200 import api

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    name = [f"collsim_{os.getpid()}_{int(time.time() * 1e6) % 10**9}"]
    if world > 1:
        dist.broadcast_object_list(name, src=0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    dt = {"fp32": api.F32, "bf16": api.BF16}[dtype]
    transport = api.Transport.nccl(name[0], world, rank, local_rank, 120000)
    # every communicator is created at setup, before the first collective
    concom = mode == "concom"
    comms_main = api.create_communicators(transport, outstanding) if concom else []
    comms_e2e = api.create_communicators(transport, outstanding) if (concom and not args.no_extras) else []
    comms_par = api.create_communicators(transport, outstanding) if (concom and args.parity) else []
    sched_outstanding = 4
    comms_sched = (api.create_communicators(transport, sched_outstanding)
                   if (not args.no_extras and not concom) else [])
    engine = api.Engine(args.engine_threads, rank, None, local_rank)
    common = dict(mode=mode, w_dtype=api.F32, g_dtype=dt, comm_dtype=dt,
                  bucket_bytes=int(bucket_mb * 2**20), issue_order=1 if args.issue_order == "descending" else 0,
                  outstanding=outstanding, lr=0.1, rescale=1.0 / (64 * world), momentum=args.momentum,
                  backward_ns=int(bwd_ms * 1e6), comm_priority=-5,
                  p2p={"nccl": 0, "p2p": 1, "nvls": 2}[args.comm], grad_views=args.grad_views,
                  zero=zero_on, order_seed=1 if args.config == "stress" else 0,
                  direct_grads=direct_active(args, mode, bucket_mb, world))
    path = {"collectives": ("identity (1 rank)" if world == 1 else
                            {"nccl": "NCCL" + (f", {outstanding} concurrent communicators" if concom else ""),
                             "p2p": (f"{outstanding} concurrent peer-memory allreduce kernels over NVLink (one per "
                                     "communicator, grids capped to co-reside; rank-order sums) + separate update"
                                     if concom else
                                     "fused allreduce+update kernel over NVLink peer memory (rank-order sums)"),
                             "nvls": "fused allreduce+update kernel, NVSwitch multicast in-switch reduction"}[args.comm]),
            "optimizer_state": ("ZeRO-1: master weights + momentum sharded 1/N, weights all-gathered in the "
                                "fused kernel" if zero_on else "replicated on every rank")}
    model = api.SynthModel(engine, transport, rank, world, keys, concom_comms=comms_main, ready_ms=ready_ms,
                           **common)
    model.init()
    info = model.info()
    gbytes = info["grad_bytes"]
    COMM = api.SynthModel.COMM
    BWD = api.SynthModel.BACKWARD
    LOCAL = api.SynthModel.LOCAL_UPDATE

    # ---- headline: aggregation steps, gradients resident in HBM
    model.run(1, BWD | COMM)  # the gradients hold this rank's values (synthetic backward once)
    model.run(max(0, args.warmup - 1), COMM)
    barrier()
    api.host_profile(reset=True)
    l0 = api.launch_count()
    with Clocks(",".join(str(d) for d in range(world)) if world > 1 else str(local_rank),
                enabled=(rank == 0)) as clk:
        clk.wait_first()
        clk.wait_first()  # aligned to the sampler's period, not its start-up
        barrier()
        ms = model.run(args.steps, COMM)
        launches = api.launch_count() - l0
        host_ms = model.last_host_ms()
        if os.environ.get("CSB_HOST_PROFILE") == "1":
            print(json.dumps({"host_profile_per_step": {k: round(v["us"] / args.steps, 2)
                                                        for k, v in api.host_profile().items()}}),
                  file=sys.stderr)
        # the timed region is short; keep the same steps running ~0.5 s so
        # the sampler sees the clocks under this exact load
        t_end = time.time() + 0.5
        while time.time() < t_end:
            model.run(args.steps, COMM)
    barrier()
    ms = max_over_ranks(ms)
    step_ms = ms / args.steps
    per_gpu = gbytes / (step_ms * 1e6)
    line = {"metric": METRIC, "value": round(per_gpu, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype.replace("fp", "f"),
            "data": "synthetic (random_uniform seeds 1000+r*K+k; torchvision key sizes)",
            "config": config, "whole_job_gbs": round(world * per_gpu, 3), "grad_bytes_per_rank": gbytes,
            "path": path, "buckets": info["num_buckets"], "gpu_launches": launches,
            "host_dispatch_ms_per_step": round(host_ms / args.steps, 4),
            "clocks": {**clk.summary(), "window": "timed region + 0.5 s of the same steps"}}

    if not args.no_extras:
        # ---- exposed communication under the synthetic backward
        # three alternating rounds, the fastest of each: both sides see the
        # same clocks / neighbours, and one disturbed round does not set the sign
        n_exp = max(3, min(args.steps, 10))
        fulls, comps = [], []
        for _ in range(3):
            model.run(1, BWD | COMM)
            barrier()
            fulls.append(max_over_ranks(model.run(n_exp, BWD | COMM)) / n_exp)
            barrier()
            model.run(1, BWD | LOCAL)
            barrier()
            comps.append(max_over_ranks(model.run(n_exp, BWD | LOCAL)) / n_exp)
            barrier()
        t_full, t_comp = min(fulls), min(comps)
        line["exposed_comm_ms"] = round(t_full - t_comp, 4)
        line["step_with_backward_ms"] = round(t_full, 4)
        line["backward_plus_update_ms"] = round(t_comp, 4)
        line["exposed_frac"] = round((t_full - t_comp) / t_full, 4) if t_full > 0 else None
        line["synthetic_backward_ms"] = round(bwd_ms, 3)
        line["synthetic_backward"] = bwd_desc

        # ---- roofline of the dominant kernel (CUDA events on the launch stream)
        api.profile_reset()
        api.profile_enable(True)
        n_prof = max(3, min(args.steps, 10))
        model.run(n_prof, COMM)
        api.profile_enable(False)
        kstats = {k: api.profile_collect(k) for k in ("pack", "sum", "sgd", "pack_sgd")}
        dom = max(kstats, key=lambda k: kstats[k]["total_ms"])
        ks = kstats[dom]
        pk = peaks()
        if world > 1 and args.comm in ("p2p", "nvls") and dom == "sum":
            # the fused allreduce+update kernel is NVLink-bound: algorithmic
            # bytes crossing the link per GPU per direction, per step
            # peer loads: (N-1)/N of the gradients in the reduce-scatter, plus
            # (N-1)/N of the reduced gradients (replicated update) or of the
            # fp32 master weights (ZeRO-1 all-gather); NVLS: 1 x bucket bytes
            second = sum(keys) * 4 if zero_on else gbytes
            link_step = ((world - 1) / world * (gbytes + second) if args.comm == "p2p" else gbytes)
            bytes_launch = link_step * n_prof / max(1, ks["launches"])
            bound, peak = "nvlink", pk.get("nvlink_gbs_per_dir", 770.0)
            peak_source = ("MEASURED_PEAKS.json nvlink_gbs_per_dir" if "nvlink_gbs_per_dir" in pk else
                           "B200_PROFILING.md measured peer copy, 770 GB/s per direction")
        else:
            bytes_launch = ks["bytes"] / max(1, ks["launches"])
            bound, peak = "hbm", pk.get("hbm_gbs", 6650.0)
            peak_source = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"
        avg_s = ks["total_ms"] / max(1, ks["launches"]) / 1e3
        achieved = bytes_launch / avg_s / 1e9 if avg_s > 0 else 0.0
        traffic = (ncu_traffic(f"{dom}_tab_kernel") if (bound == "hbm" and args.config == "resnet50"
                                                       and bucket_mb == 100 and world == 1) else None)
        if bound == "nvlink":
            # 770 is the one-way peer copy; an allreduce loads every link both
            # ways, where tools/nvlink_probe.cu measures this pool's ceiling
            ceil = {2: 692.5, 4: 581.2}.get(world)
            ceiling = ({"gbs": ceil, "frac": round(achieved / ceil, 4),
                        "source": f"profiles/r2_nvlink_probe_n{world}.txt: best all-to-all pattern "
                                  "(copy engines, every GPU sending and receiving)"} if ceil else None)
        line["roofline"] = {"bound": bound, "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                            "unit": "GB/s", "frac": round(achieved / peak, 4),
                            "traffic": traffic["bytes"] if traffic else None,
                            "traffic_source": traffic["source"] if traffic else None,
                            "launches": ks["launches"],
                            "avg_launch_us": round(1000 * ks["total_ms"] / max(1, ks["launches"]), 2),
                            "bytes_per_launch": round(bytes_launch),
                            "peak_source": peak_source,
                            **({"all_to_all_ceiling": ceiling} if bound == "nvlink" else {}),
                            "kernels": {k: {"launches": v["launches"],
                                            "ms_per_step": round(v["total_ms"] / n_prof, 4),
                                            "GBps": round(v["bytes"] / (v["total_ms"] * 1e6), 1) if v["total_ms"] else None}
                                        for k, v in kstats.items()}}

        # ---- the paper's three schedules on the same gradient set
        scheds = {mode: {"value": line["value"], "ms_per_step": line["ms_per_step"],
                         "collectives": path["collectives"]}}
        for sched in ("funnel", "depcha", "concom"):
            if sched in scheds:
                continue
            if sched == "concom":
                if not comms_sched:
                    continue
                kw = {**common, "mode": "concom", "outstanding": sched_outstanding, "zero": False, "p2p": 0,
                      "bucket_bytes": 25 << 20, "direct_grads": False}
                coll = (f"NCCL, {sched_outstanding} communicators, 25 MiB buckets" if world > 1 else
                        f"identity (1 rank), {sched_outstanding} communicators, 25 MiB buckets")
                cc = comms_sched
            else:
                kw = {**common, "mode": sched, "zero": common["zero"] and sched == "depcha"}
                coll = path["collectives"]
                cc = []
            ms_s = api.SynthModel(engine, transport, rank, world, keys, concom_comms=cc, **kw)
            ms_s.init()
            ms_s.run(args.warmup, COMM)
            barrier()
            t_s = max_over_ranks(ms_s.run(args.steps, COMM)) / args.steps
            scheds[sched] = {"value": round(gbytes / (t_s * 1e6), 3), "ms_per_step": round(t_s, 4),
                             "collectives": coll}
            ms_s.close()
        line["schedules"] = scheds

        # ---- allreduce bus bandwidth per bucket size (N>1)
        if world > 1:
            line["allreduce_busbw"] = busbw_sweep(api, transport, rank, world, max_over_ranks)

        # ---- the same aggregation with gradient-as-bucket-view (no pack copy)
        if not args.grad_views and bucket_mb > 0:
            model_v = api.SynthModel(engine, transport, rank, world, keys, concom_comms=comms_main,
                                     **{**common, "grad_views": True})
            model_v.init()
            model_v.run(args.warmup, COMM)
            barrier()
            ms_v = max_over_ranks(model_v.run(args.steps, COMM)) / args.steps
            line["grad_views"] = {"value": round(gbytes / (ms_v * 1e6), 3), "unit": "GB/s",
                                  "ms_per_step": round(ms_v, 4),
                                  "note": "gradients produced in place in the comm buckets (DDP "
                                          "gradient_as_bucket_view): push copies nothing; same collective "
                                          "and fused update"}
            model_v.close()

        # ---- the reference's own arithmetic: fp64 weights + gradients, plain SGD
        if dtype == "fp32" and not concom:
            kw64 = {**common, "w_dtype": api.F64, "g_dtype": api.F64, "comm_dtype": api.F64, "momentum": 0.0,
                    "grad_views": False, "backward_ns": 0}
            m64 = api.SynthModel(engine, transport, rank, world, keys, **kw64)
            m64.init()
            m64.run(1, BWD | COMM)
            m64.run(max(0, args.warmup - 1), COMM)
            barrier()
            t64 = max_over_ranks(m64.run(args.steps, COMM)) / args.steps
            m64.close()
            g64 = sum(keys) * 8
            line["f64"] = {"value": round(g64 / (t64 * 1e6), 3), "unit": "GB/s", "ms_per_step": round(t64, 4),
                           "value_same_basis_as_headline": round(gbytes / (t64 * 1e6), 3),
                           "note": "fp64 weights and gradients, plain SGD (momentum 0): the reference's own "
                                   "arithmetic (model.cpp:17-27), directly comparable to the --impl reference "
                                   "line; value counts fp64 bytes, value_same_basis_as_headline the headline's"}
            if args.parity:
                line["f64"]["parity"] = parity_check(api, engine, transport, rank, world, keys, kw64, [], api.F64,
                                                     args.parity_steps, barrier, dist)

        # ---- end to end through the C ABI with host buffers
        model_e2e = api.SynthModel(engine, transport, rank, world, keys, concom_comms=comms_e2e,
                                   host_source=True, **{**common, "backward_ns": 0})
        model_e2e.init()
        model_e2e.run_e2e(2, BWD | COMM)
        barrier()
        wall = max_over_ranks(model_e2e.run_e2e(args.steps, BWD | COMM))
        e2e_step = wall / args.steps
        line["e2e"] = {"value": round(gbytes / (e2e_step * 1e6), 3), "unit": "GB/s",
                       "h2d_bytes_per_step": model_e2e.info()["h2d_bytes_per_step"], "d2h_bytes_per_step": 8,
                       "ms_per_step": round(e2e_step, 4),
                       "note": "wall clock through the C ABI: per step one pinned-host H2D of the gradients, "
                               "the step, a weight checksum read back D2H; the host reads step i's result "
                               "after queueing step i+1"}
        model_e2e.close()

        # ---- CPU baseline: the reference on this host, bounded sample
        if world == 1 and rank == 0:
            try:
                ref = run_reference(keys, mode, outstanding, 1, 1, args.cpu_steps, ELEM[dtype])
            except Exception as e:  # reported, not fatal
                ref = None
                line["cpu_baseline"] = {"error": str(e)}
            if ref:
                line["cpu_baseline"] = {
                    "value": round(ref["per_gpu"], 4), "unit": "GB/s", "cores": ref["cores"], "kind": "reference",
                    "sample": f"{len(keys)} keys fp64, 1 rank thread x {ref['threads']} engine threads, "
                              f"{args.cpu_steps} steps after 1 warm-up (oracle/_ref = unmodified reference)",
                    "ms_per_step": round(ref["ms_per_step"], 2)}
    model.close()

    # ---- parity of the benchmarked config (after every timed region)
    if args.parity:
        line["parity"] = parity_check(api, engine, transport, rank, world, keys, common, comms_par, dt,
                                      args.parity_steps, barrier, dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier()
    engine.close()
    transport.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
