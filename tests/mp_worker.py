"""One rank of a multi-process (one process per GPU) scenario over the NCCL
transport; launched by tests/test_nccl_multigpu.py through torchrun.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/mp_worker.py <case> <outdir>

run_colocated() runs the same cases as rank THREADS on one GPU over a local
peer transport (tests/test_peer_local_gpu.py): the fused peer-memory kernels
then run on plain device pointers instead of CUDA-IPC-mapped peers.

Writes <outdir>/<case>_r<rank>.npz / .json; the test compares them with the
oracle and the golden fixtures.  torch.distributed (gloo) is plumbing only:
it passes the ledger name and joins the ranks at the end.
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import _oracle as O  # noqa: E402
from paper_1802_06949_b200 import (DeadlockTimeout, Engine, KvConfig, KvStore, MismatchError,  # noqa: E402
                                   Slot, TraceSink, Transport, api, create_communicators)


def t64(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def run_rank(case, rank, world, tr, dev, outdir, sink, colocated=False, shared_comms=None):
    """One rank of `case` on transport `tr` (NCCL across processes, or a local
    peer transport shared by rank threads on one GPU when colocated).  Writes
    the rank's .npz; returns the rank's JSON record."""
    local = dev.index
    out = {}

    if case == "allreduce":
        # acceptance criterion 1 inputs (acceptance.cpp:42-84), fp64
        eng = Engine(2, rank, None, local)
        s = eng.lane_stream(0)
        res = []
        for i in range(100):
            n = 1 + (i * 7) % 64
            b = t64(O.random_uniform(n, O.mix_seed(world * 1000 + i, rank)), dev)
            tr.allreduce_sum(0, rank, b, i, s)
            res.append(b)
        torch.cuda.synchronize(dev)
        eng.wait_all()
        np.savez(outdir / f"{case}_r{rank}.npz", *[x.cpu().numpy() for x in res])
        eng.close()
    elif case.split("_")[0] in ("funnel", "depcha", "concom"):
        mode = case.split("_")[0]
        split = case.endswith("_p2psplit")  # one pull_update per key: buckets not whole
        zero = case.endswith("_p2pzero")  # ZeRO-1: sharded master weights + all-gather
        p2p = case.endswith("_p2p") or split or zero
        gold = np.load(HERE / "golden" / "train_steps.npz")
        sizes = [int(x) for x in gold["sizes"]]
        K, lr, rescale = len(sizes), float(gold["lr"]), 1.0 / (64 * world)
        outstanding = 2 if mode == "concom" else 1
        # colocated rank threads share ONE transport: its communicators are
        # created once for all of them (run_colocated), not once per rank
        comms = ((shared_comms if shared_comms is not None else create_communicators(tr, outstanding))
                 if mode == "concom" else [])
        eng = Engine(4, rank, sink, local)
        cfg = KvConfig(mode, outstanding, K, bucket_bytes=16 * 1024 if p2p else 0, p2p=int(p2p), zero=int(zero))
        store = KvStore(eng, tr, rank, cfg, comms)
        case_mode = mode
        ws = [Slot(t64(O.random_uniform(n, O.mix_seed(7, k)) if rank == 0 else np.zeros(n), dev),
                   eng.new_variable()) for k, n in enumerate(sizes)]
        gs = [Slot(t64(O.random_uniform(n, 1000 + rank * K + k), dev), eng.new_variable())
              for k, n in enumerate(sizes)]
        for k in range(K):
            store.init(k, ws[k])
        eng.wait_all()
        src = [g.value.clone() for g in gs]
        for _ in range(3):
            for k in reversed(range(K)):
                sp, dp, n = src[k].data_ptr(), gs[k].value.data_ptr(), sizes[k]
                eng.push_stream(lambda st, sp=sp, dp=dp, n=n: api.synth_backward(sp, dp, n, api.F64, 0, 0, st),
                                [], [gs[k].tag], api.COMPUTE, k)
            if case_mode == "depcha" and split:
                store.push(list(range(K)), gs)
                for k in range(K):
                    store.pull_update(k, ws[k], lr, rescale)
            elif case_mode == "depcha":
                store.push(list(range(K)), gs)
                store.pull_update(list(range(K)), ws, lr, rescale)
            else:
                since = 0
                groups = {}
                for k in range(K):  # one push / pull per fusion bucket (1:1 without buckets)
                    groups.setdefault(store.key_map(k)[0], []).append(k)
                for b in sorted(groups):
                    keys = groups[b]
                    store.push(keys, [gs[k] for k in keys])
                    store.pull_update(keys, [ws[k] for k in keys], lr, rescale)
                    if case_mode == "concom":
                        since += 1
                        if since == outstanding:
                            store.barrier()
                            since = 0
                if case_mode == "concom" and since:
                    store.barrier()
            eng.wait_all()
        np.savez(outdir / f"{case}_r{rank}.npz", *[w.value.cpu().numpy() for w in ws])
        store.close()
        eng.close()
    elif case == "p2p_api":
        # cs_allreduce_p2p directly: reduce only, fused update keeping the
        # whole sum, fused update keeping only the own shard (shard_only)
        n = 4 << 20  # 16 MiB fp32: its own allocator segment, so the IPC base is the tensor
        eng = Engine(1, rank, None, local)
        s = eng.lane_stream(0)
        g = torch.from_numpy(O.random_uniform(n, 1000 + rank).astype(np.float32)).to(dev)
        w0 = torch.from_numpy(O.random_uniform(n, O.mix_seed(7, 0)).astype(np.float32)).to(dev)
        buf = torch.empty(n, dtype=torch.float32, device=dev)
        peers = tr.share_buffer(buf.data_ptr(), rank)
        res = {}
        buf.copy_(g)
        torch.cuda.synchronize(dev)
        tr.allreduce_p2p(0, rank, peers, n, api.F32, 0, None, s)
        torch.cuda.synchronize(dev)
        res["sum"] = buf.cpu().numpy()
        for so in (0, 1):
            buf.copy_(g)
            w = w0.clone()
            m = torch.zeros(n, dtype=torch.float32, device=dev)
            torch.cuda.synchronize(dev)
            ents = [(w.data_ptr(), buf.data_ptr(), m.data_ptr(), n)]
            tr.allreduce_p2p(0, rank, peers, n, api.F32, 1, (ents, api.F32, 0.1, 1.0 / 64, 0.9, so), s)
            torch.cuda.synchronize(dev)
            res[f"w{so}"], res[f"m{so}"], res[f"buf{so}"] = w.cpu().numpy(), m.cpu().numpy(), buf.cpu().numpy()
        np.savez(outdir / f"{case}_r{rank}.npz", **res)
        eng.close()
    elif case == "stress_order":
        # deadlock stress (scaled): every rank produces
        # its gradients in its own random order; the schedules must still
        # issue one collective sequence, and the weights cannot depend on it
        from paper_1802_06949_b200 import keysets
        sizes = [min(n, 1 << 16) for n in keysets.stress_keys(96)]
        out["sums"] = {}
        for mode, p2p, zero in (("depcha", 1, 1), ("depcha", 1, 0), ("funnel", 1, 0), ("depcha", 0, 0)):  # noqa
            for seed in (0, 11):
                eng = Engine(4, rank, None, local)
                m = api.SynthModel(eng, tr, rank, world, sizes, mode=mode, bucket_bytes=(256 * 1024 if p2p else 0),
                                   issue_order=1, lr=0.1, rescale=1.0 / 64, momentum=0.9, backward_ns=int(2e6),
                                   p2p=p2p, zero=bool(zero), order_seed=seed)
                m.init()
                m.run(3, m.BACKWARD | m.COMM)
                out["sums"][f"{mode}_p{p2p}_z{zero}_s{seed}"] = m.checksum()
                m.close()
                eng.close()
    elif case == "zero_vs_replicated":
        # the same fp32 weights / bf16 comm / momentum run through the fused
        # kernel with a replicated update and with ZeRO-1: identical weights
        sizes = [1, 7, 64, 300, 4097, 70000, 1 << 18]
        K = len(sizes)
        f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)  # noqa: E731
        res = {}
        for zero in (0, 1):
            for cdt in (api.F32, api.BF16):
                eng = Engine(4, rank, None, local)
                store = KvStore(eng, tr, rank, KvConfig("depcha", 1, K, comm_dtype=cdt, bucket_bytes=256 * 1024,
                                                        issue_order=1, p2p=1, zero=zero))
                ws = [Slot(f32(O.random_uniform(n, O.mix_seed(7, k)) if rank == 0 else np.zeros(n)),
                           eng.new_variable()) for k, n in enumerate(sizes)]
                gs = [Slot(f32(O.random_uniform(n, 1000 + rank * K + k)), eng.new_variable())
                      for k, n in enumerate(sizes)]
                for k in range(K):
                    store.init(k, ws[k])
                eng.wait_all()
                for _ in range(3):
                    store.push(list(range(K)), gs)
                    store.pull_update(list(range(K)), ws, 0.1, 1.0 / 64, 0.9)
                eng.wait_all()
                for k in range(K):
                    res[f"z{zero}_c{cdt}_k{k}"] = ws[k].value.cpu().numpy()
                store.close()
                eng.close()
        np.savez(outdir / f"{case}_r{rank}.npz", **res)
    elif case in ("direct", "direct_mismatch"):
        # gradients in one registered region (KvStore.register_grads): the
        # fused peer kernels read every rank's gradients in place instead of
        # staging them; weights must equal the staged run's bit for bit.
        # direct_mismatch: each rank lays its keys out at rank-dependent
        # offsets -> MismatchError before any launch (layout in the signature)
        sizes = [1, 7, 64, 300, 4097, 70000, 1 << 18]
        K = len(sizes)
        res = {}
        variants = ([("depcha", z, g, d) for z in (0, 1) for g in (api.F32, api.BF16) for d in (0, 1)] +
                    [("funnel", 0, g, d) for g in (api.F32, api.BF16) for d in (0, 1)]
                    if case == "direct" else [("depcha", 1, api.F32, 1)])
        for mode, zero, gdt, direct in variants:
            tdt, esz = (torch.float32, 4) if gdt == api.F32 else (torch.bfloat16, 2)
            shift = 256 * rank if case == "direct_mismatch" else 0
            offs, o = [], shift
            for n in sizes:
                offs.append(o)
                o += (n * esz + 255) // 256 * 256
            garena = torch.zeros(o, dtype=torch.uint8, device=dev)
            eng = Engine(4, rank, None, local)
            store = KvStore(eng, tr, rank, KvConfig(mode, 1, K, comm_dtype=gdt, bucket_bytes=256 * 1024,
                                                    issue_order=1, p2p=1, zero=zero))
            ws = [Slot(torch.from_numpy(np.ascontiguousarray(
                O.random_uniform(n, O.mix_seed(7, k)) if rank == 0 else np.zeros(n), dtype=np.float32)).to(dev),
                eng.new_variable()) for k, n in enumerate(sizes)]
            gs = []
            for k, n in enumerate(sizes):
                g = garena[offs[k]:offs[k] + n * esz].view(tdt)
                g.copy_(torch.from_numpy(O.random_uniform(n, 1000 + rank * K + k)).to(dev).to(tdt))
                gs.append(Slot(g, eng.new_variable()))
            for k in range(K):
                store.init(k, ws[k])
            eng.wait_all()
            if direct:
                store.register_grads(garena.data_ptr(), garena.numel())
            try:
                for _ in range(3):
                    store.push(list(range(K)), gs)
                    store.pull_update(list(range(K)), ws, 0.1, 1.0 / 64, 0.9)
                eng.wait_all()
                out["error"] = None
            except MismatchError as e:
                out["error"] = type(e).__name__ + ": " + str(e)
            if out.get("error") is None:
                tag = "" if mode == "depcha" else "f"
                for k in range(K):
                    res[f"{tag}z{zero}_g{gdt}_d{direct}_k{k}"] = ws[k].value.cpu().numpy()
            store.close()
            eng.close()
        np.savez(outdir / f"{case}_r{rank}.npz", **res)
    elif case in ("torch_dp", "torch_dp_zero"):
        # real-backward producer over the fused NVLink kernel: save every
        # rank's per-step gradients and weights; the test replays the oracle
        from paper_1802_06949_b200.torch_dp import TorchKvStoreDP
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).to(dev)
        eng = Engine(4, rank, sink, local)
        dp = TorchKvStoreDP(model, eng, tr, rank, world, lr=0.05, momentum=0.9, bucket_mb=0.05, p2p=1,
                            zero=case == "torch_dp_zero")
        flat = lambda ts: np.concatenate([t.detach().cpu().numpy().ravel() for t in ts])  # noqa: E731
        res = {"w0": flat(dp.params), "buckets": np.array(len(dp.groups))}
        gen = torch.Generator(device=dev).manual_seed(100 + rank)
        for step in range(3):
            x = torch.randn(16, 64, device=dev, generator=gen)
            y = torch.randint(0, 10, (16,), device=dev, generator=gen)
            dp.zero_grad()
            torch.nn.functional.cross_entropy(model(x), y).backward()
            dp.step()
            torch.cuda.synchronize(dev)
            res[f"g{step}"] = flat([p.grad for p in dp.params])
            res[f"w{step + 1}"] = flat(dp.params)
        np.savez(outdir / f"{case}_r{rank}.npz", **res)
        dp.close()
        eng.close()
    elif case == "nvls":
        # fp32 DepCha over NVSwitch multicast (in-switch reduction): the test
        # compares with the fp64 oracle of the fp32-rounded inputs
        sizes = [1, 7, 64, 300, 4097, 70000]
        K = len(sizes)
        eng = Engine(4, rank, sink, local)
        store = KvStore(eng, tr, rank, KvConfig("depcha", 1, K, bucket_bytes=64 * 1024, p2p=2))
        f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)  # noqa: E731
        ws = [Slot(f32(O.random_uniform(n, O.mix_seed(7, k)) if rank == 0 else np.zeros(n)), eng.new_variable())
              for k, n in enumerate(sizes)]
        gs = [Slot(f32(O.random_uniform(n, 1000 + rank * K + k)), eng.new_variable()) for k, n in enumerate(sizes)]
        for k in range(K):
            store.init(k, ws[k])
        eng.wait_all()
        store.push(list(range(K)), gs)
        store.pull_update(list(range(K)), ws, 0.1, 1.0 / 64, 0.9)
        eng.wait_all()
        out["nvls_active"] = bool(tr.p2p_capable())
        np.savez(outdir / f"{case}_r{rank}.npz", *[w.value.cpu().numpy() for w in ws])
        store.close()
        eng.close()
    elif case == "mismatch":
        eng = Engine(1, rank, None, local)
        b = torch.zeros(4 if rank == 0 else 6, dtype=torch.float64, device=dev)
        try:
            tr.allreduce_sum(0, rank, b, 0, eng.lane_stream(0))
            out["error"] = None
        except MismatchError as e:
            out["error"] = "MismatchError"
            out["message"] = str(e)
        eng.close()
    elif case == "deadlock":
        eng = Engine(1, rank, None, local)
        b = torch.zeros(4, dtype=torch.float64, device=dev)
        try:
            if rank == 0:
                tr.allreduce_sum(0, rank, b, 0, eng.lane_stream(0))
            else:
                time.sleep(5)  # never issues its call
            out["error"] = None
        except DeadlockTimeout as e:
            out["error"] = "DeadlockTimeout"
            out["message"] = str(e)
        eng.close()
    else:
        raise SystemExit(f"unknown case {case}")

    if case.split("_")[0] in ("funnel", "depcha", "concom"):
        out["trace"] = [f"{e['kind']}:{e['comm']}:{e['seq']}:{e.get('key', -1)}"
                        for e in sink.snapshot()
                        if e["event"] == "coll_enqueued" and (not colocated or e.get("rank") == rank)]
    (outdir / f"{case}_r{rank}.json").write_text(json.dumps(out))
    return out


def main():
    case, outdir = sys.argv[1], Path(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    name = [f"csb_test_{os.getpid()}_{time.time_ns() % 10**9}"]
    dist.broadcast_object_list(name, src=0)
    sink = TraceSink()
    watchdog = 3000 if case in ("mismatch", "deadlock") else 60000
    tr = Transport.nccl(name[0], world, rank, local, watchdog, sink)
    run_rank(case, rank, world, tr, dev, outdir, sink)
    dist.barrier()
    tr.close()
    dist.destroy_process_group()


def run_colocated(case, world, outdir, watchdog_ms=60000):
    """The same case with `world` rank THREADS on cuda:0 over a local peer
    transport: every cross-GPU kernel (fused allreduce+update, ZeRO-1, the
    pair barriers and epochs) runs on one device, grids capped to co-reside.
    Returns the per-rank JSON records."""
    import threading
    sink = TraceSink()
    tr = Transport.local(world, watchdog_ms, sink, peer=True)
    assert tr.p2p_capable()
    outs, errs = [None] * world, []
    dev = torch.device("cuda", 0)
    shared_comms = create_communicators(tr, 2) if case.split("_")[0] == "concom" else None

    def body(r):
        try:
            torch.cuda.set_device(0)
            # every rank thread on its own framework stream: a rank's torch work
            # must never queue behind another rank's wait on a peer kernel
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                outs[r] = run_rank(case, r, world, tr, dev, outdir, sink, colocated=True, shared_comms=shared_comms)
        except BaseException as e:  # re-raised on the caller's thread
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    tr.close()
    if errs:
        raise errs[0]
    return outs


if __name__ == "__main__":
    main()
