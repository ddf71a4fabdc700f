"""Real-backward producer: data-parallel training of a torch.nn.Module through
the KvStore hot path.

The reference's producer is its own toy model: `push_forward_backward`
(R/core/src/trainer.cpp:36-72) pushes each parameter's gradient op into the
engine and `train_epoch` (trainer.cpp:112-141) pushes / pulls per key.  Here
the producer is PyTorch autograd on its own CUDA stream:

* every parameter is a key (``model.parameters()`` order, like the
  reference's key = layer index); the gradients live in one flat arena with
  256-B aligned slots so their device pointers never change -- or, with
  ``bucket_views=True``, directly in the KvStore's comm buckets
  (gradient-as-bucket-view: push copies nothing).  After step() the view
  buffers are NOT this rank's gradient and, at world > 1, not the full sum
  either: the fused peer kernel keeps only this rank's shard of the sum in
  the bucket (shard_only; the rest still holds this rank's own gradient), and
  with ``zero=True`` no sum at all (the reduction stays in registers).  Code
  that reads p.grad after step() (clipping, logging) must read it before
  step() or run with ``p2p=0``.  The arena is registered (``direct_grads``,
  KvStore.register_grads; at world > 1 with the peer-memory kernel): the
  fused kernels read the gradients in place, so push stages nothing;
* a post-accumulate-grad hook counts ready gradients per fusion bucket; when a
  bucket is complete it records a CUDA event on the autograd stream,
  ``Engine.import_event`` turns it into the latest write of the gradients
  (and of the weights, which the rest of the backward no longer reads), and the
  bucket's keys are pushed (DepCha: packed as soon as they exist, while the
  rest of the backward still runs);
* ``step()`` (after ``loss.backward()``) pulls every key with the fused SGD /
  momentum update (``KvStore.pull_update``) and makes the framework stream
  wait for the engine (``Engine.stream_wait``), so the next forward sees the
  new weights without a host synchronisation.

Everything on the data path runs in libcollsim_b200.so; this module only
wires autograd to the C ABI.
"""
from __future__ import annotations

from typing import Sequence

import torch

from . import api
from ._lib import UsageError

_ALIGN = 256  # bytes: every gradient slot starts on a 16-B vector boundary (kvstore.cpp bucket rule)


class TorchKvStoreDP:
    """One rank of data-parallel SGD through the KvStore.

    ``rescale`` multiplies the aggregated (summed) gradient, e.g. 1/world for
    a mean over ranks of per-rank mean losses (the reference passes
    1/global_batch, trainer.cpp:96).
    """

    def __init__(self, model: torch.nn.Module, engine: api.Engine, transport: api.Transport, rank: int,
                 world: int, *, mode: str = "depcha", lr: float = 0.1, momentum: float = 0.0,
                 rescale: float | None = None, bucket_mb: float = 25.0, p2p: int = 1, outstanding: int = 1,
                 concom_comms: Sequence[int] = (), comm_dtype: int = -1, bucket_views: bool = False,
                 zero: bool = False, direct_grads: bool = True):
        if mode not in ("depcha", "funnel"):
            raise ValueError("TorchKvStoreDP drives the DepCha / Funnel schedules (push during backward, "
                             "pull after it)")
        self.model = model
        self.engine = engine
        self.rank, self.world = rank, world
        self.lr, self.momentum = lr, momentum
        self.rescale = (1.0 / world) if rescale is None else rescale
        self.params = [p for p in model.parameters() if p.requires_grad]
        if not self.params:
            raise ValueError("model has no trainable parameters")
        dev = self.params[0].device
        if dev.type != "cuda" or any(p.device != dev for p in self.params):
            raise ValueError("every parameter must live on the same CUDA device")
        dt = self.params[0].dtype
        if any(p.dtype != dt for p in self.params):
            raise ValueError("parameters must share one dtype")
        K = len(self.params)

        if bucket_views and (bucket_mb <= 0 or comm_dtype not in (-1, api.dtype_code(dt))):
            raise ValueError("bucket views need fusion buckets and comm dtype == parameter dtype")
        esz = torch.tensor([], dtype=dt).element_size()
        if not bucket_views:
            # flat gradient arena: stable pointers, one memset to zero
            offs, off = [], 0
            for p in self.params:
                offs.append(off)
                off += (p.numel() * esz + _ALIGN - 1) // _ALIGN * _ALIGN // esz
            self.grad_arena = torch.zeros(max(off, 1), dtype=dt, device=dev)
            for p, o in zip(self.params, offs):
                p.grad = self.grad_arena[o:o + p.numel()].view_as(p)

        self.w_slots = [api.Slot(p.data, engine.new_variable()) for p in self.params]
        cfg = api.KvConfig(mode, outstanding, K, comm_dtype=comm_dtype,
                           bucket_bytes=int(bucket_mb * 2**20), issue_order=1, comm_priority=-5,
                           p2p=p2p if world > 1 else 0, zero=int(zero and world > 1))
        self.kv = api.KvStore(engine, transport, rank, cfg, concom_comms)
        torch.cuda.synchronize(dev)  # the weights were written on the framework stream
        for k in range(K):
            self.kv.init(k, self.w_slots[k])  # rank 0's weights broadcast (kvstore.cpp:95)
        if direct_grads and not bucket_views and (world == 1 or p2p == 1):
            # the flat arena is registered (a setup collective): the fused
            # kernels read the gradients in place (every rank's over NVLink at
            # world > 1), nothing is staged into the comm buckets
            self.kv.register_grads(self.grad_arena.data_ptr(), self.grad_arena.numel() * esz)
        # gradient-ready groups = fusion buckets (built here, identically on every rank)
        groups: dict[int, list[int]] = {}
        for k in range(K):
            groups.setdefault(self.kv.key_map(k)[0], []).append(k)
        if bucket_views:
            # DDP's gradient_as_bucket_view: autograd accumulates straight into
            # the comm buckets, so push copies nothing
            base, nbytes = self.kv.arena()
            self.grad_arena = api.device_tensor(base, nbytes // esz, api.dtype_code(dt), dev.index)
            self.grad_arena.zero_()
            for k, p in enumerate(self.params):
                p.grad = self.kv.bucket_view_tensor(k, p.numel(), api.dtype_code(dt), dev.index).view_as(p)
        self.g_slots = [api.Slot(p.grad, engine.new_variable()) for p in self.params]
        self.bucket_of = [0] * K
        self.groups = list(groups.values())
        for gi, keys in enumerate(self.groups):
            for k in keys:
                self.bucket_of[k] = gi
        self._ready = [0] * len(self.groups)
        self._events: list[torch.cuda.Event] = []
        self._pushed = 0
        self._hooks = [p.register_post_accumulate_grad_hook(self._hook(k)) for k, p in enumerate(self.params)]
        all_tags = [s.tag for s in self.w_slots] + [s.tag for s in self.g_slots]
        self._all_tags = all_tags
        # the framework stream must see the broadcast weights before the first forward
        engine.stream_wait(all_tags, torch.cuda.current_stream(dev).cuda_stream)

    def _hook(self, k: int):
        def fn(_p):
            b = self.bucket_of[k]
            self._ready[b] += 1
            if self._ready[b] == len(self.groups[b]):
                keys = self.groups[b]
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream())
                self._events.append(ev)
                # the event also releases the bucket's weights: the backward
                # reads a parameter only in its own node, which precedes its
                # AccumulateGrad (tied parameters accumulate once, after all uses)
                self.engine.import_event(ev.cuda_event, [self.g_slots[j].tag for j in keys] +
                                         [self.w_slots[j].tag for j in keys], key=keys[0])
                self.kv.push(keys, [self.g_slots[j] for j in keys])
                self._pushed += 1
        return fn

    def zero_grad(self) -> None:
        """Zero every gradient with one memset on the framework stream (ordered
        after the engine's reads by the previous step's stream_wait)."""
        self.grad_arena.zero_()

    def step(self) -> None:
        """After loss.backward(): fused aggregation + SGD for every key, then
        the framework stream waits for the new weights."""
        if self._pushed != len(self.groups):
            raise UsageError(-2, f"step(): {self._pushed} of {len(self.groups)} gradient buckets were "
                                     "pushed (did every parameter receive a gradient?)")
        K = len(self.params)
        self.kv.pull_update(list(range(K)), self.w_slots, self.lr, self.rescale, self.momentum)
        self.engine.stream_wait(self._all_tags, torch.cuda.current_stream().cuda_stream)
        self._ready = [0] * len(self.groups)
        self._events.clear()
        self._pushed = 0

    def close(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []
        self.engine.wait_all()
        self.kv.close()
