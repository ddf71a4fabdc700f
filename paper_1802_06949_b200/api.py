"""Python mirror of the reference API over the C ABI.

Names, argument meaning and error behaviour follow collsim
(R/core/include/collsim/{engine,collective,kvstore,trace}.hpp) so the tests
read like the reference's own tests:

    Engine(num_worker_threads, rank=0, trace=None, device=-1)
        .new_variable() / .push(body, reads, mutates, kind, key) / .wait_for(tag)
        .wait_all() / .shutdown()
    Transport.local(num_ranks, watchdog_ms, trace)      in-process ranks, kernel (b)
    Transport.nccl(name, num_ranks, rank, device, ...)  one process per GPU
        .allreduce_sum(comm, rank, buf, key, stream) / .broadcast / .barrier
    KvStore(engine, transport, rank, KvConfig, concom_comms)
        .init(key, slot) / .push(keys, slots) / .pull(keys, slots)
        .pull_update(keys, slots, lr, rescale, momentum) / .barrier() / .comm_buf(key)

B200 extensions: KvConfig(bucket_bytes, issue_order, comm_dtype, p2p=1 (fused
NVLink allreduce+update kernel) / 2 (NVLS), zero=1 (ZeRO-1)),
KvStore.bucket_view[_tensor] (gradient-as-bucket-view), Engine.import_event /
stream_wait (a framework's own CUDA stream as producer / consumer),
Transport.allreduce_p2p / allreduce_nvls, SynthModel (the bench's trainer).

Device buffers are torch tensors (plumbing only); everything they are handed
to runs in libcollsim_b200.so.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import tempfile
import threading
import weakref
from dataclasses import dataclass
from typing import Callable, Iterable, Sequence

from . import _lib
from ._lib import check, lib


def _close_children(parent) -> None:
    """An Engine / Transport outlives every KvStore / SynthModel built on it:
    closing the parent first closes its live children, so no native
    destructor (a KvStore drains its engine) ever runs against an engine or a
    transport that is already gone -- whichever order the caller, or the
    garbage collector on some other thread, gets to them."""
    for child in list(getattr(parent, "_children", ())):
        child.close()


def _adopt(child, *parents) -> None:
    for p in parents:
        p._children.add(child)

try:  # torch is plumbing: device memory and streams
    import torch
except ImportError:  # pragma: no cover
    torch = None

F64, F32, BF16 = _lib.CS_F64, _lib.CS_F32, _lib.CS_BF16
COMPUTE, COPY, COLLECTIVE, OTHER = 0, 1, 2, 3
INLINE, POOL = _lib.CS_DISPATCH_INLINE, _lib.CS_DISPATCH_POOL
MODES = {"funnel": 0, "depcha": 1, "concom": 2, "naive": 3}


def dtype_code(dt) -> int:
    if isinstance(dt, int):
        return dt
    if torch is not None:
        if dt == torch.float64:
            return F64
        if dt == torch.float32:
            return F32
        if dt == torch.bfloat16:
            return BF16
    raise ValueError(f"unsupported dtype {dt}")


def torch_dtype(code: int):
    return {F64: torch.float64, F32: torch.float32, BF16: torch.bfloat16}[code]


def device_count() -> int:
    n = C.c_int()
    check(lib.cs_device_count(C.byref(n)))
    return n.value


def _u64_array(xs: Sequence[int]):
    arr = (C.c_uint64 * max(1, len(xs)))(*xs)
    return arr, len(xs)


# ------------------------------------------------------------------- trace

class TraceSink:
    """R/core/include/collsim/trace.hpp:57-78."""

    def __init__(self):
        h = C.c_void_p()
        check(lib.cs_trace_create(C.byref(h)))
        self.h = h

    def count(self) -> int:
        n = C.c_uint64()
        check(lib.cs_trace_count(self.h, C.byref(n)))
        return n.value

    def write_jsonl(self, path: str) -> None:
        check(lib.cs_trace_write_jsonl(self.h, str(path).encode()))

    def snapshot(self) -> list[dict]:
        fd, path = tempfile.mkstemp(suffix=".jsonl")
        os.close(fd)
        try:
            self.write_jsonl(path)
            with open(path) as f:
                return [json.loads(line) for line in f if line.strip()]
        finally:
            os.unlink(path)

    def gauges(self) -> tuple[int, bool]:
        a, b = C.c_int(), C.c_int()
        check(lib.cs_trace_gauges(self.h, C.byref(a), C.byref(b)))
        return a.value, bool(b.value)

    def close(self):
        if self.h:
            lib.cs_trace_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ engine

class Engine:
    """Stream/event-mapped dependency engine (R/core/include/collsim/engine.hpp:41-74)."""

    def __init__(self, num_worker_threads: int, rank: int = 0, trace: TraceSink | None = None,
                 device: int = -1):
        h = C.c_void_p()
        check(lib.cs_engine_create(num_worker_threads, rank, device, trace.h if trace else None,
                                   C.byref(h)))
        self.h = h
        self._children = weakref.WeakSet()
        self.device = device
        self._keep: dict[int, object] = {}
        self._keep_mu = threading.Lock()
        self._next = 0

    def new_variable(self) -> int:
        t = C.c_uint64()
        check(lib.cs_engine_new_variable(self.h, C.byref(t)))
        return t.value

    def _hold(self, obj) -> int:
        with self._keep_mu:
            self._next += 1
            self._keep[self._next] = obj
            return self._next

    def _release(self, token: int) -> None:
        with self._keep_mu:
            self._keep.pop(token, None)

    def push(self, body: Callable[[], None], reads: Iterable[int] = (), mutates: Iterable[int] = (),
             kind: int = OTHER, key: int = -1) -> int:
        """Host body, reference semantics: runs on the pool once every earlier
        conflicting op has completed (device work included)."""
        holder = {}

        def tramp(_arg):
            try:
                body()
                return 0
            except BaseException:  # body failure poisons the engine
                return 1
            finally:
                self._release(holder["t"])

        cb = _lib.HOST_FN(tramp)
        holder["t"] = self._hold(cb)
        r, nr = _u64_array(list(reads))
        m, nm = _u64_array(list(mutates))
        op = C.c_uint64()
        try:
            check(lib.cs_engine_push_host(self.h, cb, None, r, nr, m, nm, kind, key, C.byref(op)))
        except Exception:
            self._release(holder["t"])
            raise
        return op.value

    def push_stream(self, body: Callable[[int], None], reads: Iterable[int] = (),
                    mutates: Iterable[int] = (), kind: int = OTHER, key: int = -1, lane: int = 0,
                    dispatch: int = INLINE) -> int:
        """Stream body: body(stream_handle) enqueues device work on the lane."""
        holder = {}

        def tramp(_arg, stream):
            try:
                body(stream or 0)
                return 0
            except BaseException:
                return 1
            finally:
                self._release(holder["t"])

        cb = _lib.STREAM_FN(tramp)
        holder["t"] = self._hold(cb)
        r, nr = _u64_array(list(reads))
        m, nm = _u64_array(list(mutates))
        op = C.c_uint64()
        try:
            check(lib.cs_engine_push_stream(self.h, cb, None, r, nr, m, nm, kind, key, lane, dispatch,
                                            C.byref(op)))
        except Exception:
            self._release(holder["t"])
            raise
        return op.value

    def wait_for(self, tag: int) -> None:
        check(lib.cs_engine_wait_for(self.h, tag))

    def import_event(self, cuda_event: int, mutates: Iterable[int], key: int = -1, lane: int = 0) -> int:
        """The writes recorded by `cuda_event` (on an external stream) become
        the latest writes of `mutates`."""
        m, nm = _u64_array(list(mutates))
        op = C.c_uint64()
        check(lib.cs_engine_import_event(self.h, cuda_event, m, nm, key, lane, C.byref(op)))
        return op.value

    def stream_wait(self, tags: Iterable[int], stream: int) -> None:
        """Make an external stream wait for every op pushed so far on `tags`."""
        t, nt = _u64_array(list(tags))
        check(lib.cs_engine_stream_wait(self.h, t, nt, stream))

    def wait_all(self) -> None:
        check(lib.cs_engine_wait_all(self.h))

    def shutdown(self) -> None:
        check(lib.cs_engine_shutdown(self.h))

    def new_lane(self, priority: int = 0) -> int:
        lane = C.c_int()
        check(lib.cs_engine_new_lane(self.h, priority, C.byref(lane)))
        return lane.value

    def lane_stream(self, lane: int = 0) -> int:
        s = C.c_void_p()
        check(lib.cs_engine_lane_stream(self.h, lane, C.byref(s)))
        return s.value or 0

    def set_watchdog(self, ms: int) -> None:
        """Device waits give up (DeadlockTimeout, every transport aborted) after ms."""
        check(lib.cs_engine_set_watchdog(self.h, int(ms)))

    def num_threads(self) -> int:
        n = C.c_int()
        check(lib.cs_engine_num_threads(self.h, C.byref(n)))
        return n.value

    def stats(self) -> tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        check(lib.cs_engine_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if self.h:
            _close_children(self)
            lib.cs_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------- transport

def _buf_args(buf, dtype=None, count=None):
    """(ptr, count, dtype) from a torch tensor or an explicit triple."""
    if torch is not None and isinstance(buf, torch.Tensor):
        return buf.data_ptr(), buf.numel(), dtype_code(buf.dtype)
    return int(buf or 0), int(count or 0), dtype_code(dtype if dtype is not None else F32)


class Transport:
    """R/core/include/collsim/collective.hpp:36-61 over device memory."""

    WORLD = 0

    def __init__(self, handle):
        self.h = handle
        self._children = weakref.WeakSet()

    @staticmethod
    def world() -> int:
        return 0

    @classmethod
    def local(cls, num_ranks: int, watchdog_ms: int = 5000, trace: TraceSink | None = None,
              peer: bool = False):
        """In-process rank threads.  peer=True: the rank threads run the fused
        peer-memory kernels on each other's buffers (one GPU; every rank's grid
        capped so all grids are co-resident) instead of the last-arriver sum."""
        h = C.c_void_p()
        fn = lib.cs_transport_create_local_peer if peer else lib.cs_transport_create_local
        check(fn(num_ranks, watchdog_ms, trace.h if trace else None, C.byref(h)))
        return cls(h)

    @classmethod
    def nccl(cls, name: str, num_ranks: int, rank: int, device: int, watchdog_ms: int = 60000,
             trace: TraceSink | None = None):
        h = C.c_void_p()
        check(lib.cs_transport_create_nccl(name.encode(), num_ranks, rank, device, watchdog_ms,
                                           trace.h if trace else None, C.byref(h)))
        return cls(h)

    @classmethod
    def ledger_only(cls, num_ranks: int, watchdog_ms: int = 5000, trace: TraceSink | None = None,
                    name: str = "", rank: int = 0):
        h = C.c_void_p()
        check(lib.cs_transport_create_ledger_only(name.encode(), num_ranks, rank, watchdog_ms,
                                                  trace.h if trace else None, C.byref(h)))
        return cls(h)

    def num_ranks(self) -> int:
        n = C.c_int()
        check(lib.cs_transport_num_ranks(self.h, C.byref(n)))
        return n.value

    def num_communicators(self) -> int:
        n = C.c_int()
        check(lib.cs_transport_num_communicators(self.h, C.byref(n)))
        return n.value

    def new_communicator(self) -> int:
        c = C.c_int()
        check(lib.cs_transport_new_communicator(self.h, C.byref(c)))
        return c.value

    def set_inject_latency(self, us: int) -> None:
        check(lib.cs_transport_set_inject_latency(self.h, int(us)))

    def abort(self) -> None:
        check(lib.cs_transport_abort(self.h))

    def allreduce_sum(self, comm: int, rank: int, buf, trace_key: int = -1, stream: int = 0,
                      dtype=None, count=None) -> None:
        p, n, dt = _buf_args(buf, dtype, count)
        check(lib.cs_allreduce_sum(self.h, comm, rank, p, n, dt, trace_key, stream))

    def broadcast(self, comm: int, rank: int, root: int, buf, trace_key: int = -1, stream: int = 0,
                  dtype=None, count=None) -> None:
        p, n, dt = _buf_args(buf, dtype, count)
        check(lib.cs_broadcast(self.h, comm, rank, root, p, n, dt, trace_key, stream))

    def barrier(self, comm: int, rank: int, trace_key: int = -1, stream: int = 0) -> None:
        check(lib.cs_barrier(self.h, comm, rank, trace_key, stream))

    def p2p_capable(self) -> bool:
        v = C.c_int()
        check(lib.cs_transport_p2p_capable(self.h, C.byref(v)))
        return bool(v.value)

    def share_buffer(self, base: int, rank: int | None = None) -> list[int]:
        """Setup collective: every rank's mapping of its peers' allocation.
        rank is required on a local peer transport (one object, many ranks)."""
        n = self.num_ranks()
        out = (C.c_void_p * n)()
        if rank is None:
            check(lib.cs_transport_share_buffer(self.h, base, out))
        else:
            check(lib.cs_transport_share_buffer_rank(self.h, rank, base, out))
        return [p or 0 for p in out]

    def p2p_stamps(self, rank: int):
        """CSB_P2P_TRACE=1: the last peer launch's per-CTA phase stamps of
        `rank` as a (CTAs, 5) uint64 array (ns; rows of unused CTAs are 0)."""
        import numpy as np
        n = C.c_int()
        check(lib.cs_transport_p2p_stamps(self.h, rank, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint64)
        if n.value:
            check(lib.cs_transport_p2p_stamps(self.h, rank, out.ctypes.data_as(C.POINTER(C.c_uint64)), n.value,
                                              C.byref(n)))
        return out.reshape(-1, 5)

    def device_failure(self) -> str:
        """A peer kernel's device timeout or an NCCL asynchronous error ("" if none)."""
        buf = C.create_string_buffer(512)
        check(lib.cs_transport_device_failure(self.h, buf, 512))
        return buf.value.decode()

    @staticmethod
    def _update_arg(update):
        if update is None:
            return None, None
        ents, wdt, lr, rescale, mom, *rest = update
        shard_only = int(bool(rest[0])) if rest else 0
        arr = (_lib.UpdateEntry * max(1, len(ents)))(*[_lib.UpdateEntry(w, g, m or None, k) for w, g, m, k in ents])
        u = _lib.P2PUpdateC(C.cast(arr, C.c_void_p), len(ents), wdt, lr, rescale, mom, shard_only)
        return C.byref(u), (arr, u)

    def allreduce_p2p(self, comm: int, rank: int, peer_bufs, n: int, dtype: int, trace_key: int = -1,
                      update=None, stream: int = 0) -> None:
        """update: (entries[(w, g, mom, n)], w_dtype, lr, rescale, momentum[, shard_only]) or None."""
        bufs = (C.c_void_p * len(peer_bufs))(*peer_bufs)
        upd, _keep = self._update_arg(update)
        check(lib.cs_allreduce_p2p(self.h, comm, rank, bufs, n, dtype, trace_key, upd, stream))

    def nvls_capable(self) -> bool:
        v = C.c_int()
        check(lib.cs_transport_nvls_capable(self.h, C.byref(v)))
        return bool(v.value)

    def alloc_nvls(self, nbytes: int) -> tuple[int, int]:
        uc, mc = C.c_void_p(), C.c_void_p()
        check(lib.cs_transport_alloc_nvls(self.h, nbytes, C.byref(uc), C.byref(mc)))
        return uc.value, mc.value

    def allreduce_nvls(self, comm: int, rank: int, uc: int, mc: int, n: int, dtype: int, trace_key: int = -1,
                       update=None, stream: int = 0) -> None:
        upd, _keep = self._update_arg(update)
        check(lib.cs_allreduce_nvls(self.h, comm, rank, uc, mc, n, dtype, trace_key, upd, stream))

    def close(self):
        if self.h:
            _close_children(self)
            lib.cs_transport_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def create_communicators(transport: Transport, count: int) -> list[int]:
    """R/core/include/collsim/kvstore.hpp:32-35."""
    arr = (C.c_int * max(1, count))()
    check(lib.cs_create_communicators(transport.h, count, arr))
    return list(arr[:count])


# ----------------------------------------------------------------- kvstore

class _CudaArray:
    """__cuda_array_interface__ over a raw device pointer (zero-copy wrap)."""

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def device_tensor(ptr: int, numel: int, dtype: int | None, device: int = 0):
    """A torch view of `numel` elements at device address `ptr` (memory owned
    by the library, e.g. a KvStore bucket slot)."""
    code = F32 if dtype is None else dtype
    if code == BF16:  # no bf16 typestr: view 16-bit storage as bfloat16
        return torch.as_tensor(_CudaArray(ptr, numel, "<i2"), device=f"cuda:{device}").view(torch.bfloat16)
    return torch.as_tensor(_CudaArray(ptr, numel, {F32: "<f4", F64: "<f8"}[code]), device=f"cuda:{device}")


@dataclass
class KvConfig:
    """R/core/include/collsim/kvstore.hpp:26-30 + B200 extensions."""
    mode: str = "funnel"
    outstanding: int = 1
    num_keys: int = 0
    comm_dtype: int = -1
    bucket_bytes: int = 0
    issue_order: int = 0
    comm_priority: int = 0
    p2p: int = 0
    zero: int = 0


@dataclass
class Slot:
    """TensorSlot (kvstore.hpp:16-19): a device tensor plus its engine tag."""
    value: "torch.Tensor"
    tag: int

    def c(self) -> _lib.SlotC:
        return _lib.SlotC(self.value.data_ptr(), dtype_code(self.value.dtype), self.value.numel(),
                          self.tag)


class KvStore:
    """Per-rank init/push/pull/barrier facade (R/core/include/collsim/kvstore.hpp:54-96)."""

    def __init__(self, engine: Engine, transport: Transport, rank: int, config: KvConfig,
                 concom_comms: Sequence[int] = ()):
        cfg = _lib.KvConfigC(MODES[config.mode] if isinstance(config.mode, str) else config.mode,
                             config.outstanding, config.num_keys, config.comm_dtype,
                             config.bucket_bytes, config.issue_order, config.comm_priority,
                             int(config.p2p), int(config.zero))
        comms = (C.c_int * max(1, len(concom_comms)))(*concom_comms)
        h = C.c_void_p()
        check(lib.cs_kv_create(engine.h, transport.h, rank, C.byref(cfg), comms, len(concom_comms),
                               C.byref(h)))
        self.h = h
        self.engine = engine
        self.transport = transport
        self.config = config
        _adopt(self, engine, transport)
        self.rank = rank

    @staticmethod
    def _lists(keys, slots):
        if isinstance(keys, int):
            keys, slots = [keys], [slots]
        karr = (C.c_int * len(keys))(*keys)
        sarr = (_lib.SlotC * len(slots))(*[s.c() for s in slots])
        return karr, sarr, len(keys)

    def init(self, key: int, weights: Slot) -> None:
        check(lib.cs_kv_init(self.h, key, weights.c()))

    def push(self, keys, grads) -> None:
        k, s, n = self._lists(keys, grads)
        check(lib.cs_kv_push(self.h, k, s, n))

    def pull(self, keys, outs) -> None:
        k, s, n = self._lists(keys, outs)
        check(lib.cs_kv_pull(self.h, k, s, n))

    def pull_update(self, keys, weights, lr: float, rescale: float, momentum: float = 0.0) -> None:
        k, s, n = self._lists(keys, weights)
        sgd = _lib.SgdC(lr, rescale, momentum)
        check(lib.cs_kv_pull_update(self.h, k, s, n, C.byref(sgd)))

    def barrier(self) -> None:
        check(lib.cs_kv_barrier(self.h))

    def outstanding_in_flight(self) -> int:
        n = C.c_int()
        check(lib.cs_kv_outstanding_in_flight(self.h, C.byref(n)))
        return n.value

    def comm_buf(self, key: int):
        """Synchronizes and returns the key's comm buffer as a CPU tensor."""
        n, dt = C.c_uint64(), C.c_int()
        check(lib.cs_kv_comm_buf(self.h, key, None, C.byref(n), C.byref(dt)))
        out = torch.empty(n.value, dtype=torch_dtype(dt.value))
        check(lib.cs_kv_comm_buf(self.h, key, C.c_void_p(out.data_ptr()), None, None))
        return out

    def key_map(self, key: int) -> tuple[int, int]:
        b, off = C.c_int(), C.c_uint64()
        check(lib.cs_kv_key_map(self.h, key, C.byref(b), C.byref(off)))
        return b.value, off.value

    def bucket_view(self, key: int) -> int:
        """Device address of the key's slot in its comm bucket (comm dtype)."""
        p = C.c_void_p()
        check(lib.cs_kv_bucket_view(self.h, key, C.byref(p)))
        return p.value or 0

    def bucket_view_tensor(self, key: int, numel: int, dtype: int, device: int = 0):
        """The key's bucket slot as a torch tensor (zero-copy; dtype = the
        comm dtype): produce the gradient into it and push it as the key's slot."""
        return device_tensor(self.bucket_view(key), numel, dtype, device)

    def register_grads(self, base: int, nbytes: int) -> None:
        """Setup collective: the allocation holding this rank's gradients
        (cudaMalloc base, same layout on every rank); whole-bucket
        pull_updates then read every rank's gradients in place (N > 1)."""
        check(lib.cs_kv_register_grads(self.h, base, nbytes))

    def arena(self) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_uint64()
        check(lib.cs_kv_arena(self.h, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def num_buckets(self) -> int:
        n = C.c_int()
        check(lib.cs_kv_num_buckets(self.h, C.byref(n)))
        return n.value

    def close(self):
        if self.h:
            lib.cs_kv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- kernels

def pack(entries: Sequence[tuple], src_dt: int, dst_dt: int, stream: int = 0) -> None:
    """Kernel (a): entries of (src_ptr, dst_ptr, n)."""
    arr = (_lib.CopyEntry * max(1, len(entries)))(*[_lib.CopyEntry(s, d, n) for s, d, n in entries])
    check(lib.cs_pack(arr, len(entries), src_dt, dst_dt, stream))


def sum_buffers(ins: Sequence[int], outs: Sequence[int], n: int, dt: int, stream: int = 0) -> None:
    """Kernel (b): every out = rank-order sum of ins."""
    a = (C.c_void_p * max(1, len(ins)))(*ins)
    b = (C.c_void_p * max(1, len(outs)))(*outs)
    check(lib.cs_sum_buffers(a, len(ins), b, len(outs), n, dt, stream))


def sgd_update(entries: Sequence[tuple], w_dt: int, g_dt: int, lr: float, rescale: float,
               momentum: float = 0.0, stream: int = 0) -> None:
    """Kernel (c): entries of (w_ptr, g_ptr, mom_ptr_or_0, n)."""
    arr = (_lib.UpdateEntry * max(1, len(entries)))(
        *[_lib.UpdateEntry(w, g, m or None, n) for w, g, m, n in entries])
    check(lib.cs_sgd_update(arr, len(entries), w_dt, g_dt, lr, rescale, momentum, stream))


def synth_backward(src: int, dst: int, n: int, dt: int, spin_ns: int = 0, ctas: int = 0,
                   stream: int = 0) -> None:
    check(lib.cs_synth_backward(src, dst, n, dt, spin_ns, ctas, stream))


def checksum(x: int, n: int, dt: int, out_dev: int, stream: int = 0) -> None:
    check(lib.cs_checksum(x, n, dt, out_dev, stream))


# --------------------------------------------------- synthetic training step

class SynthModel:
    """The reference trainer's loop shapes (trainer.cpp:112-141) over a key
    set with a synthetic backward, driven entirely in the native library."""

    BACKWARD, COMM, LOCAL_UPDATE, CHECKSUM = 1, 2, 4, 8

    def __init__(self, engine: Engine, transport: Transport, rank: int, nranks: int, sizes,
                 mode: str = "depcha", w_dtype: int = F32, g_dtype: int = F32, comm_dtype: int = F32,
                 bucket_bytes: int = 0, issue_order: int = 0, outstanding: int = 1, lr: float = 0.1,
                 rescale: float = 1.0, momentum: float = 0.0, backward_ns: int = 0,
                 backward_ctas: int = 0, fused_update: bool = True, comm_priority: int = 0, p2p: bool = False,
                 host_source: bool = False, concom_comms: Sequence[int] = (),
                 ready_ms: Sequence[float] | None = None, grad_views: bool = False, zero: bool = False,
                 order_seed: int = 0, direct_grads: bool = False):
        cfg = _lib.SynthConfigC(MODES[mode], w_dtype, g_dtype, comm_dtype, bucket_bytes, issue_order,
                                outstanding, lr, rescale, momentum, backward_ns, backward_ctas,
                                int(fused_update), comm_priority, int(host_source), int(p2p), int(grad_views),
                                int(zero), int(order_seed), int(direct_grads))
        sz = (C.c_uint64 * len(sizes))(*sizes)
        comms = (C.c_int * max(1, len(concom_comms)))(*concom_comms)
        h = C.c_void_p()
        rd = (C.c_double * len(sizes))(*ready_ms) if ready_ms is not None else None
        check(lib.cs_synth_create_profiled(engine.h, transport.h, rank, nranks, C.byref(cfg), sz, rd,
                                           len(sizes), comms, len(concom_comms), C.byref(h)))
        self.h = h
        self.engine = engine
        self.transport = transport
        _adopt(self, engine, transport)
        self.sizes = list(sizes)
        self.w_dtype = w_dtype

    def init(self) -> None:
        check(lib.cs_synth_init(self.h))

    def step(self, flags: int) -> None:
        check(lib.cs_synth_step(self.h, flags))

    def run(self, steps: int, flags: int) -> float:
        ms = C.c_double()
        check(lib.cs_synth_run(self.h, steps, flags, C.byref(ms)))
        return ms.value

    def run_e2e(self, steps: int, flags: int) -> float:
        ms = C.c_double()
        check(lib.cs_synth_run_e2e(self.h, steps, flags, C.byref(ms)))
        return ms.value

    def checksum(self) -> float:
        v = C.c_double()
        check(lib.cs_synth_checksum(self.h, C.byref(v)))
        return v.value

    def read_weights(self):
        """Every key's weights (numpy, the weight dtype), keys concatenated."""
        import numpy as np
        dt = {F64: np.float64, F32: np.float32, BF16: np.uint16}[self.w_dtype]
        out = np.empty(int(sum(self.sizes)), dtype=dt)
        check(lib.cs_synth_read_weights(self.h, out.ctypes.data, out.nbytes))
        return out

    def last_host_ms(self) -> float:
        v = C.c_double()
        check(lib.cs_synth_last_host_ms(self.h, C.byref(v)))
        return v.value

    def info(self) -> dict:
        g, h2d, nb = C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib.cs_synth_info(self.h, C.byref(g), C.byref(h2d), C.byref(nb)))
        return {"grad_bytes": g.value, "h2d_bytes_per_step": h2d.value, "num_buckets": nb.value}

    def close(self):
        if self.h:
            lib.cs_synth_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def launch_count() -> int:
    n = C.c_uint64()
    check(lib.cs_launch_count(C.byref(n)))
    return n.value


def profile_enable(on: bool) -> None:
    check(lib.cs_profile_enable(int(on)))


def profile_reset() -> None:
    check(lib.cs_profile_reset())


def host_profile(reset: bool = False) -> dict:
    buf = C.create_string_buffer(4096)
    check(lib.cs_host_profile(buf, 4096, int(reset)))
    return json.loads(buf.value.decode())


def profile_collect(kind: str) -> dict:
    n, ms, b = C.c_uint64(), C.c_double(), C.c_double()
    check(lib.cs_profile_collect(_lib.KERNEL_KINDS[kind], C.byref(n), C.byref(ms), C.byref(b)))
    return {"launches": n.value, "total_ms": ms.value, "bytes": b.value}
