"""B200-native gradient-aggregation hot path of arXiv 1802.06949 (collsim drop-in).

KvStore init/push/pull/barrier over a CUDA stream/event dependency engine,
collectives matched by a host ledger and executed by hand-written sm_100a
kernels (in-process ranks) or NCCL over NVLink (one process per GPU), with
fused SGD / momentum updates.  The native library is
paper_1802_06949_b200/lib/libcollsim_b200.so (C ABI: include/collsim_b200.h).
"""
from ._lib import (ConfigError, CsError, CudaError, DeadlockTimeout, EngineError,  # noqa: F401
                   MismatchError, NcclError, UsageError, LIB_PATH)
from .api import (BF16, F32, F64, Engine, KvConfig, KvStore, Slot, TraceSink,  # noqa: F401
                  Transport, create_communicators, device_count)

__all__ = [
    "Engine", "Transport", "KvStore", "KvConfig", "Slot", "TraceSink", "create_communicators",
    "device_count", "F64", "F32", "BF16", "ConfigError", "UsageError", "MismatchError",
    "DeadlockTimeout", "EngineError", "CudaError", "NcclError", "CsError", "LIB_PATH",
]
