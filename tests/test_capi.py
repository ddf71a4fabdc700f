"""The drop-in boundary: libcollsim_b200.so loads (no GPU needed) and exports
every entry point include/collsim_b200.h declares; status codes map to the
reference error kinds (R/core/include/collsim/error.hpp:10-31).  CPU only."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "collsim_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|char\s*\*|const char\s*\*)\s+\**\s*(cs_\w+)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert len(names) > 50
    for must in ("cs_pack", "cs_sum_buffers", "cs_sgd_update", "cs_engine_push_stream", "cs_allreduce_sum",
                 "cs_kv_push", "cs_kv_pull", "cs_kv_pull_update", "cs_create_communicators"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1802_06949_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # and the ctypes table binds exactly the declared set
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_library_is_sm100a_only():
    from paper_1802_06949_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_status_names_mirror_reference_error_kinds():
    from paper_1802_06949_b200._lib import lib
    names = {s: lib.cs_status_name(s).decode() for s in range(-8, 1)}
    assert names[0] == "OK"
    assert names[-1] == "ConfigError" and names[-2] == "UsageError" and names[-3] == "MismatchError"
    assert names[-4] == "DeadlockTimeout" and names[-5] == "EngineError"


def test_errors_cross_the_boundary_as_status_codes():
    from paper_1802_06949_b200 import ConfigError, Engine, Transport, UsageError
    with pytest.raises(ConfigError):
        Engine(0)  # engine.cpp:23-25
    with pytest.raises(ConfigError):
        Transport.ledger_only(0)
    with pytest.raises(ConfigError):
        Transport.ledger_only(2, watchdog_ms=0)
    e = Engine(1)
    with pytest.raises(UsageError):
        e.push_stream(lambda s: None)  # host-only engine: no lanes
    with pytest.raises(UsageError):
        e.wait_for(12345)  # unknown tag


def test_kernels_reject_bad_arguments_without_a_gpu():
    from paper_1802_06949_b200 import UsageError, api
    with pytest.raises(UsageError):
        api.sum_buffers([], [1], 10, api.F32)
    with pytest.raises(UsageError):
        api.sum_buffers([1] * 17, [1], 10, api.F32)
    with pytest.raises(UsageError):
        api.sgd_update([(16, 32, 0, 4)], api.F32, api.F32, 0.1, 1.0, 0.9)  # momentum needs a buffer


def test_device_count_is_zero_here_or_positive_on_box():
    from paper_1802_06949_b200 import device_count
    assert device_count() >= 0


def test_kvstore_config_validation_before_any_device_work():
    """kvstore.cpp:41-51 checks plus the B200 options: every inconsistent
    configuration is a ConfigError raised by the constructor, on any host."""
    from paper_1802_06949_b200 import ConfigError, Engine, KvConfig, KvStore, Transport
    eng = Engine(1, 0, None, -1)  # host-only engine
    tr = Transport.ledger_only(2)
    bad = [
        (KvConfig("funnel", 1, 0), "num_keys"),
        (KvConfig("concom", 0, 4), "outstanding"),
        (KvConfig("depcha", 1, 4, p2p=1), "fusion buckets"),
        (KvConfig("concom", 1, 4, bucket_bytes=1 << 20, p2p=2), "one ordered comm stream"),
        (KvConfig("funnel", 1, 4, bucket_bytes=1 << 20, p2p=1, zero=1), "ZeRO-1"),
        (KvConfig("depcha", 1, 4, bucket_bytes=1 << 20, zero=1), "ZeRO-1"),
    ]
    for cfg, msg in bad:
        with pytest.raises(ConfigError, match=msg):
            KvStore(eng, tr, 0, cfg, [1] * cfg.outstanding if cfg.mode == "concom" else [])
    with pytest.raises(ConfigError, match="CUDA device"):  # a valid config still needs a device engine
        KvStore(eng, tr, 0, KvConfig("depcha", 1, 4))
    eng.close()
    tr.close()


def test_interop_and_peer_memory_entry_points_reject_misuse_without_a_gpu():
    """The B200 entry points fail with status codes, never crash: a null
    framework event, stream ops on a host-only engine, peer-memory / NVLS
    collectives on a transport that has no peer path."""
    from paper_1802_06949_b200 import Engine, Transport, UsageError, api
    e = Engine(1)  # host-only
    t = e.new_variable()
    with pytest.raises(UsageError, match="null event"):
        e.import_event(0, [t])
    e.stream_wait([t], 0)  # nothing pushed on the tag: nothing to wait for
    tr = Transport.ledger_only(2)
    assert not tr.p2p_capable() and not tr.nvls_capable()
    with pytest.raises(UsageError, match="peer-memory"):
        tr.share_buffer(0x1000)
    with pytest.raises(UsageError):
        tr.allreduce_p2p(0, 0, [0x1000, 0x2000], 64, api.F32)
    with pytest.raises(UsageError):
        tr.alloc_nvls(1 << 20)
    tr.close()
    e.close()
