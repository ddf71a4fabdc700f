"""Rank-thread fixtures mirroring the reference's (test_kvstore.cpp:18-40
`kv_ranks`, test_collective.cpp:18-26 `on_ranks`)."""
from __future__ import annotations

import threading

from paper_1802_06949_b200 import Engine, KvConfig, KvStore, create_communicators


def on_ranks(n: int, fn) -> None:
    errs = [None] * n

    def run(r):
        try:
            fn(r)
        except BaseException as e:  # surfaced after join
            errs[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e


def kv_ranks(num_ranks: int, engine_threads: int, config: KvConfig, transport, sink, body,
             device: int = 0, swallow=()):
    """One engine + store per rank thread over a shared transport; runs
    body(rank, engine, store), drains, closes.  Exceptions of the types in
    `swallow` are returned per rank instead of raised."""
    comms = create_communicators(transport, config.outstanding) if config.mode == "concom" else []
    errors = [None] * num_ranks

    def run(r):
        eng = Engine(engine_threads, r, sink, device)
        store = None
        try:
            store = KvStore(eng, transport, r, config, comms)
            body(r, eng, store)
        except BaseException as e:
            errors[r] = e
        try:
            eng.wait_all()
        except BaseException:
            pass  # drained; the body already observed the failure (test_kvstore.cpp:31-35)
        if store is not None:
            store.close()
        eng.shutdown()
        eng.close()

    th = [threading.Thread(target=run, args=(r,)) for r in range(num_ranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errors:
        if e is not None and not isinstance(e, tuple(swallow)):
            raise e
    return errors
