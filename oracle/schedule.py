"""Restatement of the host-side schedule contracts (issue order and key ->
comm-buffer map).  TEST INFRASTRUCTURE ONLY (the checker for the product's
C++ KvStore, never imported by the product).

Reference anchors (R = /root/reference/proj):
  * trainer loop shapes          R/core/src/trainer.cpp:112-141
  * init broadcasts, key order   R/core/src/kvstore.cpp:76-97
  * concom key -> comm           R/core/src/kvstore.cpp:119 (key % outstanding, ids 1..outstanding)
  * 1:1 comm_buf[key]            R/core/src/kvstore.cpp:84

The fusion-bucket map has no reference counterpart (parity unpinned, new on
the B200 side); this file is its specification: keys are taken in issue order
(ascending or descending key), a bucket is closed when adding the next key
would exceed bucket_bytes (a key larger than bucket_bytes gets its own
bucket), and inside a bucket each key's slot starts at a multiple of 256
bytes.  bucket_bytes == 0 reproduces the reference's 1:1 map.
"""
from __future__ import annotations

ALIGN_BYTES = 256


def bucket_map(sizes, elem_size: int, bucket_bytes: int, issue_order: int = 0):
    """-> (bucket_of_key, offset_of_key (elements), groups: keys per bucket in bucket order)."""
    K = len(sizes)
    order = list(range(K)) if issue_order == 0 else list(reversed(range(K)))
    if bucket_bytes == 0:
        return list(range(K)), [0] * K, [[k] for k in order]
    align = ALIGN_BYTES // elem_size
    bucket = [0] * K
    offset = [0] * K
    groups: list[list[int]] = []
    cur: list[int] = []
    cur_bytes = 0
    cur_count = 0
    for k in order:
        b = sizes[k] * elem_size
        if cur and cur_bytes + b > bucket_bytes:
            groups.append(cur)
            cur, cur_bytes, cur_count = [], 0, 0
        bucket[k] = len(groups)
        offset[k] = cur_count
        cur.append(k)
        cur_count = (cur_count + sizes[k] + align - 1) // align * align
        cur_bytes += b
    if cur:
        groups.append(cur)
    return bucket, offset, groups


def issue_sequence(mode: str, K: int, iters: int, outstanding: int = 1):
    """Per-rank `kind:comm:seq:key` list the trainer loop shape produces with
    the 1:1 map (identical on every rank).  For concom the per-communicator
    subsequences are the contract (cross-comm interleaving is unordered)."""
    out = [f"broadcast:0:{k}:{k}" for k in range(K)]
    world_seq = K
    comm_seq = {c: 0 for c in range(1, outstanding + 1)}
    for _ in range(iters):
        if mode in ("funnel", "depcha"):
            for k in range(K):
                out.append(f"allreduce:0:{world_seq}:{k}")
                world_seq += 1
        elif mode == "concom":
            since = 0
            for k in range(K):
                c = 1 + k % outstanding
                out.append(f"allreduce:{c}:{comm_seq[c]}:{k}")
                comm_seq[c] += 1
                since += 1
                if since == outstanding:
                    out.append(f"barrier:0:{world_seq}:-1")
                    world_seq += 1
                    since = 0
            if since:
                out.append(f"barrier:0:{world_seq}:-1")
                world_seq += 1
        else:
            raise ValueError(mode)
    return out
