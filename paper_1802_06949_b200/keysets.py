"""Gradient key sets of BASELINE.json's configs.

ResNet-50 / AlexNet / ResNet-152 / Inception-v3 sizes are the
``parameters()`` numels of the torchvision models, in parameter order (key k
= the k-th parameter, as MXNet's KVStore numbers them); frozen in
keysets.json by ``python -m paper_1802_06949_b200.keysets --freeze`` so the
bench does not need torchvision at run time.  C5 ("deadlock stress", 2048
keys, 1 KiB - 64 MiB log-uniform) is pinned here: u = top 53 bits of
std::mt19937_64(0) as in the reference generator (tensor.cpp:28-38),
bytes = floor(2^(10 + 16u) / 16) * 16.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
FROZEN = HERE / "keysets.json"


def _mt19937_64(seed: int):
    mt = [0] * 312
    mt[0] = seed & 0xFFFFFFFFFFFFFFFF
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
    idx = 312
    while True:
        if idx >= 312:
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & 0xFFFFFFFFFFFFFFFF
        y ^= (y << 37) & 0xFFF7EEE000000000 & 0xFFFFFFFFFFFFFFFF
        y ^= y >> 43
        yield y & 0xFFFFFFFFFFFFFFFF


def stress_keys(n: int = 2048, elem_bytes: int = 4) -> list[int]:
    g = _mt19937_64(0)
    out = []
    for _ in range(n):
        u = (next(g) >> 11) * 2.0 ** -53
        b = int(2 ** (10 + 16 * u)) // 16 * 16
        out.append(max(1, b // elem_bytes))
    return out


def freeze() -> dict:
    import torchvision.models as tvm
    sets = {}
    for name, ctor in (("resnet50", lambda: tvm.resnet50()), ("alexnet", lambda: tvm.alexnet()),
                       ("resnet152", lambda: tvm.resnet152()),
                       ("inception_v3", lambda: tvm.inception_v3(aux_logits=True, init_weights=False))):
        sets[name] = [int(p.numel()) for p in ctor().parameters()]
    FROZEN.write_text(json.dumps(sets))
    return sets


def load(name: str) -> list[int]:
    if name == "stress":
        return stress_keys()
    if name.startswith("uniform"):  # uniform<K>x<N>, e.g. uniform16x1048576 (config 0)
        k, n = name[len("uniform"):].split("x")
        return [int(n)] * int(k)
    return json.loads(FROZEN.read_text())[name]


if __name__ == "__main__":
    if "--freeze" in sys.argv:
        s = freeze()
        print({k: (len(v), sum(v)) for k, v in s.items()})
