"""Parity of the sm_100a kernels (a) pack/cast, (b) rank-order sum, (c) SGD /
momentum update against the CPU oracle (oracle/oracle.c), which is pinned to
the reference in tests/test_oracle.py.

Bars: fp64 and fp32 bit-exact (the kernels use round-to-nearest intrinsics,
no FMA contraction, fixed rank order); bf16 bit-exact against the oracle's
bf16 restatement (fp32 accumulation, one RNE rounding); against the fp64
reference the north-star tolerances hold (1e-6 relative fp32, 1e-2 bf16).
"""
import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(a: np.ndarray):
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def stream():
    return torch.cuda.current_stream().cuda_stream


SIZES = [1, 7, 8, 9, 4095, 4096, 4097, 65536 + 3, 1 << 20]


# ------------------------------------------------------------------ (a) pack

@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("pair", ["f64f64", "f32f32", "f32bf16", "bf16f32", "f64f32", "bf16bf16"])
def test_pack_cast_matches_oracle(gpu, n, pair):
    from paper_1802_06949_b200 import api
    x64 = O.random_uniform(n, 11 + n)
    if pair.startswith("f64"):
        src, sdt = x64, api.F64
    elif pair.startswith("f32"):
        src, sdt = x64.astype(np.float32), api.F32
    else:
        src, sdt = O.f32_to_bf16_bits(x64.astype(np.float32)), api.BF16
    dname = pair[4:] if pair.startswith("bf16") else pair[3:]
    ddt = {"f64": api.F64, "f32": api.F32, "bf16": api.BF16}[dname]
    # expected
    if ddt == api.F64:
        exp = src.astype(np.float64) if sdt != api.BF16 else O.bf16_bits_to_f32(src).astype(np.float64)
    elif ddt == api.F32:
        exp = (O.bf16_bits_to_f32(src) if sdt == api.BF16 else src.astype(np.float32))
    else:
        exp = src if sdt == api.BF16 else O.f32_to_bf16_bits(src.astype(np.float32))
    s = dev(src)
    d = torch.empty(n, dtype=api.torch_dtype(ddt), device="cuda")
    api.pack([(s.data_ptr(), d.data_ptr(), n)], sdt, ddt, stream())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host(d), exp)


def test_pack_table_many_keys_and_misaligned(gpu):
    """A 600-entry table (split over two 512-entry launches), ragged sizes,
    misaligned (scalar-path) entries mixed with aligned ones."""
    from paper_1802_06949_b200 import api
    rng = np.random.default_rng(0)
    sizes = [int(x) for x in rng.integers(1, 3000, size=600)]
    total = sum(sizes) + 600
    src = dev(O.random_uniform(total, 5).astype(np.float32))
    dst = torch.zeros(total + 8, dtype=torch.float32, device="cuda")
    entries, off, expect = [], 0, np.zeros(total + 8, dtype=np.float32)
    hsrc = host(src)
    doff = 0
    for i, n in enumerate(sizes):
        mis = i % 3 == 0  # every third entry deliberately misaligned by one element
        so, do = off + (1 if mis else 0), doff + (1 if mis else 0)
        entries.append((src.data_ptr() + 4 * so, dst.data_ptr() + 4 * do, n))
        expect[do:do + n] = hsrc[so:so + n]
        off += n + 1
        doff += n + 1
    api.pack(entries, api.F32, api.F32, stream())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host(dst), expect)


# ------------------------------------------------------------------- (b) sum

@pytest.mark.parametrize("R", [2, 4, 8])
def test_sum_acceptance_criterion_1_fp64_bit_exact(gpu, R):
    """acceptance.cpp:42-84: R ranks x 100 tensors, n = 1 + (i*7) % 64,
    inputs random_uniform(n, mix_seed(R*1000+i, r)); the reference holds
    1e-12, the kernel is bit-exact."""
    from paper_1802_06949_b200 import api
    for i in range(100):
        n = 1 + (i * 7) % 64
        ins = [O.random_uniform(n, O.mix_seed(R * 1000 + i, r)) for r in range(R)]
        exp = O.rank_order_sum(ins, "f64")
        bufs = [dev(x) for x in ins]
        api.sum_buffers([b.data_ptr() for b in bufs], [b.data_ptr() for b in bufs], n, api.F64, stream())
        torch.cuda.synchronize()
        for b in bufs:
            np.testing.assert_array_equal(host(b), exp)


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8, 16])
@pytest.mark.parametrize("kind", ["f64", "f32", "bf16"])
@pytest.mark.parametrize("n", [1, 13, 4096, 4099, 300001])
def test_sum_multi_buffer(gpu, m, kind, n):
    from paper_1802_06949_b200 import api
    ins64 = [O.random_uniform(n, 100 + r) for r in range(m)]
    if kind == "f64":
        ins, dt = ins64, api.F64
    elif kind == "f32":
        ins, dt = [x.astype(np.float32) for x in ins64], api.F32
    else:
        ins, dt = [O.f32_to_bf16_bits(x.astype(np.float32)) for x in ins64], api.BF16
    exp = O.rank_order_sum(ins, kind)
    bufs = [dev(x) for x in ins]
    outs = [torch.empty_like(bufs[0]) for _ in range(2)]
    api.sum_buffers([b.data_ptr() for b in bufs], [o.data_ptr() for o in outs], n, dt, stream())
    torch.cuda.synchronize()
    for o in outs:
        np.testing.assert_array_equal(host(o), exp)
    # north-star tolerance against the fp64 reference sum of the rounded inputs
    ref = O.rank_order_sum([(O.bf16_bits_to_f32(x) if kind == "bf16" else x).astype(np.float64)
                            for x in ins], "f64")
    got = (O.bf16_bits_to_f32(host(outs[0])) if kind == "bf16" else host(outs[0])).astype(np.float64)
    scale = np.sum([np.abs((O.bf16_bits_to_f32(x) if kind == "bf16" else x).astype(np.float64))
                    for x in ins], axis=0)
    tol = {"f64": 0.0, "f32": 1e-6, "bf16": 1e-2}[kind]
    assert np.all(np.abs(got - ref) <= tol * scale + (0 if kind == "f64" else 1e-30))


# ---------------------------------------------------------------- (c) update

@pytest.mark.parametrize("momentum", [0.0, 0.9])
@pytest.mark.parametrize("n", [1, 4096, 4097, 1 << 18])
def test_sgd_fp64_bit_exact(gpu, momentum, n):
    """model.cpp:17-27 (momentum 0) -- bit-exact, no FMA contraction."""
    from paper_1802_06949_b200 import api
    w0, g = O.random_uniform(n, 7), O.random_uniform(n, 8)
    m0 = O.random_uniform(n, 9) if momentum else None
    lr, rescale = 0.1, 1.0 / 128
    ew, em = O.sgd_update(w0, g, lr, rescale, momentum, m0, "f64")
    w, gd = dev(w0), dev(g)
    md = dev(m0) if momentum else None
    api.sgd_update([(w.data_ptr(), gd.data_ptr(), md.data_ptr() if md is not None else 0, n)],
                   api.F64, api.F64, lr, rescale, momentum, stream())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host(w), ew)
    if momentum:
        np.testing.assert_array_equal(host(md), em)


@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_sgd_fp32_and_bf16_grad(gpu, momentum):
    from paper_1802_06949_b200 import api
    n = 100003
    w0 = O.random_uniform(n, 17).astype(np.float32)
    g32 = O.random_uniform(n, 18).astype(np.float32)
    m0 = O.random_uniform(n, 19).astype(np.float32) if momentum else None
    lr, rescale = 0.1, 1.0 / 512
    ew, em = O.sgd_update(w0, g32, lr, rescale, momentum, m0, "f32")
    w, gd = dev(w0), dev(g32)
    md = dev(m0) if momentum else None
    api.sgd_update([(w.data_ptr(), gd.data_ptr(), md.data_ptr() if md is not None else 0, n)],
                   api.F32, api.F32, lr, rescale, momentum, stream())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host(w), ew)  # fp32 restatement, bit-exact
    # bf16 gradient (comm buffer) into fp32 weights: exact vs the oracle fed
    # the bf16-rounded gradient promoted to fp32
    gb = O.f32_to_bf16_bits(g32)
    ew2, _ = O.sgd_update(w0, O.bf16_bits_to_f32(gb), lr, rescale, momentum, m0, "f32")
    w2 = dev(w0)
    md2 = dev(m0) if momentum else None
    api.sgd_update([(w2.data_ptr(), dev(gb).data_ptr(), md2.data_ptr() if md2 is not None else 0, n)],
                   api.F32, api.BF16, lr, rescale, momentum, stream())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host(w2), ew2)


def test_sgd_table_update(gpu):
    """Many keys in one launch (the fused bucket update)."""
    from paper_1802_06949_b200 import api
    rng = np.random.default_rng(3)
    sizes = [int(x) for x in rng.integers(1, 20000, size=70)]
    ws, gs, exp, entries = [], [], [], []
    for k, n in enumerate(sizes):
        w0, g = O.random_uniform(n, 1000 + k), O.random_uniform(n, 2000 + k)
        exp.append(O.sgd_update(w0, g, 0.1, 1 / 64)[0])
        ws.append(dev(w0))
        gs.append(dev(g))
        entries.append((ws[-1].data_ptr(), gs[-1].data_ptr(), 0, n))
    api.sgd_update(entries, api.F64, api.F64, 0.1, 1 / 64, 0.0, stream())
    torch.cuda.synchronize()
    for w, e in zip(ws, exp):
        np.testing.assert_array_equal(host(w), e)


# ---------------------------------------------------- full-size properties

def test_large_sum_linearity_and_checksum(gpu):
    """At BASELINE sizes (a 2,359,296-element ResNet-50 key, 8 ranks): the sum
    of checksums equals the checksum of the sum (fp64), spot indices match
    the oracle bit-for-bit."""
    from paper_1802_06949_b200 import api
    n, R = 2_359_296, 8
    gen = torch.Generator(device="cuda").manual_seed(0)
    bufs = [torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1 for _ in range(R)]
    out = torch.empty_like(bufs[0])
    api.sum_buffers([b.data_ptr() for b in bufs], [out.data_ptr()], n, api.F64, stream())
    cs = torch.zeros(R + 1, dtype=torch.float64, device="cuda")
    for r, b in enumerate(bufs):
        api.checksum(b.data_ptr(), n, api.F64, cs[r:].data_ptr(), stream())
    api.checksum(out.data_ptr(), n, api.F64, cs[R:].data_ptr(), stream())
    torch.cuda.synchronize()
    c = cs.cpu().numpy()
    assert abs(c[:R].sum() - c[R]) <= 1e-9 * np.abs(c[:R]).sum() + 1e-6
    idx = np.random.default_rng(1).integers(0, n, size=1000)
    hb = [b.cpu().numpy()[idx] for b in bufs]
    np.testing.assert_array_equal(out.cpu().numpy()[idx], O.rank_order_sum(hb, "f64"))


# ------------------------------------------------------- guard regions (OOB)

@pytest.mark.parametrize("dt", ["f64", "f32", "bf16"])
def test_kernels_never_write_outside_their_keys(gpu, dt):
    """compute-sanitizer is closed on the pool, so out-of-bounds writes are
    checked with canaries: every destination key of kernels (a), (b), (c)
    sits inside one buffer between guard gaps at odd element offsets (tails
    not a multiple of 8, unaligned keys: the scalar paths), and every guard
    element must come back bit-identical."""
    from paper_1802_06949_b200 import api
    code = {"f64": api.F64, "f32": api.F32, "bf16": api.BF16}[dt]
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dt]
    sizes, gap = [1, 7, 9, 63, 1000, 4097, 70001], 37
    offs, o = [], 5
    for n in sizes:
        offs.append(o)
        o += n + gap
    total = o
    guard = torch.full((total,), -1234.5, device="cuda", dtype=tdt)
    mask = torch.ones(total, dtype=torch.bool, device="cuda")
    for off, n in zip(offs, sizes):
        mask[off:off + n] = False

    def check(buf):
        torch.cuda.synchronize()
        assert torch.equal(buf[mask], guard[mask]), "a kernel wrote into a guard gap"

    s = stream()
    # (a) pack into the guarded buffer
    dst = guard.clone()
    src = [torch.randn(n, device="cuda").to(tdt) for n in sizes]
    api.pack([(x.data_ptr(), dst[off:].data_ptr(), n) for x, off, n in zip(src, offs, sizes)], code, code, s)
    check(dst)
    for x, off, n in zip(src, offs, sizes):
        assert torch.equal(dst[off:off + n], x)
    # (c) SGD (+ momentum) on guarded weights and momentum
    wdt, mdt = (api.F64, torch.float64) if dt == "f64" else (api.F32, torch.float32)
    w = torch.full((total,), -1234.5, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
    v = torch.full((total,), -1234.5, device="cuda", dtype=mdt)
    wguard = w.clone()
    g = [torch.randn(n, device="cuda").to(tdt) for n in sizes]
    api.sgd_update([(w[off:].data_ptr(), x.data_ptr(), v[off:].data_ptr(), n) for x, off, n in zip(g, offs, sizes)],
                   wdt, code, 0.1, 0.01, 0.9, s)
    torch.cuda.synchronize()
    assert torch.equal(w[mask], wguard[mask]) and torch.equal(v[mask], wguard.to(mdt)[mask])
    # (b) rank-order sum into a guarded output slice (one key at a time)
    out = guard.clone()
    for off, n in zip(offs, sizes):
        ins = [torch.randn(n, device="cuda").to(tdt) for _ in range(3)]
        api.sum_buffers([x.data_ptr() for x in ins], [out[off:].data_ptr()], n, code, s)
    check(out)
