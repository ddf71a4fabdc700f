"""numpy face of the CPU oracle (oracle/oracle.c) and of the compiled reference
(oracle/_ref/libcollsim_ref.so).  TEST INFRASTRUCTURE ONLY: the checker, never
the thing measured or shipped."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "_build" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libcollsim_ref.so"


def _load_oracle() -> C.CDLL:
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "all"], check=True)
    lib = C.CDLL(str(ORACLE_SO))
    lib.or_mix_seed.restype = C.c_uint64
    lib.or_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.or_random_uniform.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
    lib.or_random_uniform_f32.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
    lib.or_f32_to_bf16_array.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    lib.or_bf16_to_f32_array.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    for n in ("or_rank_order_sum_f64", "or_rank_order_sum_f32", "or_rank_order_sum_bf16"):
        getattr(lib, n).argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
    for n in ("or_sgd_update_f64", "or_sgd_update_f32"):
        getattr(lib, n).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                    C.c_double, C.c_double]
    lib.or_synth_expect.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                    C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int]
    return lib


O = _load_oracle()


def ref_lib() -> C.CDLL | None:
    """The reference itself, when oracle/_ref was built (this container, or
    shipped to the GPU box as a prebuilt .so)."""
    if not REF_SO.exists():
        return None
    lib = C.CDLL(str(REF_SO))
    lib.ref_mix_seed.restype = C.c_uint64
    lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.ref_random_uniform.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
    lib.ref_allreduce.argtypes = [C.c_int, C.c_int64, C.c_void_p]
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_train_steps.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_char_p]
    lib.ref_run_scenario.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_uint64, C.c_char_p, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
    lib.ref_bench.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                              C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p]
    return lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def mix_seed(seed: int, salt: int) -> int:
    return int(O.or_mix_seed(seed, salt))


def random_uniform(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    O.or_random_uniform(_p(out), n, seed)
    return out


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    O.or_f32_to_bf16_array(_p(x), _p(out), x.size)
    return out


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    out = np.empty(h.shape, dtype=np.float32)
    O.or_bf16_to_f32_array(_p(h), _p(out), h.size)
    return out


def _ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def rank_order_sum(arrs: list[np.ndarray], kind: str = "f64") -> np.ndarray:
    """collective.cpp:228-236 restated; kind f64 | f32 | bf16 (uint16 bit arrays)."""
    arrs = [np.ascontiguousarray(a) for a in arrs]
    n = arrs[0].size
    out = np.empty_like(arrs[0])
    fn = {"f64": O.or_rank_order_sum_f64, "f32": O.or_rank_order_sum_f32,
          "bf16": O.or_rank_order_sum_bf16}[kind]
    fn(_ptr_array(arrs), len(arrs), _p(out), n)
    return out


def sgd_update(w: np.ndarray, g: np.ndarray, lr: float, rescale: float, momentum: float = 0.0,
               mom: np.ndarray | None = None, kind: str = "f64"):
    """model.cpp:17-27 restated (+ MXNet momentum); returns (w_new, mom_new)."""
    w = np.array(w, copy=True)
    g = np.ascontiguousarray(g)
    m = None if mom is None else np.array(mom, copy=True)
    fn = O.or_sgd_update_f64 if kind == "f64" else O.or_sgd_update_f32
    fn(_p(w), _p(g), _p(m) if m is not None else None, w.size, lr, rescale, momentum)
    return w, m


DT = {"f64": 0, "f32": 1, "bf16": 2}


def synth_expect(sizes, ranks: int, steps: int, *, wdt: str = "f32", gdt: str = "f32", cdt: str | None = None,
                 lr: float = 0.1, rescale: float = 1.0 / 64, momentum: float = 0.0, seed_base: int = 1000,
                 ref64: bool = True, threads: int = 0, keys=None):
    """Expected weights of the synthetic model (csrc/trainer.cpp SynthModel)
    after `steps` BACKWARD|COMM steps with the fused pull_update, every rank
    (oracle.c or_synth_expect).  keys: indices to check (default all).
    Returns (w in wdt, fp64 restatement or None, per-element tolerance scale
    or None), the selected keys concatenated."""
    import os
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    ids = None if keys is None else np.ascontiguousarray(keys, dtype=np.int32)
    total = int(sizes.sum() if ids is None else sizes[ids].sum())
    w = np.empty(total, dtype=np.float64 if wdt == "f64" else np.float32)
    r64 = np.empty(total, dtype=np.float64) if ref64 else None
    sc = np.empty(total, dtype=np.float64) if ref64 else None
    rc = O.or_synth_expect(DT[wdt], DT[gdt], DT[cdt or gdt], _p(sizes), len(sizes),
                           _p(ids) if ids is not None else None, 0 if ids is None else len(ids), ranks, steps,
                           seed_base, lr, rescale, momentum, _p(w), _p(r64) if ref64 else None,
                           _p(sc) if ref64 else None, threads or (os.cpu_count() or 1))
    if rc != 0:
        raise RuntimeError("or_synth_expect failed")
    return w, r64, sc
