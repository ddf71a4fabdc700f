"""Build the native library in-tree: paper_1802_06949_b200/lib/libcollsim_b200.so.

Kernels are compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``),
host runtime (engine / ledger / transport / kvstore / C ABI) as C++20.  The CUDA
runtime is linked statically; NCCL is the venv's libnccl.so.2 (2.28.9, the one
torch loads), found through an rpath.  ``python -m paper_1802_06949_b200.build``
rebuilds whatever is stale.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "lib" / "libcollsim_b200.so"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")


def _nccl_dir() -> Path:
    site = Path(sysconfig.get_paths()["purelib"])
    d = site / "nvidia" / "nccl"
    if not (d / "include" / "nccl.h").exists():
        raise RuntimeError(f"NCCL headers not found under {d}")
    return d


ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _compile_cmd(src: Path, obj: Path, nccl: Path):
    inc = [f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{nccl / 'include'}", f"-I{CUDA / 'include'}"]
    if src.suffix == ".cu":
        return [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++20", "--expt-relaxed-constexpr",
                "-Xcompiler", "-fPIC,-pthread", "-diag-suppress", "177", *inc,
                "-c", str(src), "-o", str(obj)]
    return ["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-pthread", "-Wall", "-Wno-unused-function",
            *inc, "-c", str(src), "-o", str(obj)]


def build(verbose: bool = False, force: bool = False) -> Path:
    nccl = _nccl_dir()
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.hpp")) + list((ROOT / "include").glob("*.h"))
    newest_header = max((h.stat().st_mtime for h in headers), default=0)
    jobs = []
    objs = []
    for src in _sources():
        obj = OBJ / (src.name + ".o")
        objs.append(obj)
        stale = force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_header)
        if stale:
            jobs.append((src, obj))

    def run(job):
        src, obj = job
        cmd = _compile_cmd(src, obj, nccl)
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {src.name}\n{r.stdout}\n{r.stderr}")
        return src.name

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for name in ex.map(run, jobs):
                if verbose:
                    print(f"  built {name}", flush=True)
    if jobs or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
                f"-L{nccl / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl / 'lib'}",
                "-lrt", "-lpthread"]
        if verbose:
            print(" ".join(link), flush=True)
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Test infrastructure: the C restatement, plus the reference itself when
    its sources are present (this container only; the GPU box uses the
    prebuilt oracle/_ref)."""
    odir = ROOT / "oracle"
    targets = ["all"]
    if Path("/root/reference/proj/core/src").exists():
        targets.append("ref")
    r = subprocess.run(["make", "-s", "-j8", "-C", str(odir), *targets], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"oracle built: {targets}")


if __name__ == "__main__":
    v = "-v" in sys.argv
    print(build(verbose=v, force="--force" in sys.argv))
    build_oracle(verbose=v)
