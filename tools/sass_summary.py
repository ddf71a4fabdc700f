#!/usr/bin/env python
"""Instruction mix of the hot kernels from the built library's SASS
(cuobjdump -sass), for profiles/: memory opcodes with their qualifiers
(LDG/STG = explicit global, .EF = evict-first streaming, .128 = 16-B vectors,
LD/ST = generic), plus registers / stack per kernel (cuobjdump -res-usage).

  python tools/sass_summary.py > profiles/r2_sass_summary.txt
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_1802_06949_b200" / "lib" / "libcollsim_b200.so"
# (label, regex on the mangled name): the fp32 / momentum instantiations the bench runs
KERNELS = [
    ("(a) pack_tab_kernel f32->f32", r"pack_tab_kernelILi1ELi1EE"),
    ("(b) sum_kernel f32 M=8", r"sum_kernelILi1ELi8EE"),
    ("(c) sgd_tab_kernel f32 momentum", r"sgd_tab_kernelILi1ELi1ELb1EE"),
    ("(a)+(c) pack_sgd_tab_kernel f32 momentum (one rank)", r"pack_sgd_tab_kernelILi1ELi1ELi1ELb1ELi1EE"),
    ("(b)+(c) p2p_allreduce_kernel f32 update momentum M=4", r"p2p_allreduce_kernelILi1ELi1ELb1ELb1ELi4ELb0EE"),
    ("(b)+(c) p2p_zero_kernel f32 momentum M=4 (ZeRO-1)", r"p2p_zero_kernelILi1ELi1ELb1ELi4EE"),
]
MEM = re.compile(r"\b((?:LDG|STG|LD|ST|LDS|STS|ATOMG|RED|LDGSTS|UBLKCP|UTMALDG|SYNCS)\.[A-Z0-9._]*|(?:LDG|STG|LD|ST)\b)")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", str(LIB)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    out = [f"# SASS memory-instruction mix, {LIB.name} (sm_100a)", ""]
    for label, pat in KERNELS:
        body = next((f for f in funcs if re.search(pat, f.split("\n", 1)[0])), None)
        if body is None:
            out.append(f"{label}: not found")
            continue
        name = body.split("\n", 1)[0].strip()
        m = re.search(re.escape(name) + r".*?\n\s*(REG:\d+ STACK:\d+ SHARED:\d+)", res, re.S)
        ops = Counter(MEM.findall(body))
        total = sum(1 for line in body.splitlines() if re.match(r"\s*/\*[0-9a-f]{4}\*/", line))
        out.append(f"{label}\n  {name}\n  {m.group(1) if m else ''}  instructions: {total}")
        for op, n in sorted(ops.items()):
            out.append(f"    {op:28s} {n}")
        out.append("")
    sys.stdout.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
