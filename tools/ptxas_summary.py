"""Registers / spills / stack per hop_kernel and pack_kernel instantiation
from an nvcc -Xptxas -v log (build/lbcu/dslash.cu.o.ptxas.txt, written by
`python -c "from paper_1401_3733_b200 import _build; _build.build(verbose=True)"`).

    python tools/ptxas_summary.py build/lbcu/dslash.cu.o.ptxas.txt > profiles/<tag>_ptxas_dslash.txt
"""
import re
import subprocess
import sys

FMT = {0: "full", 1: "su2", 2: "r12", 3: "as4", 4: "as4r", 5: "r10"}
EPI = {0: "store", 1: "store+norm", 2: "cg"}


def main(path):
    text = open(path).read()
    blocks = re.split(r"ptxas info\s+: Compiling entry function '", text)[1:]
    rows = []
    for b in blocks:
        name = b.split("'", 1)[0]
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        if "hop_kernel" not in dem and "pack_kernel" not in dem:
            continue
        regs = re.search(r"Used (\d+) registers", b)
        spill = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
        stack = re.search(r"(\d+) bytes stack frame", b)
        m = re.search(r"(hop_kernel|pack_kernel)<([^>]*)>", dem)
        args = [a.strip() for a in m.group(2).split(",")] if m else []
        rows.append((m.group(1) if m else dem, args, regs and int(regs.group(1)),
                     stack and int(stack.group(1)), spill and int(spill.group(1)), spill and int(spill.group(2))))
    print("kernel        D  real fmt   bnd epi         minb zs  regs stack spill_st spill_ld")
    for k, a, r, st, ss, sl in sorted(rows, key=lambda x: (x[0], x[1])):
        if k == "hop_kernel" and len(a) == 7:
            D, real, fmt, bnd, epi, minb, zs = a
            fmt_s = FMT.get(int(fmt), fmt)
            print(f"{k:12s} {D:>2s} {real:>5s} {fmt_s:5s} {bnd:>4s} {EPI.get(int(epi), epi):11s} {minb:>4s} "
                  f"{zs:>3s} {r:5d} {st:5d} {ss:8d} {sl:8d}")
        else:
            print(f"{k:12s} {','.join(a):40s} {r:5d} {st:5d} {ss:8d} {sl:8d}")


if __name__ == "__main__":
    main(sys.argv[1])
