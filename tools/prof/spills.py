"""Registers / spills of every K2 slot-kernel instantiation from the ptxas log."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else
           "paper_2605_07391_b200/csrc/build/kernels.ptxas.log").read()
for b in re.split(r"ptxas info    : Compiling entry function '", log)[1:]:
    name = b.split("'")[0]
    pat = sys.argv[2] if len(sys.argv) > 2 else "spmv_slot_kernel"
    if pat not in name:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
    r = re.search(r"Used (\d+) registers", b)
    short = re.search(pat + r"I(\w+?)EEv", name)
    print(short.group(1) if short else name[:80], "regs", r.group(1), "spill st/ld", m.groups())
