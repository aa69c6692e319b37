"""Per-source-line instruction counts of two ncu reports of the same kernel
source (e.g. the PageRank and plain SpMV instantiations), largest
differences first: `python scripts/ncu_line_diff.py a.ncu-rep b.ncu-rep`."""
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    d, f, cols = {}, "", None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            f = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Line No":
            cols = r
        elif cols and len(r) == len(cols):
            try:
                ie = int(r[cols.index("Instructions Executed")])
                st = int(r[cols.index("Warp Stall Sampling (All Samples)")])
            except ValueError:
                continue
            k = (f, r[0], r[1].strip()[:80])
            a = d.setdefault(k, [0, 0])
            a[0] += ie
            a[1] += st
    return d


a, b = load(sys.argv[1]), load(sys.argv[2])
print("instructions", sum(v[0] for v in a.values()), sum(v[0] for v in b.values()))
print("stall samples", sum(v[1] for v in a.values()), sum(v[1] for v in b.values()))
rows = sorted(((a.get(k, [0, 0])[0] - b.get(k, [0, 0])[0]), k) for k in set(a) | set(b))
for dv, k in rows[::-1][:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{dv:>12} {a.get(k, [0, 0])[1]:>7} {b.get(k, [0, 0])[1]:>7}  {k[0]}:{k[1]} {k[2]}")
