"""Top source lines by warp-stall samples from an ncu report (--page source
with -lineinfo): `python scripts/ncu_hot_lines.py rep.ncu-rep [N]`."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = i
        break
h = rows[hdr]
si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
li = h.index("# Address") if "# Address" in h else (h.index("Line") if "Line" in h else 0)
acc = []
for r in rows[hdr + 1:]:
    if len(r) <= wi:
        continue
    try:
        acc.append((int(r[wi]), r[li], r[si][:110]))
    except ValueError:
        pass
tot = sum(a[0] for a in acc) or 1
for s, l, src in sorted(acc, reverse=True)[:top]:
    print(f"{100.0 * s / tot:5.1f}%  {l:>6}  {src}")
