"""Summarise an ncu report's SASS source page: warp-stall samples per
opcode and the hottest instructions (ncu -i REP --page source --csv
--print-source sass)."""
import collections
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    # first line: kernel name; then the header
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
    return rows


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = load(rep)
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    by_op = collections.Counter()
    reasons = collections.Counter()
    rkeys = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
    for r in rows:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        by_op[op.split(".")[0]] += s
        for k in rkeys:
            reasons[k] += int(r[k] or 0)
    print(f"total samples {tot}")
    print("by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in reasons.most_common(10)))
    print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in by_op.most_common(15)))
    hot = sorted(enumerate(rows), key=lambda t: -int(t[1]["Warp Stall Sampling (All Samples)"] or 0))
    for i, r in hot[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        rs = sorted(((int(r[k] or 0), k[6:]) for k in rkeys), reverse=True)[:3]
        print(f"{i:5d} {s / tot:6.2%}  {r['Source'].strip()[:60]:60s} "
              + " ".join(f"{n}:{v}" for v, n in rs if v))


if __name__ == "__main__":
    main()
