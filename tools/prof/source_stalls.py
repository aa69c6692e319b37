"""Warp-stall samples of an ncu report per CUDA source line (needs
--import-source on and -lineinfo): ncu -i REP --page source --csv
--print-source cuda,sass, aggregated over each line's SASS.
python tools/prof/source_stalls.py REP [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if len(sys.argv) > 3:
        cmd += ["-k", "regex:" + sys.argv[3]]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # rows: ["Line No","Source","Address","Source", metrics...]; a line row
    # carries the line number, its SASS rows follow with an empty line no.
    hdr = None
    lines = {}
    reasons = {}
    cur = None
    fname = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6:
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip())
            try:
                lines[cur] = lines.get(cur, 0) + int(r[4] or 0)
                rs = reasons.setdefault(cur, {})
                for k, v in zip(hdr, r):
                    if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "-"):
                        rs[k[6:]] = rs.get(k[6:], 0) + int(v)
            except ValueError:
                pass
    tot = sum(lines.values()) or 1
    for (f, ln, src), s in sorted(lines.items(), key=lambda t: -t[1])[:top]:
        rs = sorted(reasons.get((f, ln, src), {}).items(), key=lambda t: -t[1])[:3]
        why = " ".join(f"{k}:{v / max(s, 1):.0%}" for k, v in rs if v)
        print(f"{s / tot:6.2%} {f}:{ln:<5d} {src[:70]:70s} {why}")


if __name__ == "__main__":
    main()
