"""Registers / stack per kernel instantiation of a built library:
python tools/prof/res_usage.py lib.so [name-substring]"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-res-usage", sys.argv[1]], capture_output=True,
                     text=True).stdout.splitlines()
key = sys.argv[2] if len(sys.argv) > 2 else ""
fn = None
for line in out:
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and fn and key in fn:
        dem = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"mbx::\(anonymous namespace\)::", "", dem)
        print(f"REG {m.group(1):>3} STACK {m.group(2):>3}  {dem[:110]}")
        fn = None
