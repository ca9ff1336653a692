"""Registers / spills per kernel from an `nvcc -Xptxas -v` log (stdin); argv[1] = name filter."""
import re, subprocess, sys
flt = sys.argv[1] if len(sys.argv) > 1 else ""
txt = sys.stdin.read()
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur and "spill" in line:
        spill = line.strip()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(.*", "", name)
        if flt in name:
            print(f"{m.group(1):>4} regs  {spill:60s} {name}")
        cur = None
