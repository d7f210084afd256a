"""Per-kernel registers / spills from `nvcc -Xptxas -v` output on stdin."""
import re
import sys
cur = None
for ln in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", ln) or re.search(r"Function properties for (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur and (int(m.group(1)) or int(m.group(2))):
        print(f"SPILL {cur}: {m.group(1)} st / {m.group(2)} ld")
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur:
        print(f"{m.group(1):>4} regs  {cur}")
