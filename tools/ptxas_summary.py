"""Registers / spills of the step kernels from paper_2308_12698_b200/ptxas_info.txt."""
import re
import sys
from pathlib import Path

s = Path(__file__).resolve().parent.parent.joinpath("paper_2308_12698_b200", "ptxas_info.txt").read_text()
cur, spill = None, ("?", "?")
pat = sys.argv[1] if len(sys.argv) > 1 else "quad_step"
for line in s.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat in cur:
        name = re.search(r"(quad_step\w*?kernel|\w*kernel)I?L?b?(\d)?", cur)
        print(f"{re.sub(r'^_ZN.*?cu_\w{8}\d+', '', cur)[:40]:42s} regs={m.group(1):>4s} spill st/ld={spill}")
