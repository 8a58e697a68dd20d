"""Summarise registers / spills / smem per kernel from _lib/build.log."""
import os
import re
import sys

log = open(os.path.join(os.path.dirname(__file__), "..", "paper_2508_16121_b200", "_lib", "build.log")).read()
pat = re.compile(r"Compiling entry function '(\S+)'.*?\n.*?\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers", re.S)
flt = sys.argv[1] if len(sys.argv) > 1 else ""
for m in pat.finditer(log):
    name, stack, ss, sl, regs = m.groups()
    if flt in name:
        print(f"{regs:>4} regs  spill {ss:>4}/{sl:<4} stack {stack:>4}  {name}")
