"""Registers / spills / smem of the sweep-family kernels from a build log (ptxas -v)."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2401_06277_b200/build.log").read()
pat = re.compile(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n"
                 r"ptxas info\s+: Used (\d+) registers")
for name, st, ss, sl, reg in pat.findall(log):
    if any(k in name for k in ("vanka", "residual_strip", "boundary", "prolong")):
        print("%-60s regs %3s stack %3s spill st/ld %s/%s" % (name[:60], reg, st, ss, sl))
