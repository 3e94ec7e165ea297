"""Opcode mix of one kernel's SASS (cuobjdump -sass LIB), optionally between two
labels: python tools/sass_mix.py LIB KERNEL_SUBSTRING"""
import collections
import re
import subprocess
import sys

lib, name = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
body = next(f for f in funcs if f.split("\n")[0].strip().find(name) >= 0)
ops = collections.Counter()
n = 0
for line in body.split("\n"):
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m:
        ops[m.group(2).split(".")[0]] += 1
        n += 1
print("total", n)
for k, v in ops.most_common(30):
    print("%-10s %5d" % (k, v))
