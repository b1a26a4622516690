"""Spill (STL/LDL) counts per source line of one kernel in a cubin: python tools/spills.py x.cubin [kernel-substring]"""
import collections
import re
import subprocess
import sys

sass = subprocess.run(["nvdisasm", "-g", "-c", sys.argv[1]], capture_output=True, text=True).stdout.split("\n")
pat = sys.argv[2] if len(sys.argv) > 2 else "ILi1024ELi1024"
cur = fn = None
cnt = collections.Counter()
for L in sass:
    m = re.search(r"\.text\.(\S+):", L)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', L)
    if m:
        cur = (m.group(1), int(m.group(2)))
    if fn and pat in fn and re.search(r"\b(STL|LDL)\b", L):
        cnt[(cur, "STL" if "STL" in L else "LDL")] += 1
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:20]:
    print(v, k)
