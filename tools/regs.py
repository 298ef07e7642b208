"""Registers / spills per apply kernel from a ptxas log: python tools/regs.py [LIBNAME]"""
import re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "libelas.so"
log = open(f"paper_2601_08374_b200/lib/{lib}.ptxas.log").read()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
    if cur and "apply" in cur and ("Used" in line or ("spill" in line and "0 bytes spill stores" not in line)):
        print(f"{cur:40s} {line.strip()[-90:]}")
