"""Registers / spills per kernel of one csrc file (ptxas -v), demangled.

    python scripts/ptxas_regs.py render.cu [name-regex] [-Dextra ...]
"""
import os
import re
import subprocess
import sys

src = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
extra = sys.argv[3:]
csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2202_05628_b200", "csrc")
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                      "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I",
                      os.path.join(csrc, "..", "..", "include"), "-I", csrc, *extra, "-c",
                      os.path.join(csrc, src), "-o", f"/tmp/ptxas_{os.getpid()}.o"],
                     capture_output=True, text=True)
name, spill = None, ("0", "0", "0")
for line in (out.stdout + out.stderr).splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and name and re.search(pat, name):
        print(f"{m.group(1):>4} regs  stack {spill[0]:>4}  spill st/ld {spill[1]}/{spill[2]}  {name[:100]}")
    if "error" in line:
        print(line)
