"""Registers / spills per kernel of libouro_b200 (ptxas -v), demangled short names.
python tools/regs.py [filter]"""
import re
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
out = subprocess.run(
    ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
     f"-I{ROOT}/include", "-Xptxas", "-v", "-c", f"{ROOT}/paper_2504_18211_b200/csrc/ouro_lib.cu", "-o", "/tmp/_regs.o"],
    capture_output=True, text=True).stderr
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
spill = 0
for line in out.splitlines():
    m = re.search(r"(?:Compiling entry function|Function properties for) '?(\S+?)'?( for|$)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(anonymous namespace\)::|ouro_dev::", "", name)
        name = re.sub(r"\(.*", "", name)
        if flt in name:
            print(f"{m.group(1):>4} regs  {spill:>4} B spilled  {name}")
        spill = 0
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        spill = int(m.group(1))
