"""Compile kernels.cu with -Xptxas -v and print one line per stencil instantiation."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2202_11819_b200/csrc/kernels.cu"
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                      "-Xptxas", "-v", "-c", src, "-o", "/tmp/kernels_regs.o"], capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        t = re.search(r"TileILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E", name)
        cur = f"TX={t.group(1)} NCW={t.group(2)} RPW={t.group(3)} NS={t.group(4)} MINB={t.group(5)} MAP={t.group(6)}" if t else name[:40]
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        stack, sst, sld = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if "TX=" in cur:
            print(f"{cur:40s} regs={m.group(1):4s} stack={stack:4s} spill={sst}/{sld}")
        cur = None
