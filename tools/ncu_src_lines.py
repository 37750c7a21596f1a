"""ncu per-line instruction/stall table mapped onto pass_device.cuh (for
NVRTC-compiled kernels whose source ncu cannot open):
    python tools/ncu_src_lines.py REPORT LAUNCH [amps] [stall]"""
import os
import re
import subprocess
import sys

rep, launch = sys.argv[1], sys.argv[2]
amps = sys.argv[3] if len(sys.argv) > 3 else str(2 ** 28)
key = sys.argv[4] if len(sys.argv) > 4 else ""
here = os.path.dirname(os.path.abspath(__file__))
out = subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, launch, amps] + ([key] if key else []),
                     capture_output=True, text=True).stdout
src = open(os.path.join(here, "..", "paper_2206_11664_b200", "csrc", "cuda", "pass_device.cuh")).read().split("\n")
for line in out.splitlines():
    m = re.match(r"\s*(\d+)\s+([\d.]+)/amp\s+([\d.]+)%stall", line)
    if m:
        n = int(m.group(1))
        txt = src[n - 1].strip()[:90] if n <= len(src) else "?"
        print(f"{n:4d} {m.group(2):>6}/amp {m.group(3):>5}%  {txt}")
    else:
        print(line)
