"""Dump the SASS of cached NVRTC pass kernels (~/.cache/simdiag_b200_jit)
whose generated source contains every given substring.
  python tools/jit_sass.py OUT_PREFIX substring [substring ...]"""
import glob
import os
import struct
import subprocess
import sys

d = os.path.expanduser("~/.cache/simdiag_b200_jit")
prefix, subs = sys.argv[1], sys.argv[2:]
hits = []
for f in sorted(glob.glob(d + "/*.cubin"), key=os.path.getmtime, reverse=True):
    b = open(f, "rb").read()
    if not b.startswith(b"SDBJ1\n"):
        continue
    ln = struct.unpack("<Q", b[6:14])[0]
    ident = b[14:14 + ln].decode()
    if all(s in ident for s in subs):
        hits.append((f, ident, b[14 + ln:]))
print(f"{len(hits)} matching kernels")
for i, (f, ident, cub) in enumerate(hits[:1]):
    open(prefix + ".cubin", "wb").write(cub)
    open(prefix + ".src", "w").write(ident)
    sass = subprocess.run(["cuobjdump", "-sass", prefix + ".cubin"], capture_output=True, text=True).stdout
    open(prefix + ".sass", "w").write(sass)
    print(prefix + ".sass", sass.count("\n"), "lines")
