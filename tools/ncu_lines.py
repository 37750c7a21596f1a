"""Per-source-line instruction counts and stall samples of one ncu launch."""
import csv
import io
import subprocess
import sys

rep, launch = sys.argv[1], sys.argv[2]
amps = float(sys.argv[3]) if len(sys.argv) > 3 else 2.0 ** 28
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "--launch-skip",
                      launch, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Instructions Executed" in r)
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) > iE and r[0] and r[2] == "-":
        try:
            lines.append((int(r[iE]), int(r[iW]), r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(x[0] for x in lines)
totw = sum(x[1] for x in lines)
print(f"thread-instr per amp: {tot * 32 / amps:.1f}")
key = 1 if len(sys.argv) > 4 and sys.argv[4] == "stall" else 0
for e, w, ln, src in sorted(lines, key=lambda x: -x[key])[:30]:
    print(f"{ln:>4} {e * 32 / amps:6.2f}/amp {100 * w / max(1, totw):5.1f}%stall  {src}")
