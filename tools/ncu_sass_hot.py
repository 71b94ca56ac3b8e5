"""Per-SASS-instruction execution counts and stall samples of one kernel from an ncu report's
source page (ncu -i REP --page source --csv --print-source sass ...), printed in address order
with the warp-instruction count, active threads and samples: where the issue slots of a loop go.

python tools/ncu_sass_hot.py REP KERNEL_REGEX [LAUNCH_SKIP] [MIN_PERCENT]"""
import csv
import subprocess
import sys

rep, regex = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
minp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.05
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{regex}", "--launch-skip", skip, "--launch-count", "1"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
print(lines[0][:160])
rows = [r for r in csv.reader(lines[1:]) if len(r) > 10]
h = rows[0]
ix = {k: h.index(k) for k in ("Address", "Source", "Instructions Executed", "Avg. Threads Executed", "# Samples")}
rows = [h] + [r for r in rows[1:] if r[ix["Instructions Executed"]].isdigit()]
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in rows[1:])
print(f"total warp instructions {tot}")
for r in rows[1:]:
    n = int(r[ix["Instructions Executed"]] or 0)
    if n >= minp * tot / 100:
        print(f"{r[ix['Address']][-5:]} {n:>11} {r[ix['Avg. Threads Executed']]:>5} {r[ix['# Samples']]:>6}  "
              f"{r[ix['Source']].strip()[:70]}")
