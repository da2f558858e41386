"""Hot lines of one kernel in an ncu report: warp-stall samples and executed
instructions per source (or SASS) line.
    python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [cuda|sass] [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
mode = sys.argv[3] if len(sys.argv) > 3 else "cuda"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", mode],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(('"Address"', '"Line"', '"#"')))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_i = h.index("Instructions Executed")
i_src = h.index("Source")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


body = [r for r in rows[1:] if len(r) > max(i_s, i_i)]
ts = sum(num(r[i_s]) for r in body) or 1.0
ti = sum(num(r[i_i]) for r in body) or 1.0
print(f"samples {ts:.0f}  instructions {ti:.0f}")
for r in sorted(body, key=lambda r: -num(r[i_s]))[:n]:
    print(f"{num(r[i_s]) / ts * 100:5.1f}% stall {num(r[i_i]) / ti * 100:5.1f}% inst | "
          f"{r[0][-6:]:>6} {r[i_src].strip()[:95]}")
