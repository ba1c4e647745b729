"""Per-source-line warp-stall samples from an ncu report (source page,
cuda+sass interleaved): prints the top lines with their share of samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, file_ = {}, None
cur = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        file_ = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:  # a source line row
        cur = (file_, r[0], r[1].strip()[:90])
        continue
    try:
        s = float(r[4] or 0)
    except (ValueError, IndexError):
        continue
    if cur:
        agg[cur] = agg.get(cur, 0.0) + s
tot = sum(agg.values()) or 1.0
for (f, ln, src), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln}  {src}")
