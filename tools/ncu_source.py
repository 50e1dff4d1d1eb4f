"""Aggregate ncu --page source per CUDA source line (instructions executed, stall samples).
usage: ncu_source.py report.ncu-rep [top]   (measurement tool)"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
extra = sys.argv[3:] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", path, *extra, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = ""
data = []
hdr = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        col = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        st = float(r[4] or 0)
        ins = float(r[7] or 0)
    except ValueError:
        continue
    data.append((st, ins, f"{fname}:{r[0]}", r[1][:100]))
tot_s = sum(d[0] for d in data) or 1
tot_i = sum(d[1] for d in data) or 1
print(f"total stall samples {tot_s:.0f}, warp-instructions {tot_i:.0f}")
for st, ins, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{100*st/tot_s:5.1f}% stall {100*ins/tot_i:5.1f}% inst  {ln:>22} {src}")
