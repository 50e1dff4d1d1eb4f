"""Print the key sections of an ncu report (measurement tool).  python tools/ncu_details.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Occupancy", "Launch Statistics", "Scheduler Statistics",
            "Warp State Statistics", "Memory Workload Analysis", "Compute Workload Analysis")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
si, mi, vi, ui, ki = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value", "Metric Unit", "Kernel Name"))
for x in r[1:]:
    if x[si] in SECTIONS:
        print(f"{x[ki][:24]:24s} | {x[si][:18]:18s} | {x[mi]:45s} {x[vi]} {x[ui]}")
