"""Summarise an `ncu --metrics gpu__time_duration.sum ... --csv --log-file X` launch list
(measurement tool): per-kernel launch count, total time and share; optional per-launch
series of one kernel.   python tools/launch_summary.py launches.csv [kernel-substring]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, mi, vi, idi, gi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
    per, names, grids = collections.defaultdict(dict), {}, {}
    for r in data:
        per[int(r[idi])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[idi])] = r[ki]
        grids[int(r[idi])] = r[gi]
    return per, names, grids


def main():
    per, names, grids = load(sys.argv[1])
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for i, m in per.items():
        n = names[i].split("(")[0]
        tot[n] += m.get("gpu__time_duration.sum", 0.0)
        cnt[n] += 1
    T = sum(tot.values())
    print("kernel,launches,total_us,share")
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f'"{n}",{cnt[n]},{v / 1e3:.1f},{v / T:.4f}')
    print(f"# total {T / 1e6:.3f} ms over {len(per)} launches")
    if len(sys.argv) > 2:
        for i in sorted(per):
            if sys.argv[2] in names[i]:
                print(i, grids[i], " ".join(f"{k.split('.')[0]}={v:.4g}" for k, v in per[i].items()))


if __name__ == "__main__":
    main()
