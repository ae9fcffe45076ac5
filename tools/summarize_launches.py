"""Summarise an ncu launch-list CSV (gpu__time_duration.sum + dram bytes per launch) into a
markdown table: python tools/summarize_launches.py launches.csv [title]."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for d in data:
    k = d["Kernel Name"].split("(")[0]
    m, v = d["Metric Name"], float(d["Metric Value"].replace(",", ""))
    a = agg[k]
    if m == "gpu__time_duration.sum":
        a[0] += 1
        a[1] += v
    elif m == "dram__bytes_read.sum":
        a[2] += v
    elif m == "dram__bytes_write.sum":
        a[3] += v
tot = sum(a[1] for a in agg.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else 'ncu launch list'}\n")
print("| kernel | launches | total s | share | DRAM read TB | DRAM write TB | per-launch read+write GB |")
print("|---|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {a[0]} | {a[1] / 1e9:.3f} | {100 * a[1] / tot:.1f} % | {a[2] / 1e12:.3f} | {a[3] / 1e12:.3f} | "
          f"{(a[2] + a[3]) / max(a[0], 1) / 1e9:.2f} |")
print(f"\nTotal {tot / 1e9:.2f} s (cold-cache, serialised: compare shares, not absolutes).")
