"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py gpurun_out/launches.csv "command" > profiles/x.md
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = r[ik].split("(")[0].replace("zolo::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    tot[name] += float(r[iv].replace(",", "")) * scale[r[iu]]
    cnt[name] += 1
T = sum(tot.values())
print(f"# ncu launch list: {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}\n")
print(f"{len(data)} launches, {T / 1e6:.1f} ms total GPU time (serialised, cold-cache replay: shares, not absolutes)\n")
print("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"| `{k}` | {cnt[k]} | {v / 1e6:.2f} | {100 * v / T:.1f}% | {v / cnt[k] / 1e3:.1f} |")
