"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
  python tools/launch_summary.py gpurun_out/launches.csv [--rounds KERNEL]  (per-launch times of one kernel)"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    rows = list(csv.reader(l for l in f if l.startswith('"')))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    try:
        d.setdefault(r[ki].split("(")[0].replace("immx_dev::<unnamed>::", ""), []).append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:56]:56s} n={len(v):5d} sum={sum(v) / 1e6:9.3f} ms avg={sum(v) / len(v) / 1e3:9.1f} us {100 * sum(v) / tot:5.1f}%")
if len(sys.argv) > 3 and sys.argv[2] == "--rounds":
    v = next(x for k, x in d.items() if sys.argv[3] in k)
    print(sys.argv[3], " ".join(f"{x / 1e3:.0f}" for x in v))
