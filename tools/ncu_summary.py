"""Summaries of ncu outputs for profiles/ (dev tooling).

  python tools/ncu_summary.py launches <launches.csv>        # per-kernel share of device time
  python tools/ncu_summary.py report <x.ncu-rep> [label]     # key metrics of a --set full capture
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Scheduler Statistics", "Active Warps Per Scheduler"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Instruction Statistics", "Executed Instructions"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Occupancy", "Achieved Occupancy"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except (ValueError, IndexError):
            continue
        name = re.sub(r"\(.*", "", r[ik])
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print("| share | launches | device ms | kernel |\n|---:|---:|---:|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if t / tot >= 0.0005:
            print(f"| {100 * t / tot:.2f}% | {c} | {t / 1e6:.2f} | `{k}` |")
    print(f"\ntotal device time of all captured launches: {tot / 1e6:.1f} ms")


def report(path, label=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    isec, iname, iunit, ival = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    kname = rows[1][h.index("Kernel Name")] if len(rows) > 1 else "?"
    got = {(r[isec], r[iname]): (r[ival], r[iunit]) for r in rows[1:] if len(r) > ival}
    print(f"### {label or path}\n\nkernel: `{kname}`\n\n| metric | value |\n|---|---:|")
    for key in KEYS:
        if key in got:
            v, u = got[key]
            print(f"| {key[1]} | {v} {u} |")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh, vv = rr[0], rr[2] if len(rr) > 2 else rr[1]
    st = []
    for k, x in zip(hh, vv):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("\nstall reasons (pc sampling): " + ", ".join(f"{k} {100 * x / tot:.1f}%" for x, k in sorted(st, reverse=True)[:6]))
    dram = {k: x for k, x in zip(hh, vv) if k in ("dram__bytes_read.sum", "dram__bytes_write.sum")}
    if dram:
        print("\nDRAM bytes: " + ", ".join(f"{k} = {v}" for k, v in dram.items()))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
