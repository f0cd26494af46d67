"""Map an ncu source-page CSV (SASS addresses) onto CUDA source lines via nvdisasm line info.

  python tools/ncu_lines.py <report.ncu-rep> <cubin> <kernel-mangled-substring> [top] [section]
Prints instructions executed and stall samples per source line (test/dev tooling).  A report
with several launches lists one section per launch; `section` picks one (default: the last)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
section = int(sys.argv[5]) if len(sys.argv) > 5 else -1
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith("//---") and kname in l)
end = next((i for i in range(start + 1, len(sass)) if sass[i].startswith("//---")), len(sass))
cur, off2line = None, {}
for l in sass[start:end]:
    m = re.search(r'//## File ".*?/([\w.]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m2:
        off2line[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
s0 = starts[section]
s1 = next((i for i in starts if i > s0), len(rows))
rows = rows[s0:s1]
h = rows[1]
ia, ie, iss = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(rows[2][ia], 16)
ex, st = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= max(ia, ie, iss) or not r[ia].startswith("0x"):
        continue
    ln = off2line.get(int(r[ia], 16) - base, "?")
    ex[ln] += int(r[ie])
    st[ln] += float(r[iss])
tot, tots = sum(ex.values()), sum(st.values())
print(f"instructions executed: {tot}")
for ln, c in ex.most_common(top):
    print(f"{ln:26s} exec {100 * c / tot:5.1f}%  stall {100 * st[ln] / tots:5.1f}%")
print("-- by stall")
for ln, c in st.most_common(top // 2):
    print(f"{ln:26s} exec {100 * ex[ln] / tot:5.1f}%  stall {100 * c / tots:5.1f}%")
