"""Per-warp-group instruction attribution for the CTA sampler (dev tooling).
  python tools/per_group.py <rep> <cubin> <kernel-substr> <edges> [G] [NW]"""
import re
import subprocess
import sys

rep, cubin, kern, edges = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
G = int(sys.argv[5]) if len(sys.argv) > 5 else 1024
NW = int(sys.argv[6]) if len(sys.argv) > 6 else 8
out = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, cubin, kern, "70"], capture_output=True,
                     text=True).stdout.split("\n")
tot = int(out[0].split()[-1])
wg = edges / G * NW
src = {}
for f in ("sampler.cu", "common.cuh"):
    src[f] = open(f"paper_2208_00613_b200/csrc/{f}").read().split("\n")
print(f"instructions per warp-group ({G // NW} edges/warp): {tot / wg:.1f}")
for l in out[1:]:
    m = re.match(r"(\S+)\s+exec\s+([\d.]+)%\s+stall\s+([\d.]+)%", l)
    if not m:
        continue
    f, p, s = m.group(1), float(m.group(2)), float(m.group(3))
    name, _, ln = f.partition(":")
    txt = src[name][int(ln) - 1].strip()[:72] if name in src and ln.isdigit() else ""
    print(f"{f:26s} {p * tot / 100 / wg:6.1f} instr  stall {s:4.1f}%  {txt}")
