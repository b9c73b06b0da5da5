"""Attribute ncu per-SASS executed instructions / stall samples to CUDA source lines.

    python scripts/line_profile.py <ncu sass csv> <nvdisasm -g -c output> <mangled-name-substring>

The csv is `ncu -i rep --page source --csv --print-source sass`; the disassembly comes from the
locally built cubin of the same source (`cuobjdump -xelf all kernels.cu.o; nvdisasm -g -c ...`)."""
import csv
import os
import re
import sys
from collections import defaultdict

csv_path, sass_path, name = sys.argv[1:4]
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
data = rows[2:]
iexe = hdr.index("Instructions Executed")
samp = hdr.index("Warp Stall Sampling (All Samples)")
addr0 = int(data[0][0], 16)
per_off = {int(r[0], 16) - addr0: (float(r[iexe] or 0), float(r[samp] or 0), r[1].strip()) for r in data}

lines = open(sass_path).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith("//-----") and name in l)
cur = None
off2line = {}
for l in lines[start + 1:]:
    if l.startswith("//-----"):
        break
    m = re.search(r'File "([^"]*)", line (\d+)', l)
    if "//##" in l and m:
        f = os.path.basename(m.group(1))
        cur = int(m.group(2)) if f == "kernels.cu" else f"{f}:{m.group(2)}"
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
inst = defaultdict(float)
stall = defaultdict(float)
for off, (n, s, txt) in per_off.items():
    ln = off2line.get(off)
    inst[ln] += n
    stall[ln] += s
tot = sum(inst.values())
tots = sum(stall.values())
print(f"total warp-inst {tot:.4g}, samples {tots:.0f}, matched offsets {sum(1 for o in per_off if o in off2line)}/{len(per_off)}")
for ln in sorted(inst, key=lambda k: -inst[k])[:45]:
    print(f"line {ln}: {100*inst[ln]/tot:5.1f}% inst  {100*stall[ln]/max(1,tots):5.1f}% stall")

# region summary when REGIONS="name:lo-hi,..." is given in the environment
import os
if os.environ.get("REGIONS"):
    for spec in os.environ["REGIONS"].split(","):
        nm, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        i = sum(v for k, v in inst.items() if isinstance(k, int) and lo <= k <= hi)
        s = sum(v for k, v in stall.items() if isinstance(k, int) and lo <= k <= hi)
        print(f"region {nm:10s} {100*i/tot:5.1f}% inst {100*s/max(1,tots):5.1f}% stall")
