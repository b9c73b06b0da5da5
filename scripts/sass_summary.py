"""Summarise an ncu report's SASS source page: executed instructions and stall samples per opcode."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rd = csv.reader(lines[start:])
h = next(rd)
ci = h.index("Instructions Executed"); cs = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source")
ex = collections.Counter(); st = collections.Counter(); tot_ex = tot_st = 0
for r in rd:
    if len(r) <= ci or not r[ci].replace('.', '').isdigit():
        continue
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"):
        op = r[src].split()[1]
    op = op.split(".")[0]
    e = float(r[ci]); s = float(r[cs] or 0)
    ex[op] += e; st[op] += s; tot_ex += e; tot_st += s
print(f"total warp-instructions {tot_ex:.3e}, stall samples {tot_st:.0f}")
for op, e in ex.most_common(25):
    print(f"{op:10s} {e/tot_ex*100:6.2f}% inst   {st[op]/max(tot_st,1)*100:6.2f}% stall")
