"""Summarise an ncu report's SASS source page: instructions executed per opcode class and the
hottest instructions by warp-stall samples.   python sass_hot.py report.ncu-rep [topN]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
which = int(__import__("os").environ.get("RESULT", "0"))  # which kernel result of a multi-result report
starts = [i for i, l in enumerate(lines) if l.startswith('"Address"')]
start = starts[which]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"') or lines[i].startswith('"Address"')),
           len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:end]))))
agg = collections.Counter()
tot = 0
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    op = op.split(".")[0]
    agg[op] += n
    tot += n
print("total warp instructions executed", tot)
for op, n in agg.most_common(30):
    print(f"{op:10s} {n:12d} {100.0 * n / tot:5.1f}%")
hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
print("\nhottest (stall samples, executed, source):")
for r in hot:
    print(r["Warp Stall Sampling (All Samples)"], r["Instructions Executed"], r["Address"][-5:], r["Source"].strip()[:90])

if len(sys.argv) > 3:  # dump a window of SASS around an address suffix
    key = sys.argv[3]
    i = next(k for k, r in enumerate(rows) if r["Address"].endswith(key))
    for r in rows[max(0, i - 30): i + 12]:
        print(r["Warp Stall Sampling (All Samples)"].rjust(5), r["Instructions Executed"].rjust(9), r["Address"][-5:],
              r["Source"].strip()[:100])

tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print("total stall samples", tot_s)
ldl = [(r["Address"][-5:], r["Instructions Executed"]) for r in rows if "LDL" in r["Source"] or "STL" in r["Source"]]
print("local-memory instructions:", len(ldl), "executed", sum(int(e or 0) for _, e in ldl))
