"""Summarise an ncu source page: top stall lines with SASS context."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
si, ci, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
data = [r for r in rows[hi + 1:] if len(r) > ci]
tot = sum(int(r[ci]) for r in data if r[ci].isdigit())
print("total samples", tot)
order = sorted(range(len(data)), key=lambda k: -int(data[k][ci]) if data[k][ci].isdigit() else 0)
for k in order[:top]:
    r = data[k]
    prev = data[k - 1][si].strip() if k else ""
    print(f"{int(r[ci]):7d} {100*int(r[ci])/tot:5.1f}% {r[ai][-5:]} {r[si].strip()[:60]:60s} | prev: {prev[:50]}")
