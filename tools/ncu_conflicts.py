"""Shared-memory instructions with excess wavefronts (bank conflicts) in an ncu
report: `python tools/ncu_conflicts.py rep [top]`."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
si, ai = h.index("Source"), h.index("Address")
ex, wf, ideal = (h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared"),
                 h.index("L1 Wavefronts Shared Ideal"))
data = [r for r in rows[hi + 1:] if len(r) > ex and r[ex].replace(".", "").isdigit()]
tot = sum(float(r[ex]) for r in data)
print(f"excess shared wavefronts: {tot:.0f}")
for r in sorted(data, key=lambda r: -float(r[ex]))[:top]:
    if float(r[ex]) == 0:
        break
    print(f"{float(r[ex]):12.0f} wf={float(r[wf]):12.0f} ideal={float(r[ideal]):12.0f} {r[ai][-5:]} {r[si].strip()[:70]}")
