"""profiles/ncu_traffic.json from the gpurun_out/traffic_<workload>.csv launch
metrics written by tools/gpu_traffic.sh (DRAM bytes read + write per launch of
each workload's persistent kernel, normalised per RK4 step).
    python tools/traffic_json.py [csv_dir]"""
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out"
script = (ROOT / "tools" / "gpu_traffic.sh").read_text()
steps = {m.group(1): int(m.group(2)) for m in re.finditer(r"^run (\S+) (\d+) ", script, re.M)}
N = {"n1e4": 10000, "n4e4": 40000, "n1000": 1000, "ens512": 1000, "ens512_exact": 1000, "n100": 100, "n1": 1}
out_path = ROOT / "profiles" / "ncu_traffic.json"
out = json.loads(out_path.read_text())
for wl, k in steps.items():
    f = src / f"traffic_{wl}.csv"
    if not f.exists():
        continue
    rows = [r for r in csv.reader(f.read_text().splitlines()) if len(r) > 14 and r[0].isdigit()]
    if not rows:
        continue
    val = {r[12]: (float(r[14].replace(",", "")), r[13]) for r in rows}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
             "msecond": 1e6, "nsecond": 1, "ms": 1e6, "s": 1e9, "second": 1e9, "Tbyte": 1e12}
    rd = val["dram__bytes_read.sum"][0] * scale.get(val["dram__bytes_read.sum"][1], 1)
    wr = val["dram__bytes_write.sum"][0] * scale.get(val["dram__bytes_write.sum"][1], 1)
    ns = val["gpu__time_duration.sum"][0] * scale.get(val["gpu__time_duration.sum"][1], 1)
    n = N[wl]
    out[wl] = {"bytes_per_rk4_step": (rd + wr) / k, "alg_bytes_per_rk4_step": 32.0 * n * n,
               "capture": f"bench.py --workload {wl} --steps 1 --warmup 0 --rk4-steps {k}",
               "kernel_ns": ns, "kernel": rows[0][4]}
out["_doc"] = out["_doc"].split(" Re-captured")[0] + " Re-captured on the round-2 final code (tools/gpu_traffic.sh, tools/traffic_json.py)."
out_path.write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps({k: v["bytes_per_rk4_step"] for k, v in out.items() if k != "_doc"}, indent=1))
