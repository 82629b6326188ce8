"""Per-kernel SASS opcode counts of libsto_b200.so: the
evidence that the Blackwell paths are what DESIGN.md says they are --
DMMA / LDTM / STTM (FP64 tensor cores, RK state in tensor memory), UBLKCP
(bulk async copies), SYNCS (mbarriers), ST.ASYNC-style DSMEM pushes, and that
the pinned kernels use DFMA only inside divisions (every MUFU.RCP64H seeds one
division: ~6-8 DFMA each, library or speculative).

    python tools/sass_summary.py [lib.so] > profiles/r02_sass_summary.txt
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2312_01121_b200" / "libsto_b200.so")
KEYS = ["DMMA", "LDTM", "STTM", "UTCBAR", "UBLKCP", "SYNCS", "LDG.E.128", "LDG.E.NA.128",
        "LDG.E.64", "STG.E.128", "STG.E.64", "LDS.128", "LDS.64", "STS.64", "ST.E.64", "STAS",
        "DFMA", "DMUL", "DADD", "MUFU.RCP64H", "CALL.REL", "SHFL.BFLY", "BAR.SYNC", "RED", "ATOM",
        "MEMBAR", "FENCE", "CCTL", "NANOSLEEP"]

sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                      text=True, check=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m:
        op = m.group(2)
        funcs[cur]["_instr"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                funcs[cur][k] += 1


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


names = list(funcs)
pretty = demangle(names)
print(f"# SASS opcode counts per kernel: cuobjdump -sass {Path(lib).name} (sm_100a)")
print("# columns: instructions, then every opcode family with a non-zero count")
for raw, nice in zip(names, pretty):
    c = funcs[raw]
    if c["_instr"] == 0:
        continue
    nice = re.sub(r"\(sto::\w+\)$", "", nice.replace("void ", ""))
    fields = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
    print(f"{nice:60s} instr={c['_instr']:6d} {fields}")
