"""SASS audit of the built library: per kernel, the instruction counts that
prove the Blackwell paths (B200_PROFILING.md: UTC*MMA = tcgen05.mma, LDTM =
tcgen05.ld, UTMALDG / UBLKCP = TMA, DMMA = FP64 tensor mma.sync) and the
register / stack / shared-memory use.

    python tools/sass_audit.py > profiles/sass_audit_<round>.json
"""
import json
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
MNEMONICS = ("UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG",
             "UBLKCP", "DMMA", "HMMA", "MUFU", "DFMA", "SHFL")


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                             check=True).stdout.splitlines()
        return dict(zip(names, out))
    except Exception:
        return {n: n for n in names}


def main():
    objs = sorted((ROOT / "build").glob("*.o"))
    report = {"library": "paper_1708_02845_b200/libpathfield_b200.so", "objects": {}}
    for o in objs:
        sass = subprocess.run(["cuobjdump", "-sass", str(o)], capture_output=True, text=True).stdout
        if not sass.strip():
            continue
        res = subprocess.run(["cuobjdump", "--dump-resource-usage", str(o)], capture_output=True,
                             text=True).stdout
        usage = {}
        for fn, body in re.findall(r"Function (\S+):\s*\n\s*(REG:.*)", res):
            usage[fn] = dict(re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", body))
        kernels = {}
        for fn, body in re.findall(r"Function : (\S+)\n(.*?)(?=\n\s*Function : |\Z)", sass, re.S):
            ops = Counter(m.split(".")[0] for m in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Z0-9_.]+)", body))
            c = {m: ops[m] for m in MNEMONICS if ops.get(m)}
            kernels[fn] = {"counts": c, "instructions": sum(ops.values()),
                           "resources": usage.get(fn, {})}
        names = demangle(list(kernels))
        report["objects"][o.name] = {names[k]: v for k, v in kernels.items()}
    totals = Counter()
    for kk in report["objects"].values():
        for v in kk.values():
            totals.update(v["counts"])
    report["totals"] = dict(totals)
    json.dump(report, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
