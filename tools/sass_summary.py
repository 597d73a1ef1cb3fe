#!/usr/bin/env python
"""Instruction-count summary of libhmxg.so's kernels from `cuobjdump -sass` (no GPU needed).

    python tools/sass_summary.py [libhmxg.so] > profiles/sass_summary.txt

Per kernel (hmxg.cu's instantiations): total SASS instructions and the counts of the
opcodes that show the data path — DMMA (FP64 tensor core MMA), UTMALDG (TMA tile loads),
UBLKCP (bulk copies), SYNCS (mbarrier operations), LDS/STS, LDG/STG, RED/ATOM, MEMBAR,
FENCE. `__graft_entry__.build()` regenerates profiles/sass_summary.txt for every build.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("DMMA", "UTMALDG", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG", "REDG", "ATOMG", "MEMBAR", "FENCE", "BAR",
        "NANOSLEEP", "DFMA", "MUFU")


def summary(lib: str) -> str:
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out = [f"# cuobjdump -sass {os.path.relpath(lib, ROOT)} (sm_100a): per-kernel instruction counts",
           "# kernel (hmxg.cu instantiation)  total  " + "  ".join(KEYS)]
    cur, counts = None, None
    rows = []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                rows.append((cur, counts))
            cur, counts = m.group(1), collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Za-z0-9_.]+)?", line)
        if cur and m:
            op, ext = m.group(1), m.group(2) or ""
            counts["total"] += 1
            counts[op] += 1
            if op == "DMMA":
                counts["DMMA" + ext] += 1
    if cur:
        rows.append((cur, counts))
    for name, c in rows:
        if "hmxg_cu" not in name:
            continue
        short = re.sub(r"_ZN4hmxg\d+_GLOBAL__N__\w+?_cu_\w+?\d+(\w+?)E.*", r"\1", name)
        short = re.sub(r"^\d+", "", short).replace("ILb0", "<false>").replace("ILb1", "<true>")
        out.append(f"{short:14s} {c['total']:6d}  " + "  ".join(f"{k}={c[k]}" for k in KEYS if c[k]))
        dm = {k: v for k, v in c.items() if k.startswith("DMMA.")}
        if dm:
            out.append(f"{'':14s}        " + "  ".join(f"{k}={v}" for k, v in sorted(dm.items())))
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1812_07152_b200", "libhmxg.so")
    sys.stdout.write(summary(lib))
