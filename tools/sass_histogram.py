#!/usr/bin/env python
"""Per-kernel SASS opcode histogram of libclatch.so (cuobjdump -sass): the mnemonics that prove which
hardware path each kernel uses (tcgen05 MMAs, TMEM loads/stores, TMA bulk copies, texture gathers, packed
fp32 FMAs, unfused fp64 — and no DFMA).

    python tools/sass_histogram.py > profiles/<visit>_sass_opcodes.json
"""
import collections
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1609_03986_b200" / "libclatch.so"
WATCH = ["UTCOMMA", "UTCIMMA", "UTCQMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "SYNCS", "TLD4", "TEX",
         "SULD", "SUST", "FFMA2", "FFMA", "DFMA", "DADD", "DMUL", "DSETP", "POPC", "LOP3", "VIMNMX3", "VIMNMX", "FMNMX3",
         "IMMA", "HMMA", "LDS", "STS", "LDG", "STG", "LDGSTS", "F2I", "I2F", "F2F", "SHFL", "VOTE", "REDUX", "BAR", "ELECT"]

out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
kernels, name = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        demangled = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"clatch::\(anonymous namespace\)::|\(clatch::\(anonymous namespace\)::\w+\)|\(.*\)$", "", demangled)
        kernels[name] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and name:
        kernels[name]["total"] += 1
        op = m.group(1)
        for w in WATCH:
            if op == w or (w in ("SYNCS", "BAR", "TEX") and op.startswith(w)):
                kernels[name][w] += 1
                break
res = {k: dict(sorted(v.items(), key=lambda kv: -kv[1])) for k, v in sorted(kernels.items())}
summary = collections.Counter()
for v in kernels.values():
    summary.update(v)
json.dump({"library": str(LIB.relative_to(ROOT)), "all_kernels": dict(summary), "DFMA_total": summary.get("DFMA", 0),
           "kernels": res}, sys.stdout, indent=1)
