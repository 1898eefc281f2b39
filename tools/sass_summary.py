#!/usr/bin/env python
"""Per-kernel SASS instruction counts of the built library (cuobjdump -sass): the tensor-core
(UTCHMMA / UTCQMMA), TMEM (LDTM / STTM), bulk-copy (UBLKCP) and FP64 (DFMA / DMUL / DADD)
mnemonics that show which pipe each kernel runs on. Writes a markdown table to stdout."""
import collections
import os
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_2411_03289_b200",
                                                          "lib", "libgpmppi_b200.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "FFMA", "FFMA2",
       "MUFU", "LDS", "STS", "LDG", "STG", "SHFL", "BAR"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
counts = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        op = m.group(1)
        counts[cur][op] += 1
        if op == "FFMA" and m.group(2) and "F32x2" in m.group(2).upper():
            counts[cur]["FFMA2"] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(.*", "", d)
    if not d:  # anonymous-namespace kernels (fit.cu): keep the plain name
        m = re.search(r"\d+([a-z_]+_[a-z_]+)E", name)
        d = "(fit.cu) " + (m.group(1) if m else name)
    return d


print("| kernel | " + " | ".join(OPS) + " | total |")
print("|---|" + "---|" * (len(OPS) + 1))
for k, c in counts.items():
    if sum(c.values()) == 0:
        continue
    print(f"| `{short(k)}` | " + " | ".join(str(c.get(o, 0)) for o in OPS) + f" | {sum(c.values())} |")
