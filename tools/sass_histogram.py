#!/usr/bin/env python
"""Per-kernel SASS opcode histogram of libadamk.so (cuobjdump -sass): the mnemonics that prove the Blackwell-native
paths (UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG / UBLKCP / UBLKPF = TMA tensor / bulk copy / bulk L2 prefetch,
SYNCS = mbarrier, FFMA2 = packed fp32 FMA, LDG/STG .STRONG.GPU = the tagged-word exchange) and the absence of HMMA.

    python tools/sass_histogram.py > profiles/r02_sass_histogram.md
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

lib = Path(__file__).resolve().parents[1] / "paper_2605_11581_b200" / "csrc" / "libadamk.so"
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
KEY = ("UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UBLKPF", "SYNCS", "FFMA2", "FADD2", "HMMA", "LDGSTS", "LDG", "STG",
       "LDS", "STS", "ATOM", "RED", "MUFU", "SHFL", "BAR", "CALL")
kernels: dict = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = kernels.setdefault(m.group(1), collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if m and cur is not None:
        cur[m.group(1)] += 1
demangle = subprocess.run(["cu++filt"] + list(kernels), capture_output=True, text=True).stdout.splitlines() if kernels else []
print("# SASS opcode histogram per kernel (`cuobjdump -sass paper_2605_11581_b200/csrc/libadamk.so`, sm_100a)\n")
print("Counts of instructions whose mnemonic starts with the column name (all variants summed); `total` = all instructions.\n")
print("| kernel | total | " + " | ".join(KEY) + " | notable variants |")
print("|---|---|" + "---|" * (len(KEY) + 1))
for (name, cnt), nice in zip(kernels.items(), demangle or kernels):
    nice = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", nice)
    cut = nice.rfind(">(")
    nice = nice[:cut + 1] if cut >= 0 else nice.split("(")[0]
    row = [sum(v for k, v in cnt.items() if k.split(".")[0] == key) for key in KEY]
    notable = sorted({k for k in cnt if any(t in k for t in ("2CTA", "STRONG", "UTMALDG", "UBLK", "LDTM", "256"))})[:8]
    print(f"| `{nice}` | {sum(cnt.values())} | " + " | ".join(str(v) for v in row) + " | " + ", ".join(f"`{k}` x{cnt[k]}" for k in notable) + " |")
