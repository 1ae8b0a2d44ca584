"""SASS opcode histogram of the built library (cuobjdump -sass), per kernel.

Evidence for DESIGN.md §4: the solver is FP64 (DADD/DMUL/DFMA, no DFMA
contraction where the reference rounds products: --fmad=false), no tensor-core
(UTCMMA/HMMA) or TMA (UTMALDG) instructions, FP32/MUFU only for α/β.
Usage: python tools/sass_hist.py [lib.so] > profiles/sass_hist_rNN.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1803_07772_b200", "libhcran_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
fn, hist = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and fn:
        hist[fn][m.group(2) + (m.group(3) or "")] += 1
CLASSES = {"fp64": ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"), "fp32": ("FADD", "FMUL", "FFMA", "FSETP", "FMNMX"),
           "mufu": ("MUFU",), "tensor/tma": ("UTCMMA", "UTCHMMA", "HMMA", "UTMALDG", "UTMASTG")}
print(f"# cuobjdump -sass {os.path.relpath(lib, ROOT)}: static instruction counts per kernel")
for f, c in hist.items():
    total = sum(c.values())
    print(f"\n{f}  total {total}")
    for cls, ops in CLASSES.items():
        n = sum(v for k, v in c.items() if k.split(".")[0] in ops)
        print(f"  class {cls:10s} {n:7d}  ({100.0 * n / total:5.2f} %)")
    for op, n in c.most_common(60):
        print(f"  {op:28s} {n:7d}")
