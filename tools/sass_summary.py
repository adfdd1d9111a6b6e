"""Per-kernel SASS instruction counts of libsas.so (cuobjdump -sass): the
mnemonics that prove the FP64 tensor path (DMMA), the bulk async copies
(UBLKCP) and mbarriers (SYNCS), plus FP64 FMA/MUL and shuffles.
Usage: python tools/sass_summary.py [libsas.so] > profiles/rNN_sass_summary.txt"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

lib = sys.argv[1] if len(sys.argv) > 1 else str(Path(__file__).resolve().parents[1] / "paper_2510_04825_b200" / "libsas.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
counts = defaultdict(Counter)
fn = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and fn:
        counts[fn][m.group(2)] += 1
KEYS = ["DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "SYNCS", "SHFL", "LDS", "STS", "LDG", "STG", "MUFU", "BAR"]
demangled = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# cuobjdump -sass {Path(lib).name}: static instruction counts per kernel")
print("kernel".ljust(70) + "".join(k.rjust(8) for k in KEYS) + "   total")
for (name, c), dm in sorted(zip(counts.items(), demangled), key=lambda x: x[1]):
    short = re.sub(r"\(.*", "", dm)[:68]
    print(short.ljust(70) + "".join(str(c.get(k, 0)).rjust(8) for k in KEYS) + str(sum(c.values())).rjust(8))
tot = Counter()
for c in counts.values():
    tot.update(c)
print("ALL".ljust(70) + "".join(str(tot.get(k, 0)).rjust(8) for k in KEYS) + str(sum(tot.values())).rjust(8))
print("# no HMMA / UTC*MMA: FP64 has no tcgen05 kind on sm_100a; DMMA (mma.sync f64) is the FP64 tensor path")
