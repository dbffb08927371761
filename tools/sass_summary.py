"""Per-kernel SASS instruction summary of the shipped library (cuobjdump -sass):
the Blackwell-native instructions each kernel uses — UTCHMMA / UTCIMMA
(tcgen05.mma bf16 / int8), UTMALDG (TMA tensor loads), UBLKCP (bulk copies),
LDTM / STTM (TMEM loads / stores), UTCBAR (tcgen05.commit), SYNCS (mbarrier
ops), plus instruction totals.

    python tools/sass_summary.py [lib] > profiles/r02_sass_summary.md
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2604_23150_b200" /
                                                 "libmoeplace_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UBLKPF",
       "LDTM", "STTM", "UTCBAR", "UTCATOMSWS", "SYNCS", "HMMA", "IMMA", "REDG", "ATOMS",
       "MATCH", "VOTE", "POPC", "DFMA", "DADD", "DMUL"]
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        op = m.group(2)
        counts[kern]["total"] += 1
        for o in OPS:
            if op == o or op.startswith(o):
                counts[kern][o] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


names = list(counts)
pretty = demangle(names)
print(f"# SASS summary of `{Path(lib).name}` (cuobjdump -sass, sm_100a)\n")
print("Static instruction counts per kernel (not executed counts). tcgen05 / TMA / TMEM "
      "mnemonics: UTCHMMA = tcgen05.mma kind::f16 (bf16), UTCIMMA = tcgen05.mma kind::i8, "
      "UTMALDG = cp.async.bulk.tensor (TMA load), UBLKCP = cp.async.bulk, LDTM / STTM = "
      "tcgen05.ld / st, UTCBAR = tcgen05.commit, SYNCS = mbarrier operations.\n")
cols = [o for o in OPS if any(c[o] for c in counts.values())]
print("| kernel | total | " + " | ".join(cols) + " |")
print("|---|---|" + "---|" * len(cols))
for n, p in zip(names, pretty):
    short = p.replace("(anonymous namespace)::", "").replace("void ", "")
    short = re.sub(r"\(.*", "", short).replace("mpb::", "")
    c = counts[n]
    print(f"| `{short[:70]}` | {c['total']} | " + " | ".join(str(c[o] or "") for o in cols) + " |")
