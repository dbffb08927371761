"""Summarises a tools/profile_round.sh run (gpurun_out/prof) into profiles/."""
import collections
import csv
import gzip
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / "prof"
DST = ROOT / "profiles"
RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
DST.mkdir(exist_ok=True)


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def kernel_rows(rep):
    res = []
    for r in raw(rep):
        d = {"kernel": r.get("Kernel Name", "")[:90]}
        for k in KEYS:
            if k in r:
                d[k] = num(r[k])
        res.append(d)
    return res


# 1. bench line
line = (SRC / "bench_n1.json").read_text().strip().splitlines()[-1]
bench = json.loads(line)
(DST / f"{RND}_bench_dsv3_n1.json").write_text(json.dumps(bench, indent=1))

# 2. launch list (gzip) + per-kernel shares of the timed step
with open(SRC / "launches.csv", "rb") as f, gzip.open(DST / f"{RND}_launches.csv.gz", "wb") as g:
    shutil.copyfileobj(f, g)
rows = list(csv.reader(open(SRC / "launches.csv")))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = [(r[ki], num(r[vi])) for r in rows[start + 1:] if len(r) > vi]
# the last step's launches: from its first k_router launch onwards (grouped
# router launches: several layers per launch, config.schedule)
router_idx = [i for i, (k, _) in enumerate(seq) if "k_router" in k]
L = bench["config"]["layers"]
sched = bench["config"].get("schedule")
if sched:
    n_router = sched["router_launches_per_step"]
else:
    sys.path.insert(0, str(ROOT))
    from paper_2604_23150_b200.pipeline import _taper_chunks  # noqa: E402
    n_router = len(_taper_chunks(L, 8))
step = seq[router_idx[-n_router]:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in step:
    name = k.split("(")[0].replace("void ", "").strip()
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
lines = [f"# {RND}: per-kernel share of one DSv3 step (ncu gpu__time_duration, cold/serialised; "
         f"{n_router} grouped router launches for {L} layers)",
         "", f"command: `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline`", "",
         "| kernel | launches | total us | share |", "|---|---|---|---|"]
for name, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {name} | {n} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
lines.append(f"| **total** | {sum(n for n, _ in agg.values())} | {tot / 1e3:.1f} | 100% |")
(DST / f"{RND}_launch_shares.md").write_text("\n".join(lines) + "\n")

# 3. full captures
router = kernel_rows(SRC / "router_full.ncu-rep")[0]
router["dram_bytes_per_launch"] = (router["dram__bytes_read.sum"] or 0) * 1e6 + \
    (router["dram__bytes_write.sum"] or 0) * 1e6  # ncu reports MB
(DST / "ncu_router_summary.json").write_text(json.dumps(
    {"deepseek-v3-shape": router, "round": RND,
     "command": "tools/prof_router.py --T 65536 --H 7168 --E 256 --k 8 (sigmoid, renorm)",
     "units": "ncu raw page (time ns, dram MB, pct)"}, indent=1))
small = kernel_rows(SRC / "small_full.ncu-rep")
(DST / f"{RND}_ncu_small_kernels.json").write_text(json.dumps(small, indent=1))
print(json.dumps(router, indent=1))
print((DST / f"{RND}_launch_shares.md").read_text())
for s in small:
    print(s["kernel"][:50], s.get("gpu__time_duration.sum"), s.get("dram__bytes_read.sum"),
          s.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"))
