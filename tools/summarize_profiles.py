"""Summarises a tools/profile_round.sh run (gpurun_out/prof) into profiles/.

    python tools/summarize_profiles.py r02

ncu values keep their units (the raw page's second row); DRAM bytes are
converted to bytes per launch for bench.py's roofline.traffic."""
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
RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
DST.mkdir(exist_ok=True)
sys.path.insert(0, str(ROOT))
from paper_2604_23150_b200.pipeline import WORKLOADS  # noqa: E402

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(rep):
    rep = Path(rep)
    csv_path = rep.with_suffix("").with_suffix(".raw.csv") if rep.suffix == ".ncu-rep" else rep
    if csv_path.exists():  # exported on the box (tools/profile_round.sh export_rep)
        out = csv_path.read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tma.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_bytes.sum", "lts__t_sectors.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second"]


def kernel_rows(rep):
    res = []
    for r, u in raw(rep):
        d = {"kernel": r.get("Kernel Name", "")[:100]}
        for k in KEYS:
            if k in r:
                d[k] = {"value": num(r[k]), "unit": u.get(k, "")}
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in d and d[k]["value"] is not None:
                b += d[k]["value"] * SCALE.get(d[k]["unit"], float("nan"))
        d["dram_bytes_per_launch"] = b
        res.append(d)
    return res


def launch_shares(w, bench):
    src = SRC / f"launches_{w}.csv"
    gz = SRC / f"launches_{w}.csv.gz"
    if gz.exists():
        shutil.copy(gz, DST / f"{RND}_launches_{w}.csv.gz")
        text = gzip.open(gz, "rt").read()
    elif src.exists():
        with open(src, "rb") as f, gzip.open(DST / f"{RND}_launches_{w}.csv.gz", "wb") as g:
            shutil.copyfileobj(f, g)
        text = src.read_text()
    else:
        return
    rows = list(csv.reader(text.splitlines()))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    seq = [(r[ki], num(r[vi]) * scale.get(r[ui], float("nan"))) for r in rows[start + 1:]
           if len(r) > vi and num(r[vi]) is not None and num(r[vi]) == num(r[vi])]  # ncu "nan": unmeasured launch
    # the last routed step: from its first router launch onwards, up to the
    # reference-statistic kernels the bench runs after the timed loop
    n_router = bench["config"]["schedule"]["router_launches_per_step"]
    router_idx = [i for i, (k, _) in enumerate(seq) if "k_router" in k]
    step = seq[router_idx[-n_router]:]
    stop = next((i for i, (k, _) in enumerate(step) if "k_sample" in k or "FillFunctor" in k),
                len(step))
    step = step[:stop]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in step:
        name = k.split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    lines = [f"# {RND}: per-kernel share of one {bench['config']['workload']} step "
             f"(ncu gpu__time_duration, cold and serialised: shares, not absolutes; "
             f"{n_router} router launches for {bench['config']['layers']} layers; the "
             f"statistics tails run beside the routers in the real step)", "",
             f"command: `python bench.py --workload {w} --steps 2 --warmup 1 --no-e2e "
             f"--no-cpu-baseline --no-a2a`", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {name} | {n} | {v:.1f} | {100 * v / tot:.1f}% |")
    lines.append(f"| **total** | {sum(n for n, _ in agg.values())} | {tot:.1f} | 100% |")
    (DST / f"{RND}_launch_shares_{w}.md").write_text("\n".join(lines) + "\n")


# 1. bench lines + launch shares
benches = {}
for w in ("dsv3", "qwen3", "maverick", "domain"):
    p = SRC / f"bench_{w}.json"
    if not p.exists() or not p.read_text().strip():
        continue
    bench = json.loads(p.read_text().strip().splitlines()[-1])
    benches[w] = bench
    (DST / f"{RND}_bench_{w}_n1.json").write_text(json.dumps(bench, indent=1))
    launch_shares(w, bench)

# 2. router full captures per workload shape (+ the plain timing / cuBLAS lines)
summary = {"round": RND, "units": "each metric {value, unit} from ncu's raw page; "
           "dram_bytes_per_launch = read + write in bytes"}
plain = []
for w in ("dsv3", "qwen3", "maverick", "domain"):
    rep = SRC / f"router_{w}.ncu-rep"
    if rep.exists() or (SRC / f"router_{w}.raw.csv").exists():
        rows = kernel_rows(rep)
        if rows:
            summary[WORKLOADS[w].name] = rows[0]
    lp = SRC / f"router_plain_{w}.log"
    if lp.exists():
        plain.append(f"## {w}\n" + lp.read_text())
if (SRC / "router_grouped_plain.log").exists():
    plain.append("## dsv3 grouped (8 layers per launch)\n" +
                 (SRC / "router_grouped_plain.log").read_text())
(DST / "ncu_router_summary.json").write_text(json.dumps(summary, indent=1))
(DST / f"{RND}_router_vs_cublas.txt").write_text(
    "tools/prof_router.py: the router kernel (GEMM + fused top-k) vs cuBLAS's bf16 GEMM alone "
    "(torch.matmul, no top-k) on the same shapes, CUDA events, same box\n\n" + "\n".join(plain))

# 3. statistics / scoring kernels
rep = SRC / "small_full.ncu-rep"
if rep.exists() or (SRC / "small_full.raw.csv").exists():
    small = kernel_rows(rep)
    (DST / f"{RND}_ncu_small_kernels.json").write_text(json.dumps(small, indent=1))
    for s in small:
        t = s.get("gpu__time_duration.sum", {})
        print(s["kernel"][:60], t.get("value"), t.get("unit"), s["dram_bytes_per_launch"])
if (SRC / "kbench_plain.log").exists():
    shutil.copy(SRC / "kbench_plain.log", DST / f"{RND}_kbench_warm.txt")
print(json.dumps({k: (v.get("gpu__time_duration.sum"), v.get("dram_bytes_per_launch"))
                  for k, v in summary.items() if isinstance(v, dict)}, indent=1))
