"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py launches <launches.csv> <round> [config]
        -> profiles/<round>_launches.csv (copy), profiles/<round>_launches.md (one step, per-kernel
           duration / DRAM bytes / share), profiles/ncu_traffic.json[config][kernel] = DRAM bytes
    python tools/ncu_summary.py full <report.ncu-rep> <round> <name>
        -> profiles/<round>_<name>_ncu.txt (SOL, tensor pipe, DRAM, stall reasons)
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

def label(kernel):
    """Short name of one of our launches from ncu's (demangled) kernel name."""
    k = kernel
    if "gae_kernel" in k:
        return "gae_scan"
    if "head_fused" in k:
        return "head_fused"
    if "update_kernel" in k:
        return "grad_update"
    if "stats_kernel" in k:
        return "stats"
    if "p2p_allreduce" in k:
        return "allreduce"
    if "p2p_moments" in k:
        return "adv_norm"
    if "gemm_tc_kernel" in k:
        epi = k.split("gemm_tc_kernel<")[1].split(">")[0].split(",")[3].strip()
        return {"0": "fwd", "4": "fwd", "1": "dX", "2": "dW", "3": "head_loss", "5": "head_sample"}.get(epi, "gemm")
    return k.split("(")[0].split("::")[-1][:40]


def launches(path, rnd, config="atari"):
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(path, os.path.join(PROF, f"{rnd}_launches.csv"))
    txt = open(path).read()
    body = "\n".join(l for l in txt[txt.index('"ID"'):].splitlines() if l.startswith('"'))
    rows = list(csv.DictReader(io.StringIO(body)))
    by = collections.OrderedDict()
    for r in rows:
        by.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(
            r["Metric Value"].replace(",", ""))
    recs = list(by.values())
    starts = [i for i, r in enumerate(recs) if ("gae_kernel" in r["kernel"])]
    k0 = min(3, len(starts) - 1)                       # the first step after 3 warm-up steps
    start = starts[k0]
    end = starts[k0 + 1] if k0 + 1 < len(starts) else len(recs)
    step = recs[start:end]
    tot = sum(r["gpu__time_duration.sum"] for r in step)
    lines = [f"# {rnd}: ncu launch list, one `srl_ppo_train_step` ({config}-shaped, 1 x B200)", "",
             "Cold-cache, serialised per-launch durations (`--metrics gpu__time_duration.sum,"
             "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`); compare shares.", "",
             "| kernel | ncu name | us | share | DRAM read MB | DRAM write MB |",
             "|---|---|---|---|---|---|"]
    traffic = {"launches": [], "dram_bytes": []}     # in launch order (bench.py matches by position)
    seen = collections.Counter()
    for r in step:
        name = label(r["kernel"])
        seen[name] += 1
        t = r["gpu__time_duration.sum"] / 1e3
        rd, wr = r.get("dram__bytes_read.sum", 0.0), r.get("dram__bytes_write.sum", 0.0)
        traffic["launches"].append(name)
        traffic["dram_bytes"].append(rd + wr)
        lines.append(f"| {name}#{seen[name]} | `{r['kernel'][:60]}` | {t:.1f} | {100 * t * 1e3 / tot:.1f}% | "
                     f"{rd / 1e6:.1f} | {wr / 1e6:.1f} |")
    lines.append(f"| **step** | | {tot / 1e3:.1f} | 100% | | |")
    jp = os.path.join(PROF, "ncu_traffic.json")
    data = json.load(open(jp)) if os.path.exists(jp) else {}
    data[config] = traffic
    data.setdefault("_source", {})[config] = f"{rnd}_launches.csv"
    open(os.path.join(PROF, f"{rnd}_launches.md"), "w").write("\n".join(lines) + "\n")
    json.dump(data, open(jp, "w"), indent=1)
    print("\n".join(lines))


def full(rep, rnd, name):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, r = rows[0], rows[1], rows[2]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__cluster_dim_x"]
    out = [f"# {rnd} ncu --set full: {name}", f"kernel: {r[h.index('Kernel Name')]}", ""]
    for k in keys:
        if k in h:
            out.append(f"{k} = {r[h.index(k)]} {units[h.index(k)]}")
    out.append("")
    out.append("stall reasons (warps per issue-active cycle):")
    st = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
    for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
        out.append(f"  {k:24s} {v:.3f}")
    open(os.path.join(PROF, f"{rnd}_{name}_ncu.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], *(sys.argv[4:5] or ["atari"]))
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4])
