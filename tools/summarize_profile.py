"""Turn a gpurun_out/ profiling capture (tools/profile_run.sh) into the tracked
summaries under profiles/:

    python tools/summarize_profile.py --tag r01 [--dir gpurun_out]

Writes profiles/<tag>_launches.txt (per-kernel share of the launch list),
profiles/<tag>_ncu_full.txt (key ncu --set full metrics per captured kernel)
and profiles/ncu_summary.json (dram bytes per launch of the dominant kernel,
read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "launch__grid_size", "smsp__inst_executed.sum"]


def to_bytes(v, unit):
    v = float(str(v).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--dir", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)

    # launch list
    rows = list(csv.reader(open(os.path.join(a.dir, "launches.csv"))))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0][:90]
                agg[k][0] += 1
                agg[k][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none) of: python bench.py "
             f"--steps 2 --warmup 3 --no-cpu-baseline --no-e2e (setup + 6 epochs; cold-cache, "
             f"serialised: compare shares)",
             f"{'total_ms':>10} {'launches':>8} {'share':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[1] / 1e6:10.3f} {v[0]:8d} {100 * v[1] / tot:6.1f}%  {k}")
    open(os.path.join(out_dir, f"{a.tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

    # full capture
    raw = subprocess.run(["ncu", "-i", os.path.join(a.dir, "prof_full.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rr[0], rr[1], rr[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out = ["# ncu --set full --clock-control none, kernels aggregate_vec4 / gemm_bf16x3 "
           "captured inside python bench.py --steps 2 --warmup 3"]
    agg_dram = []
    for d in data:
        name = d[idx["Kernel Name"]]
        out.append(f"\n## {name[:100]}")
        for k in KEYS:
            if k in idx:
                out.append(f"  {k}: {d[idx[k]]} {units[idx[k]]}")
        if "aggregate_vec4" in name:
            agg_dram.append(to_bytes(d[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]]) +
                            to_bytes(d[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]]))
    open(os.path.join(out_dir, f"{a.tag}_ncu_full.txt"), "w").write("\n".join(out) + "\n")
    if agg_dram:
        json.dump({"aggregate_dram_bytes_per_launch": int(sum(agg_dram) / len(agg_dram)),
                   "launches_captured": len(agg_dram), "source": f"profiles/{a.tag}_ncu_full.txt"},
                  open(os.path.join(out_dir, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
