"""Round-2 ncu summaries (gpurun_out/prof2 -> profiles/): the bench command's launch
list as per-kernel shares, the --set full metrics per captured kernel, and the
per-config DRAM traffic of the dominant kernel (profiles/ncu_traffic.json, read by
bench.py for roofline.traffic)."""
import csv
import json
import os
import re
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys
# usage: summarize.py [src dir under gpurun_out] [tag]   (defaults: prof2 r02)
SRC = os.path.join(ROOT, "gpurun_out", sys.argv[1] if len(sys.argv) > 1 else "prof2")
TAG = sys.argv[2] if len(sys.argv) > 2 else "r02"
OUT = os.path.join(ROOT, "profiles")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
        "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}


def short(name):
    name = re.sub(r"\(CUtensorMap_st.*|\(gdx::.*|\(unnamed>::.*|\((unsigned|const|float|int|double).*", "", name)
    return name.replace("void ", "").replace("gdx::<unnamed>::", "").replace("unnamed>::", "")


def launches():
    rows = [r for r in csv.reader(open(os.path.join(SRC, "launches.csv"))) if len(r) > 10]
    hdr = rows[0]
    i = {h: k for k, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[i["Metric Name"]] != "gpu__time_duration.sum":
            continue
        ms = float(r[i["Metric Value"]].replace(",", "")) * UNIT.get(r[i["Metric Unit"]], 1e-6)
        k = short(r[i["Kernel Name"]])
        tot[k] += ms
        cnt[k] += 1
    all_ms = sum(tot.values())
    lines = ["# round 2: ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "
             "--no-hbm-pass` (gpu__time_duration.sum, --clock-control none; cold-cache, serialised:",
             "# shares are what matters, absolute times are not bench numbers)",
             f"# {sum(cnt.values())} launches, {all_ms:.2f} ms total", "",
             f"{'kernel':60s} {'launches':>8s} {'ms':>9s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:60]:60s} {cnt[k]:8d} {v:9.3f} {v / all_ms:7.1%}")
    open(os.path.join(OUT, f"{TAG}_launches.txt"), "w").write("\n".join(lines) + "\n")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tma.sum"]
LABEL = ["ms", "dramR GB", "dramW GB", "dram%", "lts%", "L2hit%", "tensor%", "lsb/issue", "regs", "occ%", "tma"]


def full():
    traffic = {}
    lines = ["# round 2: ncu --set full --clock-control none --import-source on captures (one GPU) of",
             "# tools/profile_target.py <workload> (the C-ABI trainer's eager epoch / the HBM-regime pass /",
             "# a papers-shape cooperative batch); the .ncu-rep files stay on the box (60 MB each), these",
             "# are their raw-page metrics.  tools/r02/profile.sh, tools/r02/summarize.py", ""]
    for t in ("reddit", "products", "hbm", "cobatch"):
        p = os.path.join(SRC, f"full_{t}.csv")
        if not os.path.exists(p):
            continue
        rows = list(csv.reader(open(p)))
        hdr, units = rows[0], rows[1]
        i = {h: k for k, h in enumerate(hdr)}
        lines += [f"## {t}", f"{'kernel':44s} " + " ".join(f"{l:>9s}" for l in LABEL)]
        agg = []
        for r in rows[2:]:
            vals = []
            for k in KEYS:
                v = r[i[k]].replace(",", "") if k in i else ""
                try:
                    x = float(v)
                except ValueError:
                    vals.append(float("nan"))
                    continue
                u = units[i[k]]
                if "bytes" in k:
                    x = x * UNIT.get(u, 1) / 1e9
                elif k == "gpu__time_duration.sum":
                    x = x * UNIT.get(u, 1e-6)
                vals.append(x)
            name = short(r[i["Kernel Name"]])
            lines.append(f"{name[:44]:44s} " + " ".join(f"{v:9.3f}" for v in vals))
            if "aggregate" in name:
                agg.append((name, vals[1] + vals[2], vals[0]))
        lines.append("")
        if agg:
            # the dominant (most frequent) aggregation kernel: mean DRAM bytes per launch
            top = max({a[0] for a in agg}, key=lambda n: sum(x[2] for x in agg if x[0] == n))
            sel = [a for a in agg if a[0] == top]
            traffic[t] = {"kernel": top, "launches": len(sel),
                          "dram_bytes_per_launch": int(sum(a[1] for a in sel) / len(sel) * 1e9),
                          "source": f"profiles/{TAG}_ncu_full.txt ({t})"}
    open(os.path.join(OUT, f"{TAG}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
    names = {"reddit": "reddit-sage", "products": "products-gcn", "hbm": "hbm-regime-products64",
             "cobatch": "papers-cobatch"}
    try:  # keep the configs this capture did not cover
        out = json.load(open(os.path.join(OUT, "ncu_traffic.json")))
    except Exception:
        out = {}
    out.update({names[k]: {"aggregate": v} for k, v in traffic.items()})
    json.dump(out, open(os.path.join(OUT, "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    launches()
    full()
