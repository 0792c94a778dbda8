"""Collect the final bench lines (gpurun_out/final/*.json + N=2 lines) into
profiles/r02_bench_lines.jsonl (one JSON line per run, as printed by bench.py)."""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
files = sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "final", "*.json")) +
               glob.glob(os.path.join(ROOT, "gpurun_out", "r02_bench_*_n2.json")))
out = []
for f in files:
    lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
    if not lines:
        continue
    d = json.loads(lines[-1])
    d["_file"] = os.path.relpath(f, ROOT)
    out.append(d)
with open(os.path.join(ROOT, "profiles", "r02_bench_lines.jsonl"), "w") as fh:
    for d in out:
        fh.write(json.dumps(d) + "\n")
for d in out:
    print(d["_file"], d.get("impl", "b200"), d.get("n_gpus"), d.get("value"), (d.get("e2e") or {}).get("value"))
