#!/bin/bash
# launch list of the cooperative-batch step (all kernels, one GPU)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/launch_cb
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 300 -c 300 --csv \
  --log-file $O/launches.csv python tools/profile_target.py cobatch --epochs 1 > $O/ncu.log 2>&1
echo "rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open('gpurun_out/launch_cb/launches.csv') if l.startswith('"')))
t = collections.defaultdict(float); n = collections.Counter(); b = collections.defaultdict(float)
order = []
for r in rows:
    k = r['Kernel Name'].split('(')[0][:60]
    v = float(r['Metric Value'].replace(',', ''))
    if r['Metric Name'] == 'gpu__time_duration.sum':
        t[k] += v / 1e6; n[k] += 1; order.append((r['ID'], k, v / 1e6))
    else:
        b[k] += v
tot = sum(t.values())
for k in sorted(t, key=lambda k: -t[k]):
    print(f"{k:60s} {n[k]:5d} {t[k]:9.3f} ms {100*t[k]/tot:5.1f}%  {b[k]/1e9/max(t[k],1e-9)/1e3:7.0f} GB/s")
print('total', round(tot, 3))
open('gpurun_out/launch_cb/order.txt','w').write('\n'.join(f'{i} {k} {v:.4f}' for i, k, v in order))
PY
