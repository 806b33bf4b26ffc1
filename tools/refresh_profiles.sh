# Copies the evidence gathered by tools/collect_round.sh (run under gpurun) from
# gpurun_out/ into profiles/ (run here, after the call).
set -e
python tools/ncu_summary.py gpurun_out/ntt_full.ncu-rep profiles/r01_ntt_fwd_ncu_full.json 1184 profiles/ntt_traffic.json > /dev/null
python - <<'PY'
import json
l = json.load(open('gpurun_out/bench.json'))
l['roofline']['traffic'] = json.load(open('profiles/ntt_traffic.json'))['bytes_per_limb'] * 1184
json.dump(l, open('profiles/r01_bench.json', 'w'))
PY
cp gpurun_out/bench_ref.json profiles/bench_r01_reference_arm.json
cp gpurun_out/bench_launches.csv profiles/r01_bench_launches.csv
python tools/launch_shares.py gpurun_out/bench_launches.csv > profiles/r01_bench_launches_shares.txt
cp gpurun_out/launches.csv profiles/r01_cloud_step_launches.csv
python tools/launch_shares.py gpurun_out/launches.csv > profiles/r01_cloud_step_shares.txt
python tools/metrics_table.py > profiles/r01_cloud_step_metrics.txt
python - <<'PY'
import collections, csv
rows = list(csv.reader(open('gpurun_out/metrics.csv')))
hi = next(i for i, r in enumerate(rows) if 'Metric Name' in r)
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.OrderedDict()
for r in data:
    per.setdefault(r[idi], {'kernel': r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')})[r[mi]] = r[vi]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size']
with open('profiles/r01_cloud_step_metrics.csv', 'w', newline='') as f:
    w = csv.writer(f)
    w.writerow(['id', 'kernel'] + keys)
    for i, m in per.items():
        w.writerow([i, m['kernel']] + [m.get(k, '') for k in keys])
PY
cat profiles/r01_cloud_step_metrics.txt
