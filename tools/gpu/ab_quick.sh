set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/ab_sleep.log 2>&1
tail -1 gpurun_out/ab_sleep.log
timeout 600 python -m pytest tests -m gpu -x -q -k "mlp or step or k2tc" > gpurun_out/ab_tests.log 2>&1; tail -3 gpurun_out/ab_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/ab_launch.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python - <<'P'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/ab_launch.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[ik][:40]].append(float(r[iv].replace(',','')))
for k,v in d.items(): print(f"{k:40s} n={len(v)} mean={sum(v)/len(v)/1000:.4f} ms")
P
