# per-kernel device times (ncu launch list, serialised) of a few cfg3 steps, A/B by env
mkdir -p gpurun_out
python tools/gpu/step_run.py 64x32x32 3 > gpurun_out/plain.log 2>&1 && \
for v in "X=1" "DNNMG_NO_ELEM_POS=1"; do
env $v ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv \
   --log-file gpurun_out/launches_$v.csv python tools/gpu/step_run.py 64x32x32 3 > /dev/null 2>&1
python - "$v" <<'PY'
import csv, sys, collections
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{v}.csv")) if len(r) > 10]
h = rows[0]; k = h.index("Kernel Name"); m = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[k][:50]].append(float(r[m].replace(",", "")))
print(v)
for n, xs in agg.items(): print(f"  {n:50s} {len(xs):3d} {sum(xs)/len(xs)/1e3:9.1f} us")
PY
done
