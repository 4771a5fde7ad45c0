mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mlp_layered.py tests/test_gpu_big_pins.py tests/test_slab_gpu.py -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -2 gpurun_out/t.log
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-aux --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/l_cfg2.csv python bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/l_cfg2.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
seq=[(r[ik][:40], float(r[iv].replace(',',''))/1e3) for r in rows[1:]]
idx=[i for i,(k,v) in enumerate(seq) if 'prolongate' in k]
i0=idx[-2]
for k,v in seq[i0:i0+11]: print(f"{k:42s} {v:8.1f} us")
P
timeout 600 python bench.py --mlp-sweep --sweep-batches 262144 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print([(p['H'],p['mode'],round(p['ms'],3),round(p['TFLOP/s']),round(p['frac'],2)) for p in d['points']])"
