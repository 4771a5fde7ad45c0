# e2e (host buffers) sensitivity: pipeline depth, repeated
for d in 2 3 4 2 3; do
  python bench.py --no-cpu-baseline --no-aux --steps 20 --warmup 5 --pipe-depth $d > gpurun_out/e2e.log 2>&1
  echo "depth $d $(tail -1 gpurun_out/e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,1))")"
done
python bench.py --no-cpu-baseline --no-aux --steps 60 --warmup 5 > gpurun_out/e2e.log 2>&1
echo "steps 60 $(tail -1 gpurun_out/e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,1))")"
