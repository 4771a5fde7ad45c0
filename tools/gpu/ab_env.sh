# A/B of one env switch on the config-3 bench: bash tools/gpu/ab_env.sh VAR=1 [VAR2=1 ...]
for v in "X=1" "$@"; do
  env $v python bench.py --no-cpu-baseline --no-e2e --no-aux --steps 20 --warmup 5 > gpurun_out/ab.log 2>&1
  echo "$v $(tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in d['kernels'].items()})")"
done
