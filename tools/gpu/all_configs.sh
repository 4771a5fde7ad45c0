# bench line of every BASELINE correction-step config (device-timed + e2e), one line each
mkdir -p gpurun_out
for c in "cfg0" "cfg1" "cfg1 --precision bf16" "cfg2" "cfg3 --precision bf16" "cfg3 --precision tf32x3"; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-aux > gpurun_out/cfg.log 2>&1
  tail -1 gpurun_out/cfg.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({'config': '$c', 'patches/s': round(d['value']), 'ms': round(d['ms_per_step'],4), 'e2e': round(d['e2e']['value']) if d.get('e2e') else None, 'kernels': {k: round(v['ms'],4) for k,v in d['kernels'].items()}}))"
done
