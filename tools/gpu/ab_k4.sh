# K4 A/B timing only: kernel means from an ncu launch list of a short bench run
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/ab_k4.log 2>&1
python -c "
import json;l=[x for x in open('gpurun_out/ab_k4.log') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
