# quick GPU check: parity tests + one short bench line (kernel breakdown)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --no-e2e --no-aux --steps 20 --warmup 5 > gpurun_out/b.log 2>&1; echo bench=$?
tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
