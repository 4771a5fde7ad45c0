mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_gather.py -x -q > gpurun_out/t_fused.log 2>&1; echo fused=$?
tail -3 gpurun_out/t_fused.log
for v in "" "DNNMG_NO_STAGED=1" "DNNMG_Y_DIRECT=1"; do
  env $v python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/b.log 2>&1
  echo "$v"; tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
done
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
