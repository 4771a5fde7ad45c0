mkdir -p gpurun_out
DNNMG_MLP_TRACE=gpurun_out/mlp_trace.bin python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b_trace.log 2>&1; echo rc=$?
python tools/mlp_trace.py gpurun_out/mlp_trace.bin > gpurun_out/mlp_trace.txt 2>&1
