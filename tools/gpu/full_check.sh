mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu/ab_k4.sh
python bench.py > gpurun_out/r2b_bench.log 2>&1; tail -1 gpurun_out/r2b_bench.log | head -c 600
