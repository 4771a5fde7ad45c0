# end-of-round check: full GPU test suite, smoke, all configs, config-4 sweep
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
bash tools/gpu/all_configs.sh > gpurun_out/r2c_all_configs.jsonl 2>&1
timeout 900 python bench.py --mlp-sweep > gpurun_out/r2c_sweep.log 2>&1; echo sweep=$?
tail -1 gpurun_out/r2c_sweep.log > gpurun_out/r2c_mlp_sweep_cfg4.json
