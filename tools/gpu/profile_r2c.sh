# Round-2 final evidence (box-form K2, lattice K1): bench line + reference arm, ncu launch
# list, ncu --set full of every step kernel (+ DRAM bytes per launch), all configs.
mkdir -p gpurun_out
python bench.py > gpurun_out/r2c_bench.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c_bench_ref.log 2>&1; echo ref=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/r2c_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2c_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux \
    > gpurun_out/r2c_ncu_launch.log 2>&1; echo launches=$?
python tools/ncu_summary.py gpurun_out/r2c_launches.csv > gpurun_out/r2c_launches.txt 2>&1
python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/r2c_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"element_kernel|node_sum|mlp_tc_kernel|scatter_update|prolongate" -s 5 -c 5 \
    -o gpurun_out/r2c_step_full -f python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/r2c_ncu_full.log 2>&1; echo full=$?
python tools/ncu_summary.py gpurun_out/r2c_step_full.ncu-rep > gpurun_out/r2c_kernels_ncu.txt 2>&1
python tools/ncu_traffic.py gpurun_out/r2c_step_full.ncu-rep > gpurun_out/r2c_dram_traffic.json 2>&1
bash tools/gpu/all_configs.sh > gpurun_out/r2c_all_configs.jsonl 2>&1
tail -1 gpurun_out/r2c_bench.log | head -c 300
