# Round-2 evidence after the K4 changes (NQ = 4, BN-scale fold, probes compiled out): bench
# line + reference arm, ncu launch list, ncu --set full of every step kernel, all configs.
mkdir -p gpurun_out
python bench.py > gpurun_out/r2b_bench.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b_bench_ref.log 2>&1; echo ref=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/r2b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux \
    > gpurun_out/r2b_ncu_launch.log 2>&1; echo launches=$?
python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/r2b_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"element_kernel|node_sum|mlp_tc_kernel|scatter_update|prolongate_owner" -s 5 -c 5 \
    -o gpurun_out/r2b_step_full python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/r2b_ncu_full.log 2>&1; echo full=$?
python tools/ncu_summary.py gpurun_out/r2b_step_full.ncu-rep > gpurun_out/r2b_kernels_ncu.txt 2>&1
bash tools/gpu/all_configs.sh > gpurun_out/r2b_all_configs.jsonl 2>&1
python tools/gpu/k2_time.py 64x32x32 > gpurun_out/r2b_k2tc_time.txt 2>&1
python tools/gpu/k2_time.py 64x32x32 jit >> gpurun_out/r2b_k2tc_time.txt 2>&1
tail -1 gpurun_out/r2b_bench.log | head -c 300
