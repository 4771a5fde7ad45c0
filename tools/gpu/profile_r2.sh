# Round-2 evidence (run on the GPU box): bench line + launch list, ncu of every step kernel,
# the tensor-core K2 study (timing, timeline, ncu + per-line attribution), tcgen05 probes.
mkdir -p gpurun_out
python bench.py > gpurun_out/r2_bench.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; echo ref=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/r2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-aux \
    > gpurun_out/r2_ncu_launch.log 2>&1; echo launches=$?
python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/r2_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"element_kernel|node_sum|mlp_tc_kernel|scatter_update|prolongate_owner" -s 5 -c 5 \
    -o gpurun_out/r2_step_full python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/r2_ncu_full.log 2>&1; echo full=$?
python tools/ncu_summary.py gpurun_out/r2_step_full.ncu-rep > gpurun_out/r2_kernels_ncu.txt 2>&1
python tools/gpu/k2_time.py 64x32x32 > gpurun_out/r2_k2tc_time.txt 2>&1
DNNMG_K2=tc python tools/gpu/k2_time.py 64x32x32 jit >> gpurun_out/r2_k2tc_time.txt 2>&1
python tools/gpu/k2_repeat.py >> gpurun_out/r2_k2tc_time.txt 2>&1
python tools/gpu/k2_err.py >> gpurun_out/r2_k2tc_time.txt 2>&1
python tools/gpu/k2_trace.py > gpurun_out/r2_k2tc_trace.txt 2>&1
bash tools/gpu/ncu_k2tc.sh > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/k2tc.ncu-rep > gpurun_out/r2_k2tc_ncu.txt 2>&1
python tools/ncu_lines.py gpurun_out/k2tc.ncu-rep 40 >> gpurun_out/r2_k2tc_ncu.txt 2>&1
./tools/ubench/tc_probe > gpurun_out/r2_tc_probe.txt 2>&1
./tools/ubench/mma_issue > gpurun_out/r2_mma_issue.txt 2>&1
tail -1 gpurun_out/r2_bench.log | head -c 400
