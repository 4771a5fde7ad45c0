# Round-end evidence: full bench line, reference arm, ncu launch list of the bench,
# one ncu --set full capture per step kernel (config 3 step driver).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"element_kernel|node_sum|mlp_tc_kernel|scatter_update|prolongate_owner" -s 5 -c 5 \
    -o gpurun_out/step_full python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/ncu_full.log 2>&1; echo full=$?
tail -1 gpurun_out/bench_full.log
