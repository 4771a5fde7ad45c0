mkdir -p gpurun_out
python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 1 -c 1 \
    -o gpurun_out/mlpprof python tools/gpu/step_run.py 64x32x32 2 > gpurun_out/ncu_mlp.log 2>&1
echo rc=$?
tail -2 gpurun_out/ncu_mlp.log
