mkdir -p gpurun_out
python tools/gpu/step_run.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:element_kernel -s 1 -c 1 \
    -o gpurun_out/k2prof python tools/gpu/step_run.py > gpurun_out/ncu_k2.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_k2.log
