# ncu --set full of one K1 launch at config 3 (64x32x32 coarse box)
mkdir -p gpurun_out
python tools/gpu/step_run.py 64x32x32 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:prolongate -s 1 -c 1 \
    -o gpurun_out/k1prof -f python tools/gpu/step_run.py 64x32x32 3 > gpurun_out/ncu_k1.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_k1.log
