# ncu --set full of one tensor-core K2 launch at config-3 size (after a plain run exits 0)
mkdir -p gpurun_out
python tools/gpu/k2_time.py 64x32x32 > gpurun_out/k2t_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2tc_kernel -s 2 -c 1 \
    -o gpurun_out/k2tc python tools/gpu/k2_time.py 64x32x32 > gpurun_out/ncu_k2tc.log 2>&1
echo rc=$?
python tools/ncu_summary.py gpurun_out/k2tc.ncu-rep > gpurun_out/k2tc_summary.txt 2>&1
head -60 gpurun_out/k2tc_summary.txt
