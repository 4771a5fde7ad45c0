# CTA-0 timeline of the fused MLP kernel: the probes are compiled in only by this build
# (-DDNNMG_MLP_TRACE_BUILD), so the library is rebuilt with them and restored afterwards.
mkdir -p gpurun_out
rm -f build/mlp_tc.o && make EXTRA=-DDNNMG_MLP_TRACE_BUILD > gpurun_out/trace_build.log 2>&1 || { cat gpurun_out/trace_build.log; exit 1; }
DNNMG_MLP_TRACE=gpurun_out/mlp_trace.bin python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b_trace.log 2>&1; echo rc=$?
python tools/mlp_trace.py gpurun_out/mlp_trace.bin > gpurun_out/mlp_trace.txt 2>&1
rm -f build/mlp_tc.o && make > /dev/null 2>&1
