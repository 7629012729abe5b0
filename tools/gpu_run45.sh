mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
python tools/bench_kernels.py 0 1 2 3 9 10
echo "--- FW wide"
DIAGMM_FW_WIDE=1 python tools/bench_kernels.py 0 1 2 3 9 10
