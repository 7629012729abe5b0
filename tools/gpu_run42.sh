mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/bench_kernels.py 0 1 2 5 6 7 8 9 10 11
echo "--- FW off"
DIAGMM_FW_MAX_RB=0 python tools/bench_kernels.py 0 2 6 7 9
