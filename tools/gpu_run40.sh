mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for nb in 8 0; do for nd in 16 0; do
echo "--- narrow_max_b=$nb narrow_dw_max_b=$nd"
DIAGMM_NARROW_MAX_B=$nb DIAGMM_NARROW_DW_MAX_B=$nd python tools/bench_kernels.py 5 6 7 8
done; done
