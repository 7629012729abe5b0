mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
for nb in 8 64 256 1024; do
echo "== DIAGMM_NARROW_MAX_B=$nb DIAGMM_NARROW_DW_MAX_B=$nb"
DIAGMM_NARROW_MAX_B=$nb DIAGMM_NARROW_DW_MAX_B=$nb timeout 300 python tools/bench_kernels.py 0 2 5 6 7 9 10 2>&1 | cut -c1-120
done
DIAGMM_NARROW_MAX_B=1024 DIAGMM_NARROW_DW_MAX_B=1024 timeout 600 python -m pytest tests -m gpu -q -x -k "products or config1 or large_batch or golden or bf16" 2>&1 | tail -1
