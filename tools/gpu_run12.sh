mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 3 gpurun_out/gpu_tests.log
timeout 600 python tools/bench_kernels.py > gpurun_out/kern.log 2>&1; echo kern=$?
cat gpurun_out/kern.log
