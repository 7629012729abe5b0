mkdir -p gpurun_out
timeout 300 python tools/kernel_smoke.py > gpurun_out/ks.log 2>&1; echo ks=$?
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python tools/bench_kernels.py > gpurun_out/kern.log 2>&1; echo kern=$?
tail -n 4 gpurun_out/ks.log gpurun_out/gpu_tests.log; cat gpurun_out/kern.log
