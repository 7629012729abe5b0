mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 3 gpurun_out/gpu_tests.log
timeout 600 python tools/bench_kernels.py > gpurun_out/kern.log 2>&1; echo kern=$?
cat gpurun_out/kern.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_product|k_dw|k_prescale" -c 10 -o gpurun_out/v5_cfg1 python tools/one_case.py 3072 768 256 0.9 f32 > /dev/null 2>&1; echo ncu1=$?
