mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 2 gpurun_out/gpu_tests.log
timeout 600 python tools/bench_kernels.py > gpurun_out/kern.log 2>&1; echo kern=$?
cat gpurun_out/kern.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_adamw_multi|k_gather|k_materialize|k_topk_grad|k_waterfill" -c 12 -o gpurun_out/step_ours python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo ncuf=$?
