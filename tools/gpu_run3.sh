mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 300 python tools/profile_step.py --route auto --rows 60 > gpurun_out/prof_auto.log 2>&1; echo p1=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/bench.log 2>&1; echo bench=$?
tail -n 5 gpurun_out/gpu_tests.log
