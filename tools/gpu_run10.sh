mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 3 gpurun_out/gpu_tests.log
timeout 300 python tools/probe_ln.py 2>&1 | grep -v Warn
timeout 300 python tools/profile_step.py --route auto --rows 40 > gpurun_out/prof_auto.log 2>&1; echo p1=$?
head -1 gpurun_out/prof_auto.log; grep diagmm gpurun_out/prof_auto.log | cut -c1-80,150-220
