mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 3 gpurun_out/gpu_tests.log
timeout 300 python tools/probe_attn.py 2>&1 | grep -v Warn | tail -3
timeout 300 python tools/profile_step.py --route auto --rows 30 > gpurun_out/prof_auto.log 2>&1; echo p1=$?
head -1 gpurun_out/prof_auto.log; grep -E "^ *(void|diagmm|nvjet|cudnn|autograd|aten::copy_|aten::cat|aten::mm|aten::addmm)" gpurun_out/prof_auto.log | cut -c1-75,150-215 | head -30
