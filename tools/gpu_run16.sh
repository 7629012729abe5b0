mkdir -p gpurun_out
timeout 120 python tools/tc_check.py > gpurun_out/tc.log 2>&1; echo tc=$?
cat gpurun_out/tc.log | tail -20
