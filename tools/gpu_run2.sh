set -x
mkdir -p gpurun_out
./tools/microbench/mb2 > gpurun_out/mb2.log 2>&1
timeout 300 python tools/profile_step.py --route auto > gpurun_out/prof_auto.log 2>&1; echo p1=$?
timeout 300 python tools/profile_step.py --route diag > gpurun_out/prof_diag.log 2>&1; echo p2=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ -c 6 -o gpurun_out/cfg1_full python tools/profile_cfg1.py > gpurun_out/ncu_cfg1.log 2>&1; echo ncu=$?
