# Round-end evidence: GPU tests, smoke, full bench (both arms), ncu launch list of the bench command,
# ncu --set full of the dominant SURVEY-§8 kernels, kernel sweep.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -n 2 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
timeout 600 python tools/bench_kernels.py > gpurun_out/kern.log 2>&1; echo kern=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo ncul=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_materialize|k_tc_gemm" -c 6 -o gpurun_out/dominant_full python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo ncuf=$?
