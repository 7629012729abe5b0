mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
python tools/bench_kernels.py > gpurun_out/bk.log 2>&1; cat gpurun_out/bk.log | tail -20
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
