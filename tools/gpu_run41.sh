mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/l_b16.csv python tools/one_case.py 4096 4096 16 0.9 bf16 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k 'regex:k_product' --launch-skip 2 -c 1 -o gpurun_out/prod16 -f python tools/one_case.py 4096 4096 16 0.9 bf16 > gpurun_out/ncu_p16.log 2>&1
tail -n 1 gpurun_out/ncu_p16.log
