mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
ncu --set full --import-source on --clock-control none -k 'regex:^k_dw$' -c 1 -o gpurun_out/cfg1_dw -f python tools/one_case.py 3072 768 256 0.9 f32 > gpurun_out/ncu2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg1_f32.csv python tools/one_case.py 3072 768 256 0.9 f32 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/b1_s99.csv python tools/one_case.py 4096 4096 1 0.99 bf16 > /dev/null 2>&1
tail -n 3 gpurun_out/ncu2.log
