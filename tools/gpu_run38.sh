mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
M="gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,launch__registers_per_thread"
for c in "4096 4096 8 0.9 bf16" "4096 4096 1 0.9 bf16" "4096 4096 64 0.9 bf16" "3072 768 256 0.9 f32"; do
n=$(echo $c | tr ' ' '_')
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l_$n.csv python tools/one_case.py $c > /dev/null 2>&1
done
