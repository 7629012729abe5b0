# current-kernel launch list for config 1 (fp32) and a bf16 mid-batch case
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio"
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/cfg1_f32.csv python tools/one_case.py 3072 768 256 0.9 f32 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/b64_bf16.csv python tools/one_case.py 4096 4096 64 0.9 bf16 > /dev/null 2>&1
python tools/bench_kernels.py > gpurun_out/bk.log 2>&1; tail -40 gpurun_out/bk.log
