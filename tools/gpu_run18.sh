mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none -k regex:"k_tc_gemm|nvjet" -c 2 -o gpurun_out/tc_k768 python tools/tc_one.py 50432 3072 768 > /dev/null 2>&1; echo ncu=$?
ncu -i gpurun_out/tc_k768.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,launch__grid_size,launch__cluster_dim_x,sm__throughput.avg.pct_of_peak_sustained_elapsed 2>/dev/null | cut -c1-40,170-600
