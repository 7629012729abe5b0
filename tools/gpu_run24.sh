mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_tc_gemm|nvjet" -c 2 -o gpurun_out/tc_k768b python tools/tc_one.py 50432 3072 768 > /dev/null 2>&1; echo ncu=$?
ncu -i gpurun_out/tc_k768b.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum 2>/dev/null | cut -c1-40,170-600
