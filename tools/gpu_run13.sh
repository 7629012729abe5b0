mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"narrow|k_dw|finalize|colsum" -c 12 -o gpurun_out/narrow python tools/one_case.py 4096 4096 1 0.9 bf16 > /dev/null 2>&1; echo ncu=$?
ncu -i gpurun_out/narrow.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active 2>/dev/null | cut -c1-60,170-400
