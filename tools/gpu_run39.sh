mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
ncu --set full --import-source on --clock-control none -k 'regex:k_product_narrow' --launch-skip 2 -c 1 -o gpurun_out/narrow8 -f python tools/one_case.py 4096 4096 8 0.9 bf16 > gpurun_out/ncu_n8.log 2>&1
tail -n 1 gpurun_out/ncu_n8.log
