mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for e in 0 1; do
ncu --set full --import-source on --clock-control none -k 'regex:k_tc_gemm' --launch-skip 1 -c 1 -o gpurun_out/tc2_epi$e -f python tools/tc_epi_one.py $e > /dev/null 2>&1
done
ls gpurun_out/tc2_epi*
