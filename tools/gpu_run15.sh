mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], json.dumps(d['roofline'])); print(d['routes']); print(d['infer'])
"
timeout 600 ncu --set full --clock-control none -k regex:"k_adamw_multi|k_gather|k_materialize" -c 4 -o gpurun_out/step_ours2 python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo ncuf=$?
ncu -i gpurun_out/step_ours2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum 2>/dev/null | cut -c1-50,180-320
