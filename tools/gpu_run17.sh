mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -n 8 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], json.dumps(d['roofline']))
"
DIAGMM_DENSE_BACKEND=cublas timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_cublas.log 2>&1; echo benchc=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_cublas.log') if l.startswith('{')][-1])
print('cublas backend', d['value'], d['ms_per_step'])
"
