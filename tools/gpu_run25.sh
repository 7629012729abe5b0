mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|assert " gpurun_out/gpu_tests.log | tail -8
timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], round(d['roofline']['frac'],3), d['e2e']['value'])
"
