mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['routes']['step_ms_by_fn'] if 'routes' in d else '')
"
timeout 300 python tools/profile_step.py --route auto --rows 25 > gpurun_out/prof_auto.log 2>&1
head -1 gpurun_out/prof_auto.log; grep -E "k_ln|k_tc|nvjet|flash|reduce_kernel|Gelu" gpurun_out/prof_auto.log | cut -c1-70,150-215
