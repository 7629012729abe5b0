mkdir -p gpurun_out
for mode in 0 bwd 1; do
DIAGMM_FUSE_MLP=$mode timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/bench_$mode.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_$mode.log') if l.startswith('{')][-1])
print('$mode', d['value'], d['ms_per_step'])
"
done
