mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for gm in auto off; do
timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 --graph $gm > gpurun_out/bg_$gm.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bg_$gm.log') if l.startswith('{')][-1])
print('graph=$gm', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'], d['clocks']['sm_mhz'], 'roof', round(d['roofline']['frac'],3))
" || tail -12 gpurun_out/bg_$gm.log
done
