# A/B of one env switch on the same box: bash tools/gpu_ab.sh VAR "v1 v2 ..."
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for rep in 1 2; do for v in $2; do
env $1=$v timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/ab_$v.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/ab_$v.log') if l.startswith('{')][-1])
print('$1=$v', round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])
" || tail -5 gpurun_out/ab_$v.log
done; done
