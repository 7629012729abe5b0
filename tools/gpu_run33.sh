mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for f in 0 bwd 1; do
DIAGMM_FUSE_MLP=$f timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/bench_fuse_$f.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_fuse_$f.log') if l.startswith('{')][-1])
print('fuse=$f', d['value'], d['ms_per_step'])
" || tail -5 gpurun_out/bench_fuse_$f.log
done
sed -i 's/max_name_column_width=70/max_name_column_width=160/' tools/profile_step.py
python tools/profile_step.py --rows 60 > gpurun_out/step_prof_wide.txt 2>&1
