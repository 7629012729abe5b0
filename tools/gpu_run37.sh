mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests -m gpu -x -q -k "gelu or mlp or tc_" 2>&1 | tail -2
DIAGMM_TC_PINGPONG=1 timeout 600 python -m pytest tests -m gpu -x -q -k "tc_" 2>&1 | tail -2
for pp in 0 1; do
echo "pingpong=$pp"; DIAGMM_TC_PINGPONG=$pp python tools/epi_bench.py
DIAGMM_TC_PINGPONG=$pp timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/bench_pp_$pp.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_pp_$pp.log') if l.startswith('{')][-1])
print('pp=$pp', d['value'], d['ms_per_step'])
" || tail -5 gpurun_out/bench_pp_$pp.log
done
