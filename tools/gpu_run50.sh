mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests -m gpu -x -q -k "gelu or mlp or tc_" 2>&1 | tail -1
DIAGMM_TC_EPI_PP=0 timeout 600 python -m pytest tests -m gpu -x -q -k "gelu or mlp" 2>&1 | tail -1
for c in 1 0; do echo "pp=$c"; DIAGMM_TC_EPI_PP=$c python tools/epi_bench.py; done
for c in 1 0; do
DIAGMM_TC_EPI_PP=$c timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/bench_pp_$c.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_pp_$c.log') if l.startswith('{')][-1])
print('pp=$c', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])
" || tail -5 gpurun_out/bench_pp_$c.log
done
