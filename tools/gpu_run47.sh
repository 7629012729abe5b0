mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests -m gpu -x -q -k "gelu or mlp or tc_" 2>&1 | tail -1
DIAGMM_TC_EPI_CFG=0 timeout 600 python -m pytest tests -m gpu -x -q -k "gelu or mlp" 2>&1 | tail -1
for c in 1 0; do echo "epi_cfg=$c"; DIAGMM_TC_EPI_CFG=$c python tools/epi_bench.py; done
for c in 1 0; do
DIAGMM_TC_EPI_CFG=$c timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/bench_ec_$c.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_ec_$c.log') if l.startswith('{')][-1])
print('epi_cfg=$c', d['value'], d['ms_per_step'])
" || tail -5 gpurun_out/bench_ec_$c.log
done
