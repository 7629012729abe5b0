mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests -m gpu -x -q -k "layer_norm or ln or vit" 2>&1 | tail -1
python tools/ln_bench.py
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ln --csv python tools/ln_bench.py 2>/dev/null | grep -E "k_ln_bwd|k_ln_fwd|k_ln_fold" | tail -6
timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/b.log 2>&1; python -c "
import json
d=json.loads([l for l in open('gpurun_out/b.log') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['clocks'])"
