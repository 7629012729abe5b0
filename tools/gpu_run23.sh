mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], json.dumps(d['e2e']))
"
DIAGMM_DP_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-extras --batch 64 > gpurun_out/bench_dp.log 2>&1; echo dp=$?
tail -c 700 gpurun_out/bench_dp.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_dp_ref.log 2>&1; echo dpref=$?
tail -c 300 gpurun_out/bench_dp_ref.log
