mkdir -p gpurun_out
python - <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_2506_11449_b200.vit import PackedQKVAttention
import torch.nn.functional as F
B,T,H,hd=4,197,12,64
h=torch.randn(B,T,3,H,hd,device="cuda",dtype=torch.bfloat16,requires_grad=True)
out=PackedQKVAttention.apply(h)
g=torch.randn_like(out)
out.backward(g)
h2=h.detach().clone().requires_grad_(True)
q,k,v=h2.permute(2,0,3,1,4).unbind(0)
o2=F.scaled_dot_product_attention(q.float(),k.float(),v.float())
o2.backward(g.float())
print("fwd err", (out.float()-o2).abs().max().item(), "bwd err", (h.grad.float()-h2.grad).abs().max().item(), h2.grad.abs().max().item())
PY
for be in cudnn flash; do
DIAGMM_VIT_ATTENTION=$be timeout 900 python bench.py --no-cpu-baseline --no-extras --steps 10 > gpurun_out/bench_$be.log 2>&1
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_$be.log') if l.startswith('{')][-1])
print('$be', d['value'], d['ms_per_step'])
" || tail -5 gpurun_out/bench_$be.log
done
