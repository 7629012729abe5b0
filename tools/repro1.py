import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2506_11449_b200 import DiagLinear, TemperatureSchedule, ops
T=float(sys.argv[1]); n=int(sys.argv[2])
lyr = DiagLinear(768, 768, 0.9, seed=1, l1_coeff=0.0, route="auto", t_schedule=TemperatureSchedule("constant", T, T, 1))
rng = np.random.default_rng(101)
with torch.no_grad():
    lyr.alpha.add_(torch.as_tensor(rng.standard_normal(lyr.candidates), device="cuda"))
sel = lyr.selection(0); print("n_act", sel.host_count(), "k", lyr.k, flush=True)
x = torch.randn(n, 768, device="cuda").to(torch.bfloat16).requires_grad_(True)
r = torch.randn(n, 768, device="cuda").to(torch.bfloat16).requires_grad_(True)
y = lyr(x, step=0, residual=r); torch.cuda.synchronize(); print("fwd ok", flush=True)
y.backward(torch.randn_like(y)); torch.cuda.synchronize(); print("bwd ok", flush=True)
