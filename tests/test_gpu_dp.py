"""The compact data-parallel exchange (dp.CompactGradExchange) on a
one-GPU box: two processes share cuda:0 over gloo, each takes half the batch.

* the exchanged gradients equal the single-process full-batch gradients
  (DiagLinear values / alpha / bias and the dense parameters), on both the fp32
  FMA route and the bf16 tensor-core route (K3 writes the buckets in both);
* only the compact payload crosses the wire (bytes counted by the exchange);
* after clip + AdamW the two replicas are bit-identical.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build(kind):
    from paper_2506_11449_b200 import TemperatureSchedule
    from paper_2506_11449_b200.vit import MLPModel

    T = TemperatureSchedule("constant", 0.05, 0.05, 1)
    torch.manual_seed(0)
    if kind == "fp32":
        m = MLPModel(sizes=(256, 768, 256, 10), kinds=("dynadiag", "dynadiag", "dense"), t_schedule=T,
                     dtype=torch.float32)
    else:
        m = MLPModel(sizes=(256, 1024, 512, 10), kinds=("dynadiag", "dynadiag", "dense"), t_schedule=T,
                     dtype=torch.float32)
        for lyr in m.layers[:2]:
            lyr.route = "auto"
    for i, lyr in enumerate(m.layers[:2]):
        rng = np.random.default_rng(40 + i)
        with torch.no_grad():
            lyr.alpha.add_(torch.as_tensor(rng.standard_normal(lyr.candidates), device="cuda"))
    return m


def _data(kind):
    g = torch.Generator(device="cuda").manual_seed(9)
    n = 64 if kind == "fp32" else 2048  # bf16: 1024 tokens per rank -> tensor-core route
    x = torch.randn(n, 256, device="cuda", generator=g)
    y = torch.randint(0, 10, (n,), device="cuda", generator=g)
    return x, y


def _loss(m, x, y, kind, fused=True):
    import torch.nn.functional as F

    from paper_2506_11449_b200 import penalties

    if kind == "bf16":
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = m(x.to(torch.bfloat16), 0)
    else:
        out = m(x, 0)
    loss = F.cross_entropy(out.float(), y)
    for p in penalties(m, fused=fused):  # fused: the l1 gradient is added by K5 at unit loss weight
        loss = loss + p
    return loss


def _worker(rank, world, port, kind, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_11449_b200 import AdamW, GlobalNormClipper, model_param_specs
    from paper_2506_11449_b200.dp import CompactGradExchange, broadcast_parameters

    m = _build(kind)
    broadcast_parameters(m)
    ex = CompactGradExchange(m)
    x, y = _data(kind)
    h = x.shape[0] // world
    _loss(m, x[rank * h:(rank + 1) * h], y[rank * h:(rank + 1) * h], kind).backward()
    ex.finish()
    n_act = [lyr._last_spec.sel.host_count() for lyr in m.layers[:2]]  # the selection this step used
    grads = {n: p.grad.detach().double().cpu().numpy().copy() for n, p in m.named_parameters()}
    specs = model_param_specs(m)
    _, sc = GlobalNormClipper(1.0).compute(specs)
    AdamW(specs, lr=1e-2).step(clip_scale=sc)
    torch.cuda.synchronize()
    params = {n: p.detach().double().cpu().numpy().copy() for n, p in m.named_parameters()}
    q.put((rank, grads, params, ex.bytes_last, n_act))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["fp32", "bf16"])
def test_compact_exchange_matches_full_batch(kind):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: rest for r, *rest in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # reference: one process, the full batch; the DP loss is the mean of the shard losses
    m = _build(kind)
    x, y = _data(kind)
    h = x.shape[0] // 2
    loss = 0.5 * (_loss(m, x[:h], y[:h], kind, False) + _loss(m, x[h:], y[h:], kind, False))
    loss.backward()
    tol = 1e-5 if kind == "fp32" else 2e-3
    for n, p in m.named_parameters():
        want = p.grad.detach().double().cpu().numpy()
        for r in (0, 1):
            got = res[r][0][n]
            assert np.abs(got - want).max() <= tol * max(1e-3, np.abs(want).max()), (n, r)
        assert np.array_equal(res[0][0][n], res[1][0][n]), n  # identical exchanged gradients
        assert np.array_equal(res[0][1][n], res[1][1][n]), n  # replicas bit-identical after AdamW
    # compact payload: active rows of each DiagLinear, alpha, bias, dense params — not (C, L)
    lay = m.layers[:2]
    compact = sum(na * lyr.diag_len * 4 + lyr.candidates * 8 + lyr.out_features * 4
                  for na, lyr in zip(res[0][3], lay))
    compact += sum(p.numel() * 4 for p in m.layers[2].parameters())
    assert res[0][2] == compact, (res[0][2], compact)
    full = sum(p.numel() * p.element_size() for p in m.parameters())
    assert res[0][2] < 0.5 * full
