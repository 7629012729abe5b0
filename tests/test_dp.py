"""Data-parallel host logic at world size 2 on CPU (gloo): the gradient
exchange reproduces the full-batch single-process gradient, buckets mixed
dtypes, and leaves replicas identical."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model(seed=0):
    torch.manual_seed(seed)
    m = torch.nn.Sequential(torch.nn.Linear(12, 16), torch.nn.ReLU(), torch.nn.Linear(16, 5))
    m.extra = torch.nn.Parameter(torch.randn(7, dtype=torch.float64))  # a float64 tensor, like alpha
    return m


def _loss(m, x, y):
    return torch.nn.functional.cross_entropy(m(x), y) + (m.extra ** 2).sum() * 1e-3


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_11449_b200.dp import GradientAllReducer, broadcast_parameters

    m = _model(seed=rank)  # different init on purpose: broadcast must fix it
    broadcast_parameters(m)
    g = torch.Generator().manual_seed(5)
    x = torch.randn(8, 12, generator=g)
    y = torch.randint(0, 5, (8,), generator=g)
    shard = slice(rank * 4, rank * 4 + 4)
    _loss(m, x[shard], y[shard]).backward()
    GradientAllReducer(m.parameters())()
    # numpy copies: pickled by value (tensors would be shared by fd and vanish with this process)
    q.put((rank, {n: p.grad.detach().numpy().copy() for n, p in m.named_parameters()},
           {n: p.detach().numpy().copy() for n, p in m.named_parameters()}))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_matches_full_batch_gradient():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (g, w)) for r, g, w in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: one process, full batch, rank-0 init; the DP loss is the mean of the two
    # shard losses (each shard's cross-entropy is a batch mean, as in the reference)
    m = _model(seed=0)
    g = torch.Generator().manual_seed(5)
    x = torch.randn(8, 12, generator=g)
    y = torch.randint(0, 5, (8,), generator=g)
    loss = 0.5 * (_loss(m, x[:4], y[:4]) + _loss(m, x[4:], y[4:]))
    loss.backward()
    for n, p in m.named_parameters():
        for r in (0, 1):
            torch.testing.assert_close(torch.from_numpy(res[r][0][n]), p.grad, rtol=1e-6, atol=1e-7)
            torch.testing.assert_close(torch.from_numpy(res[r][1][n]), p.detach())
        assert (res[0][0][n] == res[1][0][n]).all()  # replicas bit-identical
