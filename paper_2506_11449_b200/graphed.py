"""Forward + backward of a training step as one CUDA graph (the step's launch-bound
chain of ~400 kernels replayed without host work or inter-launch gaps).

The captured part is everything up to the gradients: TopK re-selection, DiagLinear
products, the caller's attention / LayerNorm / loss and the backward.  The optimizer
stays eager because the Adam step count (bias corrections) changes every step.  The
capture is valid while the per-step host arguments it bakes in stay fixed: the soft
TopK temperature (a constant schedule) and the l1 coefficients; inputs are copied into
the captured buffers before each replay."""

from __future__ import annotations

import torch

from . import _lib


class GraphedStep:
    """``fwd_bwd(inputs...) -> loss`` captured once; ``step(*inputs)`` copies the inputs
    into the captured buffers (when they are other tensors), replays, returns the
    captured loss tensor.  Gradients stay in the graph's static tensors (``.grad`` of
    the parameters), overwritten by every replay."""

    def __init__(self, fwd_bwd, params, *static_inputs: torch.Tensor, warmup: int = 1):
        self.inputs = static_inputs
        dev = static_inputs[0].device
        for p in params:
            p.grad = None
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm the side stream's allocator pool
            for _ in range(warmup):
                fwd_bwd(*static_inputs)
                for p in params:
                    p.grad = None
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        n0 = _lib.load().diagmm_launch_count()
        with torch.cuda.graph(self.graph):
            self.loss = fwd_bwd(*static_inputs)
        self.launches = _lib.load().diagmm_launch_count() - n0  # our kernels per replay
        torch.cuda.synchronize(dev)

    def step(self, *inputs: torch.Tensor) -> torch.Tensor:
        for dst, src in zip(self.inputs, inputs):
            if src is not dst:
                dst.copy_(src, non_blocking=True)
        self.graph.replay()
        return self.loss


def schedules_constant(model: torch.nn.Module) -> bool:
    """True when every DiagLinear's temperature is the same at every step."""
    from .layer import DiagLinear

    return all(m.t_schedule.kind == "constant" or m.t_schedule.t_init == m.t_schedule.t_final
               for m in model.modules() if isinstance(m, DiagLinear))


class GraphedTrainStep:
    """The WHOLE training step — soft TopK re-selection, forward, backward, global-norm
    clip and AdamW — captured as ONE CUDA graph and replayed for every step of an
    annealing / sparsity schedule: the per-step scalars (temperature, k, learning
    rate, Adam bias corrections) come from ``schedule.DeviceSchedule``'s device buffer,
    which ``step()`` refreshes (stream-ordered) before each replay.

    ``fwd_bwd(*inputs)`` runs forward + backward and returns what the caller wants
    back (loss, outputs); it must not read anything back to the host.  The warm-up
    (allocator pools, library handles) runs forward + backward only, so the
    parameters are untouched until the first ``step()``."""

    def __init__(self, fwd_bwd, specs, optimizer, clipper, schedule, *static_inputs, warmup: int = 1,
                 first_step: int = 0):
        self.inputs, self.opt, self.sched = static_inputs, optimizer, schedule
        dev = static_inputs[0].device
        for s in specs:
            s.tensor.grad = None
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                schedule.set_step(first_step)
                fwd_bwd(*static_inputs)
                for s in specs:
                    s.tensor.grad = None
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        n0 = _lib.load().diagmm_launch_count()
        steps0 = [st["t"] for st in optimizer.state]
        with torch.cuda.graph(self.graph):
            self.out = fwd_bwd(*static_inputs)
            self.norm, scale = clipper.compute(specs)
            optimizer.step(clip_scale=scale, sched=schedule.adam)
        for st, t0 in zip(optimizer.state, steps0):  # capture ran no update: undo its host bookkeeping
            st["t"] = t0
        self.launches = _lib.load().diagmm_launch_count() - n0
        torch.cuda.synchronize(dev)

    def step(self, step: int, *inputs: torch.Tensor, lr: float | None = None):
        self.sched.set_step(step, lr=lr)
        for dst, src in zip(self.inputs, inputs):
            if src is not dst:
                dst.copy_(src, non_blocking=True)
        self.graph.replay()
        self.opt.advance_steps()
        return self.out
