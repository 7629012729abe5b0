"""Per-step schedule scalars on the device, so ONE captured CUDA graph replays a
whole dynamic-sparse-training step — soft TopK re-selection at the step's
temperature and budget, forward, backward, clip and AdamW — for every step of an
annealing run.

The reference recomputes these host scalars every step: the temperature
(``temperature_at``, selection.py:189-200, clamped past the horizon by
layers.py:217-219), each layer's budget k (``_schedule_layer_budgets`` ->
``set_k``, training.py:608-619) and AdamW's bias corrections and learning rate
(training.py:346-358, 393-403).  A graph bakes its kernel arguments at capture
time, so here the host computes the same floats (same Python arithmetic as the
reference) and writes them into one small device buffer before each replay
(pinned double buffer, stream-ordered async copy); K4, K5 and the AdamW kernel
read them from there (``diagmm_topk_job.params``, ``diagmm_topk_grad`` /
``diagmm_adamw_multi`` ``params`` / ``sched``).

Buffer layout (float64): [lr, 1 - beta1^t, 1 - beta2^t, T_0, k_0, T_1, k_1, ...].
"""

from __future__ import annotations

import torch

from .errors import NonPositiveTemperature


class DeviceSchedule:
    """Device copy of a training step's schedule scalars for ``model``'s DiagLinear
    layers and (optionally) an ``optim.AdamW``."""

    def __init__(self, model: torch.nn.Module, optimizer=None):
        from .layer import DiagLinear

        seen, self.layers = set(), []
        for m in model.modules():
            if isinstance(m, DiagLinear) and id(m) not in seen:
                seen.add(id(m))
                self.layers.append(m)
        dev = self.layers[0].alpha.device if self.layers else torch.device("cuda")
        n = 3 + 2 * len(self.layers)
        self.dev = torch.zeros(n, dtype=torch.float64, device=dev)
        self._host = [torch.zeros(n, dtype=torch.float64).pin_memory() for _ in range(2)]
        self._events = [None, None]
        self._i = 0
        self.opt = optimizer
        for j, m in enumerate(self.layers):
            m._sched_params = self.dev[3 + 2 * j: 5 + 2 * j]

    @property
    def adam(self) -> torch.Tensor:
        """{lr, 1 - beta1^t, 1 - beta2^t} for ``AdamW.step(sched=...)``."""
        return self.dev[0:3]

    def set_step(self, step: int, lr: float | None = None) -> None:
        """Write step ``step``'s scalars: every layer's T(step) and current k (after any
        ``set_k`` / ``schedule_layer_budgets``), and the optimizer's learning rate and
        bias corrections for its next update (t = host step count + 1).  Stream-ordered
        with the work that follows on the current stream."""
        vals = [0.0, 0.0, 0.0]
        if self.opt is not None:
            b1, b2 = self.opt.betas
            t = self.opt.next_step()
            vals = [float(self.opt.lr if lr is None else lr), 1.0 - b1 ** t, 1.0 - b2 ** t]
        for m in self.layers:
            T = m.temperature(step)
            if not T > 0.0:
                raise NonPositiveTemperature(f"temperature must be positive, got {T}")
            if not 1 <= m.k <= m.candidates:
                raise ValueError(f"k={m.k} outside [1, {m.candidates}]")
            vals += [T, float(m.k)]
        b = self._i % 2
        if self._events[b] is not None:
            self._events[b].synchronize()  # the copy that last read this pinned buffer is done
        buf = self._host[b]
        buf.copy_(torch.tensor(vals, dtype=torch.float64))
        self.dev.copy_(buf, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev.device))
        self._events[b] = ev
        self._i += 1

    def detach(self) -> None:
        for m in self.layers:
            m._sched_params = None
