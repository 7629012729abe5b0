"""paper_2506_11449_b200 — DynaDiag's diagonal-sparse linear layer on B200 (sm_100a).

The package is the drop-in replacement for the reference's DiagLinear hot path
(``DynaDiagLayer`` + its custom op + the DST mask-update API, reference
``pkg/src/diagsparse/layers.py`` / ``selection.py``): Python/PyTorch host code
over a thin C ABI (``include/diagmm.h``) into hand-written sm_100a kernels
(``csrc/``).  There is no CPU fallback: importing works anywhere, but every op
raises ``NativeLibraryError`` without the built library and a CUDA device.
"""

from .errors import (  # noqa: F401
    DiagSparseError,
    EmptyLayerList,
    NativeLibraryError,
    NonPositiveTemperature,
    ShapeMismatch,
    StepOutOfRange,
)
from .selection import (  # noqa: F401
    EPS_ACTIVE,
    BudgetAllocation,
    SparsitySchedule,
    TemperatureSchedule,
    allocate_budgets,
    candidate_count,
    layer_diagonal_counts,
    required_diagonals,
    schedule_layer_budgets,
    select_hard,
    soft_topk,
    soft_topk_grad,
    sparsity_at,
    temperature_at,
)
from .layer import (  # noqa: F401
    DiagHeurLinear,
    DiagLinear,
    DiagMatrix,
    DiagMMFunction,
    DiagMLP,
    FrozenDiagLinear,
    ParamSpec,
    deferred_topk_grads,
    diagheur_update,
    penalties,
    preselect,
)
from .optim import AdamW, GlobalNormClipper, lr_at, model_param_specs  # noqa: F401

__version__ = "0.1.0"
