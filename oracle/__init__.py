"""CPU float64 oracle for the DiagLinear hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy, the reference algorithm of DynaDiag's
diagonal-sparse layer (reference: /root/reference/pkg/src/diagsparse, cited
file:line in every function).  It exists so that

* ``tests/`` can check the CUDA path against it on identical inputs,
* ``__graft_entry__.smoke()`` can check one small CUDA invocation, and
* ``bench.py`` can time it as the ``cpu_baseline`` / ``--impl reference`` arm.

Nothing in the product package (``paper_2506_11449_b200``) imports, links or
executes anything from here; the product path fails loudly when its CUDA
library is missing instead of falling back to this code.

Pinning: ``tests/golden/make_golden.py`` ran the reference itself (imported
read-only from /root/reference in the build container) and committed its
outputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks
this restatement against those vectors (masks/offsets bit-exact, floats to
1e-12 relative), plus the reference's own known-answer cases.
"""

from .geometry import (  # noqa: F401
    candidate_count,
    required_diagonals,
    entry_coords,
    dense_matrix,
    transpose_diagonals,
    diag_spmm,
    csr_spmm,
)
from .topk import (  # noqa: F401
    EPS_ACTIVE,
    waterfill,
    soft_topk,
    soft_topk_grad,
    select_hard,
    temperature_at,
    sparsity_at,
    l1_term,
    allocate_budgets,
)
from .layer import (  # noqa: F401
    OracleDiagLayer,
    diag_matmul_forward,
    diag_matmul_backward,
    adamw_update,
    clip_by_global_norm,
    lr_at,
    diagheur_swap,
)
