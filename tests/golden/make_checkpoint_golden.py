"""Golden checkpoint fixture produced by the REFERENCE itself (training.py:721-766).

Run in the build container (the reference is mounted read-only there):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \\
        python tests/golden/make_checkpoint_golden.py

Builds the reference's MLPModel (DynaDiag / DynaDiag / dense, 48 -> 64 -> 40 -> 6),
perturbs alpha and values so hard top-K and the baked soft scores are
non-trivial, writes ``ref_checkpoint.json`` with the reference's own
``save_checkpoint`` and ``ref_checkpoint_io.npz`` with features and the
reference InferenceModel's logits (``load_checkpoint`` -> ``predict_logits``).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("DIAGSPARSE_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from diagsparse import training  # noqa: E402
from diagsparse.selection import TemperatureSchedule  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    cfg = training.TrainConfig(model=training.ModelConfig(layer_sizes=(48, 64, 40, 6),
                                                          layer_kinds=("dynadiag", "dynadiag", "dense")),
                               sparsity=0.8, t_schedule=TemperatureSchedule("cosine", 2.0, 0.05, 10), seed=3)
    model = training.build_model(cfg, 10)
    rng = np.random.default_rng(5)
    for layer in model.layers:
        if hasattr(layer, "alpha"):
            layer.alpha.value = layer.alpha.value + rng.standard_normal(layer.alpha.value.shape)
            layer.values.value = layer.values.value + 0.1 * rng.standard_normal(layer.values.value.shape)
        if getattr(layer, "bias", None) is not None:
            layer.bias.value = 0.1 * rng.standard_normal(layer.bias.value.shape)
    path = OUT / "ref_checkpoint.json"
    training.save_checkpoint(model, cfg, str(path))
    inf, _ = training.load_checkpoint(str(path))
    x = rng.standard_normal((9, 48))
    np.savez(OUT / "ref_checkpoint_io.npz", x=x, logits=inf.predict_logits(x))


if __name__ == "__main__":
    main()
