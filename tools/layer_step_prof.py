"""ncu target: BASELINE config 1's DiagLinear step (K4 + fwd + dX + dW + K5, fp32,
B = 256) as the bench times it, eager then graphed; per-kernel times come from
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/layer_step_prof.py"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import profiling

print(profiling.layer_step_case(reps=3))
