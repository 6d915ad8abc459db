"""Minimal launch sequence for ncu: one warm-up + the kernels of interest
(fused exact step, propagate, collide) on the C2 tile."""
import os
import sys
sys.argv = [sys.argv[0], "--reps", "1"] + sys.argv[1:]
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kernel_variants import main  # noqa: E402
main()
