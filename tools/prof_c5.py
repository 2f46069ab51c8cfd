"""The papers100M-shape epoch (bench_models.run_papers100m) with one warm-up
and one timed step, for ncu: python tools/prof_c5.py [scale]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import bench_models as bm  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
r = bm.run_papers100m(steps=1, warmup=1, scale=scale)
print(r["ms"], r["rank0_kernels_ms"])
