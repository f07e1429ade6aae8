set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py
timeout 900 python bench.py --config C2 --steps 3 --warmup 2 --no-cpu --levels-out gpurun_out/c2_levels_v5.npz 2>&1 | tail -2 | python scripts/summarize.py
