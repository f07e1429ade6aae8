python scripts/micro_getrf.py 2048 2048 3 --trace 2>&1 | head -7
timeout 900 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -3
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/c2_levels_v22.npz 2>&1 | tail -1 | python scripts/summarize.py | head -2
