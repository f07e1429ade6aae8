timeout 900 python bench.py --config C2 --steps 2 --warmup 1 --no-cpu --levels-out gpurun_out/c2_levels_v20.npz 2>&1 | tail -1 | python scripts/summarize.py | head -3
