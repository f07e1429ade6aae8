timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/c2_levels_v69.npz 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python scripts/trace_levels.py C2 2>&1 | tail -14
