timeout 900 python -m pytest tests/test_device_solve.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu --levels-out gpurun_out/c5_levels_v42.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -4
