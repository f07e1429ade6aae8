timeout 900 python -m pytest tests/test_dist_device.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python scripts/micro_getrf.py 2048 2048 3 --trace 2>&1 | tail -14
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/c2_levels_v29.npz 2>&1 | tail -1 | python scripts/summarize.py | head -3
