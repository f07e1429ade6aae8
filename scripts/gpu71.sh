timeout 900 python -m pytest tests/test_device_parity.py tests/test_dist_device.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/c2_levels_v71.npz 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
