timeout 900 python -m pytest tests/test_band_getrf.py -x -q 2>&1 | tail -3
timeout 1500 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu --levels-out gpurun_out/c3_levels_v46.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -4
timeout 1500 python bench.py --config C3 --plan regular:2000 --steps 2 --warmup 1 --no-cpu --levels-out gpurun_out/c3r2000_levels_v46.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
