timeout 900 python -m pytest tests/test_band_getrf.py tests/test_device_parity.py tests/test_dist_device.py -x -q 2>&1 | tail -3
timeout 1500 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu --levels-out gpurun_out/c3_levels_v47.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
timeout 1500 python scripts/balance_bench.py C5 --sizes 500,2000 --repeats 3 2>&1 | grep "^#" | cut -c1-300
