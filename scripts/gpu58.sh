timeout 900 python -m pytest tests/test_band_getrf.py tests/test_device_parity.py -x -q 2>&1 | tail -2
timeout 1500 python scripts/balance_bench.py C5 --sizes 200,500,2000 --repeats 3 2>&1 | grep "^#" | cut -c1-300
timeout 900 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu --levels-out gpurun_out/c5_levels_v58.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
