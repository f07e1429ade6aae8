# quick perf check (run under gpurun): GPU parity tests + C2 bench line summary
timeout 900 python -m pytest tests/test_device_parity.py tests/test_band_getrf.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
