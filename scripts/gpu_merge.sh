timeout 900 python -m pytest tests/test_device_parity.py tests/test_band_getrf.py tests/test_device_solve.py -x -q 2>&1 | tail -2
for c in C2 C3 C5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1; done
LBK_NO_MERGE=1 timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
