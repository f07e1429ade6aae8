python scripts/micro_getrf.py 2048 2048 3 --trace 2>&1 | head -7
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
timeout 900 python bench.py --config C2 --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py
