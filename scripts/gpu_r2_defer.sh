for d in 0 148 222 296; do echo "defer_ctas=$d"; for rep in 1 2; do LBK_DEFER_CTAS=$d timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1; done; done
for c in C1 C5 C3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1; done
timeout 900 python -m pytest tests/test_device_parity.py -x -q 2>&1 | tail -2
