timeout 900 python -m pytest tests/test_device_solve.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
