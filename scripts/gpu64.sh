timeout 900 python -m pytest tests/test_device_solve.py -x -q 2>&1 | tail -5
python scripts/solve_time.py C2 2>&1 | tail -1
python scripts/solve_time.py C3 2>&1 | tail -1
