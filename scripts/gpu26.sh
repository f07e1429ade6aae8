timeout 900 python -m pytest tests/test_dist_device.py -x -q 2>&1 | tail -30
