timeout 300 python scripts/micro_getrf.py 2048 2048 3 --trace 2>&1 | tail -14
