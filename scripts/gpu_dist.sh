timeout 1500 python scripts/dist_check.py C2 4 2>&1 | grep -v Warning | tail -3
timeout 1500 python scripts/dist_check.py C3 2 2>&1 | grep -v Warning | tail -3
