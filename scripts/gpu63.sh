python scripts/solve_time.py C2 2>&1 | tail -1
LBK_SOLVE_SKIP_UPD=1 python scripts/solve_time.py C2 2>&1 | tail -1
LBK_SOLVE_SKIP_DIAG=1 python scripts/solve_time.py C2 2>&1 | tail -1
