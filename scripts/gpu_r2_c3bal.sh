timeout 2400 python scripts/balance_bench.py C3 --sizes 1000,2000,5000 --repeats 3 --out gpurun_out/r2_balance_c3.jsonl 2>&1 | grep "^#"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c2_solve_launches.csv python scripts/solve_profile.py C2 > /dev/null 2>&1; echo ncu=$?
