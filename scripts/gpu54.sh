timeout 1500 python scripts/balance_bench.py C3 --sizes 2000 --repeats 2 --taus 0.02,0.05 2>&1 | cut -c1-330
