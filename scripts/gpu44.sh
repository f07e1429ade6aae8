timeout 900 python -m pytest tests/test_band_getrf.py tests/test_device_parity.py -x -q 2>&1 | tail -3
timeout 1500 python scripts/balance_bench.py C5 --sizes 500,1000,2000,5000 --repeats 3 --out gpurun_out/balance_c5_v44.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 2400 python scripts/balance_bench.py C3 --sizes 2000,5000 --repeats 2 --out gpurun_out/balance_c3_v44.jsonl 2>&1 | grep "^#" | cut -c1-300
