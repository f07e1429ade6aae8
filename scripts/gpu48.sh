timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1500 python scripts/balance_bench.py C3 --sizes 2000,5000 --repeats 2 --out gpurun_out/balance_c3_v48.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 1500 python scripts/balance_bench.py C5 --sizes 500,1000,2000,5000 --repeats 3 --out gpurun_out/balance_c5_v48.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
