timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1500 python scripts/balance_bench.py C3 --sizes 2000,5000 --repeats 2 --out gpurun_out/r1_balance_c3.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 1500 python scripts/balance_bench.py C5 --repeats 3 --taus 0.05,0.25,0.5 --out gpurun_out/r1_balance_c5.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
