free -g | head -2; nproc
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -4
timeout 1500 python scripts/balance_bench.py C5 --sizes 500,1000,2000,5000 --repeats 3 --out gpurun_out/balance_c5.jsonl 2>&1 | grep "^#\|status" | cut -c1-400
