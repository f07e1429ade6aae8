# After a band-sweep change (run under gpurun): GPU suite + smoke, C3/C5 bench lines with CPU baseline, band statistics.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/r1_bench_c3.json 2>/dev/null; tail -1 gpurun_out/r1_bench_c3.json | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/r1_bench_c5.json 2>/dev/null; tail -1 gpurun_out/r1_bench_c5.json | python scripts/summarize.py 2>/dev/null | head -1
timeout 300 python scripts/band_stats.py C5 > gpurun_out/r1_band_stats_c5.txt 2>&1
timeout 300 python scripts/band_stats.py C3 > gpurun_out/r1_band_stats_c3.txt 2>&1
timeout 600 python scripts/balance_bench.py C5 --sizes 200,500,5000 --out gpurun_out/r1_balance_c5.jsonl 2>&1 | grep "^#"
