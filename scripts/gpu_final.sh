# Final round pass (run under gpurun): GPU suite + smoke, all bench lines + ncu (profile_round.sh),
# irregular-vs-regular balance on C5/C3, band statistics.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
bash scripts/profile_round.sh
timeout 900 python scripts/balance_bench.py C5 --out gpurun_out/r1_balance_c5.jsonl 2>&1 | grep "^#"
timeout 1200 python scripts/balance_bench.py C3 --sizes 500,1000,2000,5000 --out gpurun_out/r1_balance_c3.jsonl 2>&1 | grep "^#"
timeout 300 python scripts/band_stats.py C5 > gpurun_out/r1_band_stats_c5.txt 2>&1
timeout 300 python scripts/band_stats.py C3 > gpurun_out/r1_band_stats_c3.txt 2>&1
