mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_parity.py -x -q -k "refined or small or named" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_full_configs.py -x -q -s 2>&1 | grep -E "compared|passed|failed|Error" | head
for c in C5 C3 C2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r2e_bench_$c.json 2>/dev/null; python scripts/summarize.py < gpurun_out/r2e_bench_$c.json 2>/dev/null | head -1; done
timeout 900 python scripts/balance_bench.py C5 bbd200000_b1_k100_s0 bbd200000_b4_k200_s0 --repeats 3 --out gpurun_out/r2e_balance.jsonl 2>&1 | grep "^#"
