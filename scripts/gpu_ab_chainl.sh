# A/B: chain-2 GETRF tasks (LBK_CHAIN_L=1: the LU task also solves L(k+1,k), releasing the other successors first) vs main
timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
LBK_CHAIN_L=1 timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
for rep in 1 2; do
  echo main; python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
  echo chainL; LBK_CHAIN_L=1 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
done
echo C5; python bench.py --config C5 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
LBK_CHAIN_L=1 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
LBK_CHAIN_L=1 timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x -k "named or large_blocks or subtree or small" 2>&1 | tail -2
