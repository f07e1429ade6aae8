# A/B: aggregated panel tile updates (LBK_PANEL_AGG, default 4) vs one task per step (1) and 8
for rep in 1 2; do for v in 4 1 8; do
  echo "agg=$v"; for c in C2 C3; do LBK_PANEL_AGG=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1; done
done; done
for v in 4 1; do LBK_PANEL_AGG=$v python bench.py --config C5 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1; done
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x -k "aggregated or named or large_blocks or subtree" 2>&1 | tail -2
