# A/B: aggregated trailing GEMM + panel updates (LBK_PANEL_AGG=4, default) vs one task per step (1)
for rep in 1 2; do for v in 4 1; do
  echo "agg=$v"; for c in C2 C3 C5; do LBK_PANEL_AGG=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1; done
done; done
timeout 600 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
LBK_PANEL_AGG=1 timeout 600 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x -k "aggregated or named or large_blocks or subtree or small" 2>&1 | tail -2
