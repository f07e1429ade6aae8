# LBK_PANEL_AGG sweep (bitwise-identical factors for every value)
for v in 4 3 6 2; do echo "agg=$v"; for c in C2 C3; do LBK_PANEL_AGG=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1; done; done
