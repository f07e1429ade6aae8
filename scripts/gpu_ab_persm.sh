# A/B: executor CTAs per SM (LBK_EXEC_PER_SM) with the round-2 final code
for rep in 1 2; do for v in 2 1; do echo "exec_per_sm=$v"; LBK_EXEC_PER_SM=$v python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py | head -1; done; done
