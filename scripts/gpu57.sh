for d in 0 74 148 296; do echo "defer_ctas=$d"; LBK_DEFER_CTAS=$d timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1; done
LBK_DEFER_CTAS=148 LBK_EXEC_PER_SM=1 timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
