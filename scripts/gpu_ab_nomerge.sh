for rep in 1 2; do
python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py | head -1
LBK_NO_MERGE=1 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py | head -1
done
