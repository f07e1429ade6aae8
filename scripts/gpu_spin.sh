timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
for v in 0 8 128; do echo spin=$v; LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_spin$v.so timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1; done
