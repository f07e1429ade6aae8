# A/B: absorbed SSSSM tiles run as chains of K-pieces inside the next executor launch
# (liblbk_absorb.so = -DLBK_ABSORB_TILES=1, LBK_ABSORB=1, piece size LBK_ABSORB_PIECE) vs main
lib=paper_2512_04389_b200/_lib/liblbk_absorb.so
for rep in 1 2; do
  echo main; python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
  for pc in 16 32 8; do echo "absorb piece=$pc"; LBK_DEV_LIB=$lib LBK_ABSORB=1 LBK_ABSORB_PIECE=$pc python bench.py --config C2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1; done
done
echo C5; python bench.py --config C5 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
LBK_DEV_LIB=$lib LBK_ABSORB=1 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
LBK_DEV_LIB=$lib LBK_ABSORB=1 timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x -k "named or large_blocks or subtree" 2>&1 | tail -2
