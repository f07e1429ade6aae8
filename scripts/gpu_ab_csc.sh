# A/B: CSC SSSSM with a 4-deep L-entry prefetch ring (main) vs the 1-deep prefetch (pf1), every block CSC
for rep in 1 2; do for v in main pf1; do
  lib=paper_2512_04389_b200/_lib/liblbk_$v.so; [ "$v" = main ] && lib=paper_2512_04389_b200/_lib/liblbk.so
  echo "$v:"; LBK_DEV_LIB=$lib timeout 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu --dense-threshold -1 --e2e-steps 1 2>/dev/null | python scripts/summarize.py 2>/dev/null | head -1
done; done
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x -k "csc" 2>&1 | tail -2
