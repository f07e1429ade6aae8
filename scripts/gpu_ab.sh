# A/B timing of liblbk variants (run under gpurun): scripts/gpu_ab.sh CONFIG variant1 variant2 ...
# ("main" = the in-tree liblbk.so); each variant's C2-style bench summary, twice, interleaved
cfg=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    lib=paper_2512_04389_b200/_lib/liblbk_$v.so; [ "$v" = main ] && lib=paper_2512_04389_b200/_lib/liblbk.so
    echo "$v:"; LBK_DEV_LIB=$lib timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
  done
done
