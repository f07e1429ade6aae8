for v in t16_0 t16_1 t8_1; do echo $v; ./tools/tile_micro_$v 2>&1 | grep -E "solve_blk|tile_lu"; done
for v in main t16n t8; do lib=paper_2512_04389_b200/_lib/liblbk_$v.so; [ $v = main ] && lib=paper_2512_04389_b200/_lib/liblbk.so; echo $v; LBK_DEV_LIB=$lib timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180; done
bash scripts/gpu_ab.sh C2 main t16n t8
