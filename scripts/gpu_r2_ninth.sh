mkdir -p gpurun_out
for v in pb8 pb16 pb32; do echo $v; ./tools/tile_micro_$v 2>&1 | grep -E "lu64|tile_lu"; done
for v in main pb8 pb32; do lib=paper_2512_04389_b200/_lib/liblbk_$v.so; [ $v = main ] && lib=paper_2512_04389_b200/_lib/liblbk.so; echo $v; LBK_DEV_LIB=$lib timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180; done
bash scripts/gpu_ab.sh C2 main pb8
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c3_solve_launches.csv python scripts/solve_profile.py C3 > /dev/null 2>&1; echo ncu=$?
