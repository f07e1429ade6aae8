timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_case.py p3d10 > gpurun_out/r2_racecheck_p3d10.txt 2>&1; tail -25 gpurun_out/r2_racecheck_p3d10.txt | cut -c1-200
timeout 900 python -m pytest tests/test_device_parity.py tests/test_full_configs.py -x -q 2>&1 | tail -2
bash scripts/gpu_ab.sh C2 main nosplit
for v in main nosplit; do lib=paper_2512_04389_b200/_lib/liblbk_$v.so; [ $v = main ] && lib=paper_2512_04389_b200/_lib/liblbk.so; echo $v; LBK_DEV_LIB=$lib timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1; done
