# Round-2 call 2: full-size parity tests, C2 level profile, the reference run to completion on full C2.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_full_configs.py -x -q -s 2>&1 | grep -v "^$" | tail -8
timeout 600 python scripts/level_profile.py C2 --top 40 > gpurun_out/r2_c2_level_profile.txt 2>&1; tail -25 gpurun_out/r2_c2_level_profile.txt
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --levels-out gpurun_out/r2_c2_levels.npz > /dev/null 2>&1
timeout 2400 python scripts/ref_ladder.py C2 64 --out gpurun_out/r2_ref_full_c2.jsonl 2>&1 | cut -c1-600
