# C5 selection / balance sweep (BASELINE configs[4]): run under gpurun.
#  seed 0: border {1,2,4}% x bodies {100,200,400}, irregular step {1,2,4} x max_num {1,3,7},
#          every PanguLU regular size, density tag tau {0.05,0.1,0.25,0.5,0.75,off} on the default plan;
#  seeds 1-9: border 2 %, 200 bodies, irregular (defaults) vs every regular size.
mkdir -p gpurun_out
OUT=gpurun_out/r2_c5_sweep.jsonl
: > $OUT
M=""
for b in 1 2 4; do for k in 100 200 400; do M="$M bbd200000_b${b}_k${k}_s0"; done; done
timeout 3000 python scripts/balance_bench.py $M --grid 1,2,4:1,3,7 --taus 0.05,0.1,0.25,0.5,0.75,off \
  --repeats 3 --out gpurun_out/r2_c5_sweep_seed0.jsonl 2>&1 | grep "^#"
M=""
for s in 1 2 3 4 5 6 7 8 9; do M="$M bbd200000_b2_k200_s${s}"; done
timeout 1800 python scripts/balance_bench.py $M --repeats 3 --out gpurun_out/r2_c5_sweep_seeds.jsonl 2>&1 | grep "^#"
cat gpurun_out/r2_c5_sweep_seed0.jsonl gpurun_out/r2_c5_sweep_seeds.jsonl > $OUT
