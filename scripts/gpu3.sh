set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -30
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --cpu-sample-s 5 2>&1 | tail -2 | cut -c1-600
timeout 600 python bench.py --config poisson3d32 --steps 3 --warmup 2 --no-cpu 2>&1 | tail -2 | cut -c1-600
for tau in 0.25 0.5 0.1; do
timeout 900 python bench.py --config C2 --steps 2 --warmup 2 --no-cpu --dense-threshold $tau --levels-out gpurun_out/c2_levels_$tau.npz 2>&1 | tail -2 | cut -c1-900
done
