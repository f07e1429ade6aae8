# GPU correctness pass (run under gpurun): the GPU test suite, smoke(), tile micro benchmarks.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
./tools/tile_micro
