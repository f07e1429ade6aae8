# A/B of DMMA SSSSM variants with the final code: no split-K, 4 stages, GBK 32 x 2 stages
bash scripts/gpu_ab.sh C2 main nosplit s4 k32 2>&1 | grep -v "Traceback\|File \|print\|BrokenPipe"
