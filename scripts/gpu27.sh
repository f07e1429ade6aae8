timeout 300 python scripts/debug_dist.py p3d 4 2>&1 | tail -30
