python scripts/micro_getrf.py 512 512 3 --trace
python scripts/micro_getrf.py 2048 2048 3 --trace
