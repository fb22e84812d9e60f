timeout 600 python tools/l2_sweep.py reddit hot 2>&1 | tail -12
