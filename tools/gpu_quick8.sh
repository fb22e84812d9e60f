timeout 600 python tools/l2_sweep.py reddit hot 2>&1 | tail -12
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
