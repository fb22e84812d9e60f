timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/quickbench.py reddit 2>&1 | tail -12
