timeout 300 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python tools/quickbench.py reddit 2>&1 | tail -11
