timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "mlp or tiny" 2>&1 | tail -2
timeout 600 python tools/mlp_exp.py reddit 0,1 2>&1 | tail -2
timeout 600 python tools/mlp_exp.py rand100k 0 2>&1 | tail -1
