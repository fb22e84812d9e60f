mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/mlp_exp.py reddit 0,6 2>&1 | tail -2
timeout 300 python tools/mlp_exp.py rand100k 0 2>&1 | tail -1
