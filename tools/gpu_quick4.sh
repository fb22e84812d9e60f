timeout 300 python tools/mlp_exp.py reddit 0,3,7,11,15
