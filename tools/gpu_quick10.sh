timeout 300 python tools/quickbench.py reddit 2>&1 | tail -12
timeout 300 python tools/step_ops.py 2>&1 | tail -10
