timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "sddmm or gat" 2>&1 | tail -3
timeout 900 python tools/l2_sweep.py reddit --sddmm 2>&1 | grep sddmm
