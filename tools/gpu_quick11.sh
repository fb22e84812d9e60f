timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for M in 0 1; do echo "== FG_SPMM_MAP=$M"; FG_SPMM_MAP=$M timeout 300 python tools/quickbench.py reddit 2>&1 | grep -v gat_ | tail -9; done
for T in 16 32 64; do echo "== map1 tile $T"; FG_L2_TILE_MB=$T timeout 300 python tools/quickbench.py reddit 2>&1 | grep "copy_u_sum_F512\|copy_u_max"; done
timeout 600 python tools/l2_sweep.py reddit 2>&1 | grep sddmm
