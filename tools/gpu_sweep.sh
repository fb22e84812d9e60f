for mb in 24 48 96 160; do echo "--- segment budget $mb MB"; FG_SDDMM_SEGMENT=1 FG_L2_TILE_MB=$mb timeout 300 python tools/quickbench.py reddit 2>&1 | grep -E "sddmm|copy_u_sum_F512"; done
