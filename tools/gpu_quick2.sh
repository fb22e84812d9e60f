timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/quickbench.py reddit 2>&1 | tail -11
for t in 0 32 128; do echo "--- FG_L2_TILE_MB=$t"; FG_L2_TILE_MB=$t timeout 300 python tools/quickbench.py reddit 2>&1 | grep -E "copy_u|umule"; done
