timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/quickbench.py reddit 2>&1 | tail -10
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tcgen05 -s 3 -c 1 -o gpurun_out/prof_mlp_r01d $B > /dev/null 2>&1; echo mlp $?
