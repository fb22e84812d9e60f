mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/quickbench.py reddit 2>&1 | tail -11
echo "--- SIMT MLP ablation"; FG_MLP_SIMT=1 timeout 300 python tools/quickbench.py reddit 2>&1 | grep mlp
echo "--- uniform sources (DRAM-bound control)"; timeout 300 python tools/quickbench.py reddit --uniform 2>&1 | tail -11
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tcgen05 -s 3 -c 1 -o gpurun_out/prof_mlp_r01b python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mlp.log 2>&1; tail -2 gpurun_out/ncu_mlp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm -s 6 -c 2 -o gpurun_out/prof_sddmm_r01b python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sddmm.log 2>&1; tail -2 gpurun_out/ncu_sddmm.log
