mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tcgen05 -s 3 -c 1 -o gpurun_out/prof_mlp_r01c $B > /dev/null 2>&1; echo mlp $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm -s 6 -c 2 -o gpurun_out/prof_sddmm_r01c $B > /dev/null 2>&1; echo sddmm $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_gather -s 9 -c 3 -o gpurun_out/prof_spmm_r01c $B > /dev/null 2>&1; echo spmm $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmax -s 3 -c 1 -o gpurun_out/prof_softmax_r01c $B > /dev/null 2>&1; echo softmax $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches $?
