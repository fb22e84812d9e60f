FG_MLP_DBG=1 timeout 300 ncu --set full --import-source on -k regex:mlp_tcgen05 -s 2 -c 1 -o gpurun_out/prof_mlp_skel python tools/prof_one.py mlp > /dev/null 2>&1; echo $?
timeout 300 ncu --set full --import-source on -k regex:mlp_tcgen05 -s 2 -c 1 -o gpurun_out/prof_mlp_full python tools/prof_one.py mlp > /dev/null 2>&1; echo $?
timeout 300 ncu --set full --import-source on -k regex:gat_fused -s 2 -c 1 -o gpurun_out/prof_gat python tools/prof_one.py gat > /dev/null 2>&1; echo $?
