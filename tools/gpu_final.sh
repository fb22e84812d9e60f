# Round measurement set (gpurun_out/ must stay under 64 MiB per call, so the
# ncu --set full captures are split over calls):
#   PART=1     tests, smoke, bench (default + uniform-sources control + reference arm), launch list, sweep
#   PART=spmm  ncu --set full of the gSpMM gather kernels of one step
#   PART=sddmm ncu --set full of the gSDDMM kernels of one step
#   PART=2     ncu --set full of softmax, MLP (tcgen05) and the fused GAT
mkdir -p gpurun_out
TAG=${TAG:-r01}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
case "${PART:-1}" in
1)
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 900 python bench.py --uniform-sources --no-cpu-baseline --no-e2e > gpurun_out/bench_uniform_$TAG.json 2>/dev/null; cat gpurun_out/bench_uniform_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>/dev/null; cat gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches $?
timeout 900 python tools/sweep.py gpurun_out/sweep_$TAG > /dev/null 2>&1; echo sweep $?
;;
spmm)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_gather -s 9 -c 3 -o gpurun_out/prof_spmm_$TAG $B > /dev/null 2>&1; echo spmm $?
;;
sddmm)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm_kernel -s 6 -c 2 -o gpurun_out/prof_sddmm_$TAG $B > /dev/null 2>&1; echo sddmm $?
;;
2)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmax -s 3 -c 1 -o gpurun_out/prof_softmax_$TAG $B > /dev/null 2>&1; echo softmax $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tcgen05 -s 3 -c 1 -o gpurun_out/prof_mlp_$TAG $B > /dev/null 2>&1; echo mlp $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gat_fused -s 1 -c 1 -o gpurun_out/prof_gat_$TAG $B > /dev/null 2>&1; echo gat $?
;;
esac
ls -la gpurun_out | tail -12
