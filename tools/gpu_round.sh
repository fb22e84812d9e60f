# Round measurement set on one B200 (gpurun_out/ must stay under 64 MiB per
# call, so the ncu --set full captures are split over calls):
#   PART=1      tests, smoke, bench (default; reference arm), launch list, TMA probe
#   PART=spmm   ncu --set full of the gSpMM gather kernels of one step
#   PART=sddmm  ncu --set full of the gSDDMM kernels of one step
#   PART=2      ncu --set full of softmax, MLP (tcgen05) and the fused GAT
#   PART=ctl    ncu --set full of the uniform-sources control (copy_u-sum, u_dot_v F=512)
#   PART=direct the same with the L2 column tiles / source segments off (DRAM-bound)
mkdir -p gpurun_out
TAG=${TAG:-r02}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
NCU="ncu --set full --clock-control none --import-source on"
python -c "from paper_2008_11359_b200.build import source_hash; print('build', source_hash())"
case "${PART:-1}" in
1)
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>/dev/null; cat gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > /dev/null 2>&1; echo launches $?
timeout 300 python tools/tma_probe.py > gpurun_out/tma_probe_$TAG.txt 2>&1; tail -4 gpurun_out/tma_probe_$TAG.txt
;;
spmm)
timeout 900 $NCU -k regex:spmm_gather -s 9 -c 3 -o gpurun_out/prof_spmm_$TAG $B > /dev/null 2>&1; echo spmm $?
;;
sddmm)
timeout 900 $NCU -k regex:"sddmm_(pf_)?kernel" -s 6 -c 2 -o gpurun_out/prof_sddmm_$TAG $B > /dev/null 2>&1; echo sddmm $?
;;
2)
timeout 600 $NCU -k regex:softmax -s 3 -c 1 -o gpurun_out/prof_softmax_$TAG $B > /dev/null 2>&1; echo softmax $?
timeout 600 $NCU -k regex:mlp_tcgen05 -s 3 -c 1 -o gpurun_out/prof_mlp_$TAG $B > /dev/null 2>&1; echo mlp $?
timeout 600 $NCU -k regex:gat_fused -s 0 -c 1 -o gpurun_out/prof_gat_$TAG python tools/prof_one.py gat > /dev/null 2>&1; echo gat $?
;;
ctl)
timeout 900 $NCU -k regex:spmm_gather -s 9 -c 1 -o gpurun_out/prof_uspmm_$TAG $B --uniform-sources > /dev/null 2>&1; echo uspmm $?
timeout 900 $NCU -k regex:"sddmm_(pf_)?kernel" -s 6 -c 1 -o gpurun_out/prof_usddmm_$TAG $B --uniform-sources > /dev/null 2>&1; echo usddmm $?
;;
direct)
export FG_L2_TILE_MB=0 FG_SDDMM_SEG_MB=0
timeout 900 $NCU -k regex:spmm_gather -s 9 -c 1 -o gpurun_out/prof_dspmm_$TAG $B --uniform-sources > /dev/null 2>&1; echo dspmm $?
timeout 900 $NCU -k regex:"sddmm_(pf_)?kernel" -s 6 -c 1 -o gpurun_out/prof_dsddmm_$TAG $B --uniform-sources > /dev/null 2>&1; echo dsddmm $?
;;
esac
# captures travel back compressed (gpurun_out/ is capped at 64 MiB per call);
# locally: gunzip gpurun_out/*.ncu-rep.gz before tools/make_profiles.py
for f in gpurun_out/*.ncu-rep; do [ -f "$f" ] && gzip -f -6 "$f"; done
ls -la gpurun_out | tail -12
