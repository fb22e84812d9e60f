set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python tools/quickbench.py reddit 2>&1 | tail -12
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; tail -3 gpurun_out/bench_r01a.err
cat gpurun_out/bench_r01a.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 21 -c 7 --csv --log-file gpurun_out/launches_r01a.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_gather -s 9 -c 1 -o gpurun_out/prof_spmm_r01a python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm -s 6 -c 1 -o gpurun_out/prof_sddmm_r01a python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full2.log 2>&1; tail -3 gpurun_out/ncu_full2.log
ls -la gpurun_out
