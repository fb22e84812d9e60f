M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,launch__grid_size,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"
for MB in 48 96; do echo "== segmented persistent $MB MB"
FG_L2_TILE_MB=$MB FG_SDDMM_SEGMENT=1 timeout 300 ncu $M --clock-control none -k regex:sddmm_kernel -s 1 -c 1 python tools/prof_one.py sddmm512 2>&1 | grep -E "dram__|lts__|smsp__|sm__|gpu__time|grid|l1tex"
done
