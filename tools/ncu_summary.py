"""Summarise an .ncu-rep (raw page) into the metrics we track."""
import csv, subprocess, sys, json
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__block_size',
        'lts__t_sectors.sum', 'l1tex__t_sector_hit_rate.pct']
def summarise(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {'kernel': vals[hdr.index('Kernel Name')][:110]}
        for w in WANT:
            if w in hdr:
                d[w] = vals[hdr.index(w)] + ' ' + units[hdr.index(w)]
        stalls = {h: vals[i] for i, h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(',', '') or 0))[:5]
        d['top_stalls'] = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): v for k, v in top}
        res.append(d)
    return res
if __name__ == '__main__':
    for p in sys.argv[1:]:
        for d in summarise(p):
            print(json.dumps(d, indent=1))
