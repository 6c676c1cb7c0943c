"""Extract the key metrics of an ncu --set full report into JSON (per launch)."""
import csv, io, json, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'lts__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'launch__shared_mem_per_block', 'launch__grid_size', 'launch__block_size',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__inst_executed.sum']
STALL = 'smsp__average_warps_issue_stalled_'
rep = sys.argv[1]
txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = {'kernel': r[hdr.index('Kernel Name')][:80]}
    for i, h in enumerate(hdr):
        if h in KEYS or (h.startswith(STALL) and h.endswith('_per_issue_active.ratio')):
            try:
                v = float(r[i].replace(',', ''))
            except ValueError:
                continue
            if h.startswith(STALL) and v < 0.05:
                continue
            d[h.replace(STALL, 'stall_').replace('_per_issue_active.ratio', '')] = [v, units[i]]
    out.append(d)
print(json.dumps(out, indent=1))
