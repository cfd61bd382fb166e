"""Summarise an `ncu --page raw --csv` dump: key metrics and top stall reasons per kernel."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]; data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
want = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
stalls = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('_not_issued')]
for d in data:
    print(d[idx['Kernel Name']][:60])
    for w in want:
        if w in idx:
            print(f'   {w:62s} {d[idx[w]]}')
    s = sorted(((float(d[idx[h]] or 0), h[len('smsp__pcsamp_warps_issue_stalled_'):]) for h in stalls), reverse=True)[:9]
    print('   stalls:', ', '.join(f'{n}={int(v)}' for v, n in s))
