"""Brief per-kernel ncu summary: duration, instructions, issue, occupancy, DRAM, top stalls."""
import csv, subprocess, sys, io
path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__registers_per_thread',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:40])
    print('   ' + ' | '.join(f"{w.split('__')[1][:28]}={r[hdr.index(w)]}" for w in want if w in hdr))
    st = sorted([(float(r[i]), h) for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_')
                 and h.endswith('per_issue_active.ratio') and r[i] not in ('', 'n/a')], reverse=True)[:6]
    print('   stalls', [(h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''),
                        round(v, 2)) for v, h in st])
