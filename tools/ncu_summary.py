"""Key ncu --set full counters of every kernel in a report (raw page)."""
import csv, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__cluster_dim_x',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg',
        'launch__shared_mem_per_block_dynamic']
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print(f"== {v[h.index('Kernel Name')][:90]}  [{rep.split('/')[-1]}]")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:60s} {v[i]:>22s} {units[i]}")
