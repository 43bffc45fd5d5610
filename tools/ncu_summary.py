"""Summarise ncu reports (raw page) for the kernels we care about."""
import csv, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'lts__t_sectors_srcunit_tex_op_red.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio',
        'lts__t_sectors_op_red.sum', 'lts__t_requests_srcunit_tex_op_red.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_red.sum', 'launch__grid_size', 'launch__occupancy_limit_shared_mem']

for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        print(rep, 'no data'); continue
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print('==', rep, v[h.index('Kernel Name')][:60] if 'Kernel Name' in h else '')
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f'  {w:66s} {v[i]:>16s} {u[i]}')
