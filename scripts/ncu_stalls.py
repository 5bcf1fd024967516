"""Print the top stall reasons, pipe utilisations and smem counters of an ncu report."""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); h, u, v = r[0], r[1], r[2]
xs = []
for i, n in enumerate(h):
    if 'smsp__average_warps_issue_stalled' in n and n.endswith('per_issue_active.ratio'):
        try: xs.append((float(v[i]), n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
        except ValueError: pass
print('stalls:', ', '.join(f'{n} {x:.2f}' for x, n in sorted(xs, reverse=True)[:8]))
for key in ['gpu__time_duration.sum', 'launch__registers_per_thread', 'sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed',
            'sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
            'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
            'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
            'local_load', 'smsp__inst_executed.sum']:
    for i, n in enumerate(h):
        if n == key or (key == 'local_load' and 'lsu_mem_local_op_ld.sum' in n and 'pct' not in n and 'per_second' not in n):
            print(n, v[i], u[i])
