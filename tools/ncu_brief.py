"""Key metrics from an ncu --set full report: SOL, occupancy, stalls, instruction mix."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'smsp__inst_executed.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'lts__t_bytes.sum']

for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for vals in rows[2:]:
        d = dict(zip(h, vals))
        print('==', d.get('Kernel Name', '')[:100], 'grid', d.get('launch__grid_size'), 'block',
              d.get('launch__block_size'))
        for k in KEYS:
            if k in d:
                print(f'   {k:60s} {d[k]:>18s}')
        st = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): float(v.replace(',', '') or 0)
              for k, v in d.items()
              if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued')}
        tot = sum(st.values()) or 1
        print('   stalls:', ', '.join(f'{k} {v / tot * 100:.0f}%'
                                     for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:7]))
