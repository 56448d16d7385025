"""Summarise an ncu report (details page) into one block per kernel."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Warp Cycles Per Issued Instruction', 'Dynamic Shared Memory Per Block', 'Block Limit Registers',
        'Block Limit Shared Mem', 'Mem Busy', 'Max Bandwidth', 'Mem Pipes Busy', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'DRAM Bandwidth']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
       'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'smsp__inst_executed.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
       'smsp__pcsamp_warps_issue_stalled_long_scoreboard', 'smsp__pcsamp_warps_issue_stalled_short_scoreboard',
       'smsp__pcsamp_warps_issue_stalled_mio_throttle', 'smsp__pcsamp_warps_issue_stalled_barrier',
       'smsp__pcsamp_warps_issue_stalled_lg_throttle', 'smsp__pcsamp_warps_issue_stalled_math_pipe_throttle',
       'smsp__pcsamp_warps_issue_stalled_wait', 'smsp__pcsamp_warps_issue_stalled_selected',
       'smsp__pcsamp_warps_issue_stalled_not_selected', 'smsp__pcsamp_warps_issue_stalled_drain']


def run(rep):
    d = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(d)))
    I = {h: i for i, h in enumerate(rows[0])}
    out = {}
    for r in rows[1:]:
        key = (r[I['ID']], r[I['Kernel Name']][:60])
        if r[I['Metric Name']] in WANT:
            out.setdefault(key, []).append(f"{r[I['Metric Name']]}={r[I['Metric Value']]} {r[I['Metric Unit']]}")
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    H = rr[0]
    for r in rr[2:]:
        key = (r[H.index('ID')], r[H.index('Kernel Name')][:60])
        for m in RAW:
            if m in H:
                out.setdefault(key, []).append(f"{m}={r[H.index(m)]}")
    for k, v in out.items():
        print('==', *k)
        for x in v:
            print('   ', x)


if __name__ == '__main__':
    run(sys.argv[1])
