"""Summarise an ncu report (details page + pipe metrics): python scripts/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'Elapsed Cycles', 'SM Active Cycles', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'Registers Per Thread', 'Grid Size', 'Block Size', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Eligible Warps Per Scheduler', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Local Memory Spilling Requests']
RAW = ['sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
       'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
       'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum', 'sm__inst_executed.sum',
       'smsp__inst_executed_op_local_ld.sum', 'smsp__inst_executed_op_local_st.sum']


def run(rep, page):
    return subprocess.run(['ncu', '-i', rep, '--page', page, '--csv'], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(run(rep, 'details'))))
    h = rows[0]
    kname = None
    for r in rows[1:]:
        if kname is None:
            kname = r[h.index('Kernel Name')]
            print('kernel:', kname[:100])
        if r[h.index('Metric Name')] in WANT:
            print(f"  {r[h.index('Metric Name')]:40s} {r[h.index('Metric Value')]:>14s} {r[h.index('Metric Unit')]}")
    rows = list(csv.reader(io.StringIO(run(rep, 'raw'))))
    h, units, v = rows[0], rows[1], rows[2]
    for name in RAW:
        if name in h:
            i = h.index(name)
            print(f"  {name:62s} {v[i]:>14s} {units[i]}")
    # top stall reasons from the source page
    rows = list(csv.reader(io.StringIO(subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                                                      capture_output=True, text=True).stdout)))
    if len(rows) > 2:
        h, d = rows[1], rows[2:]
        cols = [j for j, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
        tot = {h[j]: sum(int(r[j]) for r in d if len(r) > j and r[j].isdigit()) for j in cols}
        s = sum(tot.values()) or 1
        print('  stall samples:', ', '.join(f"{k[6:]}={100 * v / s:.0f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:6]))


if __name__ == '__main__':
    main(sys.argv[1])
