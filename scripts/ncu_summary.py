"""Key metrics of an ncu --set full report (per kernel launch)."""
import csv, io, subprocess, sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput',
        'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Issue Slots Busy', 'Block Limit Shared Mem',
        'Block Limit Registers', 'Dynamic Shared Memory Per Block', 'Waves Per SM', 'No Eligible',
        'Grid Size', 'Block Size']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
       'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
       'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']


def summarize(path):
    out = []
    d = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(d)))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT and (r[ki], r[mi]) not in seen:
            seen.add((r[ki], r[mi]))
            out.append(f"  {r[mi]:32s} {r[vi]:>14s} {r[ui]}")
    name = rows[1][ki].split('(')[0] if len(rows) > 1 else '?'
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        h, u, v = rr[0], rr[1], rr[2]
        for m in RAW:
            if m in h:
                out.append(f"  {m:32s} {v[h.index(m)]:>14s} {u[h.index(m)]}")
    return name + "\n" + "\n".join(out)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(p)
        print(summarize(p))
