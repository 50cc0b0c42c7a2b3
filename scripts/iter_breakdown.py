"""Print the launches of one FGMRES iteration from an ncu launch-list CSV
(gpu__time_duration.sum, optionally dram__bytes_read.sum)."""
import csv, re, sys
U = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3,
     'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'B': 1, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui, gi, mi, ii = (h.index(x) for x in ('Kernel Name', 'Metric Value', 'Metric Unit',
                                                   'Grid Size', 'Metric Name', 'ID'))
    D, order = {}, []
    for r in rows[1:]:
        k = r[ii]
        if k not in D:
            n = re.sub(r'\(.*', '', re.sub(r'^void ', '', r[ki])).replace('<unnamed>::', '')
            D[k] = {'n': n, 'g': r[gi]}
            order.append(k)
        D[k][r[mi]] = float(r[vi].replace(',', '')) * U.get(r[ui], 1)
    return [D[k] for k in order]


if __name__ == '__main__':
    L = load(sys.argv[1])
    back = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    idx = [i for i, d in enumerate(L) if d['n'].startswith('k_pre')]
    i0, i1 = idx[-back], idx[-back + 1]
    tot = 0
    for d in L[i0:i1]:
        t = d['gpu__time_duration.sum']
        b = d.get('dram__bytes_read.sum', 0)
        print(f"{d['n']:20s} {d['g']:>16s} {t:8.2f} us  {b / 1e6:8.2f} MB  {b / t / 1e3:7.0f} GB/s")
        tot += t
    print('iteration total us', round(tot, 1))
