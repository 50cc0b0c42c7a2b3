"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, re, sys

def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    out = []
    for r in rows[1:]:
        name = re.sub(r'^void ', '', r[ki])
        name = re.sub(r'\(.*', '', name).replace('<unnamed>::', '')
        v = float(r[vi].replace(',', ''))
        v = {'nsecond': v / 1e3, 'ns': v / 1e3, 'usecond': v, 'us': v, 'msecond': v * 1e3, 'ms': v * 1e3}[r[ui]]
        out.append((name, v))
    return out

def summary(path, top=25):
    L = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in L:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':44s} {'launches':>8s} {'total_ms':>10s} {'share':>6s} {'avg_us':>9s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"{k:44s} {c:8d} {t/1e3:10.3f} {100*t/tot:5.1f}% {t/c:9.2f}")
    lines.append(f"total {len(L)} launches, {tot/1e3:.3f} ms (serialised, cold-cache ncu times)")
    return "\n".join(lines)

if __name__ == '__main__':
    print(summary(sys.argv[1]))
