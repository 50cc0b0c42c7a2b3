"""Hottest CUDA source lines (warp-stall samples) of an ncu report (-lineinfo build)."""
import csv, io, subprocess, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
L, tot, fname = [], 0, ''
for r in rows:
    if r and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if len(r) > 4 and r[0] not in ('', 'Line No') and r[4].isdigit():
        v = int(r[4])
        tot += v
        L.append((v, f"{fname}:{r[0]}", r[1].strip()[:100]))
L.sort(reverse=True)
for v, ln, s in L[:top]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {ln:24s} {s}")
