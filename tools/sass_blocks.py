"""Summarise an ncu --import-source report per SASS basic block (instructions
executed, samples).  Usage: python tools/sass_blocks.py rep.ncu-rep [lo hi]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
print(r[0][0][:200] if r[0] else "")
h = r[1]
rows = r[2:]
I, S, A, SRC, T = (h.index(k) for k in ("Instructions Executed", "# Samples", "Address", "Source",
                                         "Avg. Threads Executed"))
base = int(rows[0][A], 16)
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
    for x in rows:
        off = int(x[A], 16) - base
        if lo <= off <= hi:
            print(f"{off:05x} {int(x[I]) / 1e6:6.2f} {float(x[T]):4.1f} {int(x[S]):5d} {x[SRC].strip()[:72]}")
    sys.exit(0)
tot = sum(int(x[I]) for x in rows)
ts = sum(int(x[S]) for x in rows)
print(f"total warp-inst {tot / 1e6:.1f}M, samples {ts}")
seg, cur = [], None
for x in rows:
    off, i, s = int(x[A], 16) - base, int(x[I]), int(x[S])
    if cur is None or i != cur[3]:
        if cur:
            seg.append(cur)
        cur = [off, off, 0, i, 0, 0, float(x[T])]
    cur[1] = off
    cur[2] += i
    cur[4] += s
    cur[5] += 1
seg.append(cur)
for a, b, ii, per, s, n, t in sorted(seg, key=lambda z: -z[2])[:40]:
    print(f"{a:05x}-{b:05x} n={n:3d} exec={per / 1e6:6.2f}M thr={t:4.1f} inst={ii / 1e6:7.1f}M "
          f"({100 * ii / tot:4.1f}%) samples={s} ({100 * s / ts:4.1f}%)")
