"""Per-panel critical-path breakdown of chol_tc_kernel from an FMAP_TRACE_FILE dump
(one CTA's second system; clock64 stamps).  Columns (cycles):
  arr->wake   last main warp's opsready arrival -> MMA warp passes its wait
  wake->LA    lookahead MMAs issued + committed
  LA->ld      lookahead landed + TMEM load done (tid 0)
  ld->dstart  tid0 load -> diagonal warp starts factoring
  diag        16x16 diagonal factor + publish
  dend->bar   diagonal factor done -> tid0 past the barrier
  trsm        tid0 TRSM
  stores      tid0 L scratch + operand stores
  st->arr     tid0 stores done -> last warp's arrival
  period      panel p+1 start -> panel p+2 start"""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64)
hdr = "  p  arr->wake wake->LA  LA->ld ld->dstart  diag dend->bar  trsm stores st->arr  period"
print(hdr)
tot = np.zeros(10)
n = 0
for p in range(1, 11):
    arr = t[700 + 8 * (p - 1): 708 + 8 * (p - 1)]
    arr = arr[arr > 0]
    if not len(arr) or not t[800 + p - 1] or not t[2 + 4 * p] or not t[2 + 4 * (p + 1)]:
        continue
    last = arr.max()
    wake, la = t[800 + p - 1], t[820 + p - 1]
    ld = t[2 + 4 * p]
    ds, de = t[900 + 4 * p + 1], t[900 + 4 * p + 2]
    bar, tr, st = t[1100 + p], t[1120 + p], t[4 + 4 * p]
    arr2 = t[700 + 8 * p: 708 + 8 * p]
    arr2 = arr2[arr2 > 0]
    last2 = arr2.max() if len(arr2) else 0
    row = [wake - last, la - wake, ld - la, ds - ld, de - ds, bar - de, tr - bar, st - tr, last2 - st,
           t[2 + 4 * (p + 1)] - ld]
    tot += row
    n += 1
    print(f"{p:3d}" + "".join(f"{int(v):10d}" for v in row))
if n:
    print("avg" + "".join(f"{int(v):10d}" for v in tot / n))

print("\nper warp, relative to the diagonal factor's end: barrier-release / TRSM done / REST-wait done / arrival")
for p in range(1, 11):
    de = t[900 + 4 * p + 2]
    if not de:
        continue
    cols = []
    for w in range(7):
        vals = [t[1400 + 8 * p + w], t[1200 + 8 * p + w], t[1300 + 8 * p + w], t[700 + 8 * p + w]]
        cols.append("/".join(str(int(v - de)) if v else "-" for v in vals))
    print(f"{p:2d} " + "  ".join(cols))
