"""Phase durations of the tensor-core solver from an FMAP_TRACE_FILE dump.
Slots (one CTA, its second system): 0 start, 1 staging done, per panel p:
2+4p tid0 panel loaded (after the lookahead wait), 3+4p diag factored (+stores),
4+4p tid0 TRSM/stores done, 5+4p MMAs issued; 300+p top-left SYRK done (row s-1);
200 panels done, 201 diag inverses done, 202 back substitution done, 203 end."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64)
t0 = t[0]
rel = lambda x: int(x - t0) if x else -1
print("staging", rel(t[1]))
prev = t[1]
p = 0
print(" p   load  diag  trsm  issue | total  (syrkTL end)")
while t[2 + 4 * p]:
    a, d, r, m = (t[2 + 4 * p + e] for e in range(4))
    tl = t[300 + p]
    bf, la = t[601 + 2 * p], t[600 + 2 * p]
    extra = f"  [barrier-f {bf - r}, LA issue {la - bf}, REST issue {m - la}]" if bf and la else ""
    print(f"{p:2d} {a - prev:6d} {d - a:5d} {r - d:5d} {m - r:5d} | {m - prev:6d}{extra}")
    prev = m
    p += 1
print("panels end", rel(t[200]), " inv", t[201] - t[200], " backsub", t[202] - t[201], " out", t[203] - t[202],
      " total", rel(t[203]))
if t[398]:
    print("pre-staging", t[398] - t0, " rhs/mask loads", t[399] - t[398])
    cb = 0
    while t[400 + 2 * cb]:
        w = t[401 + 2 * cb]
        print(f"  chunk {cb}: start {t[400 + 2 * cb] - t0}  wait {w - t[400 + 2 * cb]}  st {t[450 + cb] - w}"
              f"  sync {t[470 + cb] - t[450 + cb]}  issue {t[490 + cb] - t[470 + cb]}")
        cb += 1
