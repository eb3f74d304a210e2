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
print(" p   period  ld->diag  diag->stores")
p = 0
while t[2 + 4 * p] and t[2 + 4 * (p + 1)]:
    a, d, r = t[2 + 4 * p], t[3 + 4 * p], t[4 + 4 * p]
    print(f"{p:2d} {t[2 + 4 * (p + 1)] - a:8d} {d - a:8d} {r - d:8d}")
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
print(" p  lastArr(w)  mmaWake  LAissued  RESTissued  LAseen(tid0)  ld(tid0)  [rel. to last opsready arrival]")
for p in range(12):
    arr = t[700 + 8 * p: 708 + 8 * p]
    if not arr.any():
        break
    la = arr.max()
    w = int(np.argmax(arr))
    f = lambda x: int(x - la) if x else None
    print(f"{p:2d}  w{w} {[int(x - arr.min()) for x in arr]}  wake {f(t[800+p])} LA {f(t[820+p])} REST {f(t[840+p])}"
          f"  LAseen {f(t[860+p+1])} ld {f(t[2+4*(p+1)])} ysync {f(t[880+p+1])}")
print(" p  diag warp: LAseen->ld  ld->factor-start  factor  stores  reload+  (rel. tid0 ld)")
for p in range(1, 12):
    w0, w1, w2, w3, d = t[900 + 4 * p], t[901 + 4 * p], t[902 + 4 * p], t[903 + 4 * p], t[3 + 4 * p]
    if not w1:
        continue
    print(f"{p:2d}  LAseen {int(w0 - t[2+4*p]) if w0 else None}  start {int(w1 - t[2+4*p])}  factor {w2 - w1}  stores {w3 - w2}  reload {d - w3}")
print(" p  [bypass warp, rel. barrier-c]  trsm  RESTwait  stores  blk-ld  exch+upd  yrdy  factor  store  -> next barrier-c")
for p in range(1, 12):
    b = t[1009 + 10 * p]
    x = [t[1000 + 10 * p + e] for e in range(8)]
    if not b or not x[7]:
        continue
    d = t[3 + 4 * (p + 1)]
    nb = t[1009 + 10 * (p + 1)]
    print(f"{p:2d}  start {int(x[0]-b)}  trsm {x[1]-x[0]}  REST {x[2]-x[1]}  st {x[3]-x[2]}  ld {x[4]-x[3]}  upd {x[5]-x[4]}"
          f"  yrdy {x[6]-x[5]}  fac {x[7]-x[6]}  store {d-x[7]}  | nextbar {int(nb - d) if nb else None}")
