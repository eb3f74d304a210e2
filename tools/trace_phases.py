"""Per-panel phase durations from an FMAP_TRACE_FILE dump (8 warps x 1024 int64).

End-of-work stamps only (a clock64() right after __syncthreads() records the
barrier's issue time, not its release):  slot 0 staging done, 1 first diag done,
8+8p+0 TRSM(p) done, +2 panel warp's diag(p+1) done, +4 bulk SYRK(p) done,
1000 factorization done, 1001 back-substitution done (panel warp)."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 1024)
NW = int(sys.argv[2]) if len(sys.argv) > 2 else (16 if t[8:].any() else 8)
t = t[:NW]
PW = NW - 1
t0 = t[:, 0].min()
print("staging:", t[:, 0].max() - t0, " first diag:", t[PW, 1] - t[:, 0].max())
prev = t[:, 1].max()
print("panel    trsm   [next-syrk end]  diag(PW)   bulk_end   panel_total")
p = 0
while True:
    b = 8 + 8 * p
    if t[:, b].max() == 0:
        break
    eA = t[:, b].max()
    row = [eA - prev]
    if t[:, b + 4].max():
        row += [t[:PW, b + 1].max() - eA if t[:, b + 1].any() else 0, t[PW, b + 2] - eA, t[:, b + 4].max() - eA]
        nxt = t[:, b + 4].max()
    else:
        row += [0, 0, 0]
        nxt = eA
    row.append(nxt - prev)
    print(f"{p:5d}", "  ".join(f"{x:9d}" for x in row))
    prev = nxt
    p += 1
print("backsub:", t[PW, 1001] - t[:, 1000].max(), " total:", t[PW, 1001] - t0)
if t[:, 1002].any():
    print("  invert diag blocks:", t[:, 1002].max() - t[:, 1000].max())
    prevb = t[:, 1002].max()
    for jbi in range(13, -1, -1):
        if 1010 + jbi < t.shape[1] and t[:, 1010 + jbi].any():
            e = t[:, 1010 + jbi].max()
            print(f"  block {jbi:2d}: {e - prevb}")
            prevb = e
