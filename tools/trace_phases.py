"""Print per-panel phase durations from an FMAP_TRACE_FILE dump (8 warps x 1024 int64)."""
import sys
import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(8, 1024)
t0 = t[0, 0]
print("setup (load+diag0): ", t[0, 1] - t0)
print("panel  B_max  B_w0  barB   C_max  barC   D_w0  D_others_max  barD  (cycles)")
p = 0
while True:
    b = 8 + 8 * p
    if t[0, b] == 0:
        break
    start = t[0, b - 3] if p > 0 else t[0, 1]
    row = [t[:, b].max() - start, t[0, b] - start, t[0, b + 1] - t[:, b].max()]
    if t[0, b + 2]:
        row += [t[:, b + 2].max() - t[0, b + 1], t[0, b + 3] - t[:, b + 2].max(),
                t[0, b + 4] - t[0, b + 3], t[1:, b + 4].max() - t[0, b + 3], t[0, b + 5] - t[:, b + 4].max()]
    print(p, *row)
    p += 1
print("backsub:", t[0, 1001] - t[0, 1000], " total:", t[0, 1001] - t0)
