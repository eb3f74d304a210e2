import sys; sys.path.insert(0, '.')
import numpy as np, oracle
import paper_2604_10377_b200 as fm
for k in (40, 48, 50, 52, 64):
    G, R, M, _, _ = oracle.random_problem(k, 2*k, 77, kind=0)
    G, R, M = (x.astype(np.float32)[None] for x in (G, R, M))
    C = fm.solve_host(G, R, M, 1.0).maps[0]
    ref = oracle.solve(G, R, M, 1.0, dtype=np.float64).maps[0]
    err = np.abs(C - ref)
    bad_cols = np.where(err.max(0) > 1e-4 * np.abs(ref).max())[0]
    print(k, "maxerr", err.max() / np.abs(ref).max(), "bad cols", bad_cols[:20], len(bad_cols))
