"""Regenerate tests/golden/ (run in the build container, where /root/reference exists).

* memory_f32_k4_12.csv, bench_columns.txt: copied verbatim from the reference's
  own golden directory (proj/tests/golden/), the fixtures its
  test_bench.cpp:194-249 compares byte-for-byte.
* solutions.npz: float64 oracle solutions of reference-generator instances
  (bench.hpp:52-93 + masks.hpp) — fixed vectors the GPU parity tests and the
  oracle test replay without /root/reference.
* generator.npz: the reference generator's output for (k=5, d=10, seed=123),
  pinning the std::mt19937_64 / seed_seq / normal_distribution stream.

    python tests/golden/make_golden.py
"""
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import oracle  # noqa: E402

REF_GOLDEN = Path("/root/reference/proj/tests/golden")

CASES = [  # name, k, d, seed, mask kind (0 comm / 1 resolvent), lambda
    ("comm_k8", 8, 16, 11, 0, 100.0),
    ("comm_k16", 16, 32, 77, 0, 1.0),
    ("res_k12", 12, 24, 5, 1, 100.0),
    ("res_k20_thin", 20, 12, 9, 1, 100.0),
    ("comm_k24_lam0", 24, 48, 78, 0, 0.0),
]


def main():
    for name in ("memory_f32_k4_12.csv", "bench_columns.txt"):
        src = REF_GOLDEN / name
        if src.exists():
            shutil.copyfile(src, HERE / name)
    out = {}
    for name, k, d, seed, kind, lam in CASES:
        G, R, M, _, _ = oracle.random_problem(k, d, seed, kind=kind)
        C = oracle.solve(G, R, M, lam).maps
        for key, val in (("G", G), ("R", R), ("M", M), ("lam", np.float64(lam)), ("C", C)):
            out[f"{name}__{key}"] = val
    np.savez_compressed(HERE / "solutions.npz", **out)
    a, b, e1, e2 = oracle.generate_instance(5, 10, 123)
    np.savez_compressed(HERE / "generator.npz", a=a, b=b, ev1=e1, ev2=e2)
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
