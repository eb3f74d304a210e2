#!/bin/bash
# GPU side of tools/ab.sh: alternate variants a / b, 5 solver launches each
for r in 1 2 3; do for v in a b; do
  echo -n "$v: "; FMAP_LIB_VARIANT=$v python tools/prof_solver.py --reps 6 "$@" | tail -1
done; done
