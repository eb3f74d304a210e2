# persistent back-substitution grid: CTAs per SM sweep (variant b) against a
for r in 1 2; do
  echo -n "a: "; FMAP_LIB_VARIANT=a python tools/prof_solver.py --reps 6 | tail -1
  for c in 1 2 3 4 6 8; do echo -n "b cps=$c: "; FMAP_BS_CTAS=$c FMAP_LIB_VARIANT=b python tools/prof_solver.py --reps 6 | tail -1; done
done
