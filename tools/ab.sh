#!/bin/bash
# A/B timing helper: build the working tree as variant "b" (libfmap_cuda_b.so) next to
# the committed build "a" (git stash of the working tree), then on the GPU:
#   for v in a b a b: FMAP_LIB_VARIANT=$v python tools/prof_solver.py --reps 5
set -e
cd "$(dirname "$0")/.."
python -m paper_2604_10377_b200.build > /dev/null
cp paper_2604_10377_b200/libfmap_cuda.so paper_2604_10377_b200/libfmap_cuda_b.so
git stash -q
python -m paper_2604_10377_b200.build > /dev/null
cp paper_2604_10377_b200/libfmap_cuda.so paper_2604_10377_b200/libfmap_cuda_a.so
git stash pop -q
python -m paper_2604_10377_b200.build > /dev/null
echo "built a (HEAD) and b (working tree)"
