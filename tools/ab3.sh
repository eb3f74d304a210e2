#!/bin/bash
# GPU side: three in-tree builds a / b / c: k = 200 device step at 64 pairs, k sweep points
for r in 1 2; do for v in a b c; do
  echo -n "$v "; FMAP_LIB_VARIANT=$v python tools/step_probe.py 64
  FMAP_LIB_VARIANT=$v python tools/sweep_k.py --b ${B:-64} --ks ${KS:-260,300} | tail -n +2 | sed "s/^/$v /"
done; done
