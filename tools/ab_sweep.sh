#!/bin/bash
# GPU side: k sweep of variants a / b (tools/ab.sh builds them)
for v in a b a b; do
  echo "== $v"; FMAP_LIB_VARIANT=$v python tools/sweep_k.py --b "${B:-64}" --ks "${KS:-48,64,80,100,112,128,144,200}" | tail -n +2
done
