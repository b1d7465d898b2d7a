#!/bin/bash
for v in "NRR_COARSE=0" "NRR_COARSE=1 NRR_AGG_CTAS=8"; do
  echo "== $v"; env $v NRR_PROF=1 timeout 120 python tools/profile_step.py --iters 5 2>&1 | tail -3
done
