#!/bin/bash
# PCG variants on the headline config (device ms per MM iteration, PCG iterations)
for v in "NRR_PCG=cluster" "NRR_PCG=grid NRR_COARSE=1 NRR_AGG_CTAS=8"; do
  echo "== $v"; env $v timeout 120 python tools/profile_step.py --iters 5 | tail -2
done
