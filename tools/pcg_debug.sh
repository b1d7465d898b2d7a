#!/bin/bash
# timing decomposition of the cluster PCG: 200 forced iterations per solve
for d in 8 9 11 15 13; do
  echo "== NRR_PCG_DEBUG=$d"; NRR_PCG_DEBUG=$d NRR_PCG_MAXIT=200 timeout 120 python tools/profile_step.py --iters 3 2>&1 | tail -1 | python3 -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().replace('np.float64','')); print('pcg ms/solve', d['pcg'], 'us/iter', 1000*d['pcg']/200)"
done
