#!/bin/bash
# A/B timing of environment variants: tools/ab_env.sh "VAR=a" "VAR=b" ...  (C5 bench, 256 problems)
for envs in "$@"; do
  env $envs python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernel_ms_per_pair']
print('$envs', d['value'], 'spread', k.get('k2f_spread'), 'interp', k.get('k2f_interp'))"
done
