#!/bin/bash
# A/B timing of library variants: tools/ab.sh lib1.so lib2.so ...  (C5 bench, 256 problems)
for lib in "$@"; do
  GS_B200_LIB=$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernel_ms_per_pair']
print('$lib', d['value'], 'spread', k.get('k2f_spread'), 'interp', k.get('k2f_interp'))"
done
