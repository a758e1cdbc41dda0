#!/bin/bash
# A/B of FFT variants: tools/ab_fft.sh "ENV=a lib" ...  (C5 bench, FFT kernel times)
for spec in "$@"; do
  env $spec python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms_per_pair']
print('$spec', d['value'], {x: k[x] for x in k if 'fft' in x})"
done
