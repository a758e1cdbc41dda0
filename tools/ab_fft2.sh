#!/bin/bash
# A/B of library variants on the C5 FFT / fold passes: tools/ab_fft2.sh lib1.so lib2.so ...
for lib in "$@"; do
  GS_B200_LIB=$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernel_ms_per_pair']
print('$lib', d['value'], {n: k[n] for n in k if 'fft' in n or 'fold' in n})"
done
