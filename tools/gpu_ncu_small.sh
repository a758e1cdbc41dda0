# ncu full captures of the small-config kernels (C3 tensor passes, C2 inverse FFT + s-step)
set -x
ncu --set full --import-source on --clock-control none -k regex:"k_uni_(fwd|adj)" -s 8 -c 4 -o gpurun_out/small_c3 python bench.py --workload c3 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_small_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_n1_ifft_crop|k_cg_qstep|k_n1_embed" -s 6 -c 3 -o gpurun_out/small_c2 python bench.py --workload c2 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_small_c2.log 2>&1
ls gpurun_out | grep small
