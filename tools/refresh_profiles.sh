set -x
python bench.py > gpurun_out/r01e_bench_c5.json 2> gpurun_out/r01e_bench_c5.err
for w in c1 c2 c3 c4; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/r01e_bench_$w.json 2> gpurun_out/r01e_bench_$w.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01e_bench_reference.json 2> gpurun_out/r01e_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01e_launches.csv python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2f_ -s 2 -c 2 -o gpurun_out/r01e_full_k2f python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"k2_fold_src|k2_cols_fft|k2_cols_ifft" -s 3 -c 3 -o gpurun_out/r01e_full_other python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_full2.log 2>&1
ls gpurun_out
