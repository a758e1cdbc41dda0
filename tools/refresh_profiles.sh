# Regenerate the judged evidence under gpurun_out/ (copy into profiles/ afterwards):
# bench lines C1-C5 + reference arm, C5 launch list, ncu full captures.
# usage (GPU box): bash tools/refresh_profiles.sh r01f
set -x
R=${1:-r01f}
python bench.py > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err
for w in c1 c2 c3 c4; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/${R}_bench_$w.json 2> gpurun_out/${R}_bench_$w.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2f_ -s 2 -c 2 -o gpurun_out/${R}_full_k2f python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"k2_fold_src|k2_cols_fft|k2_cols_ifft|k2_fold_lines" -s 3 -c 4 -o gpurun_out/${R}_full_other python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none -k regex:"k_uni_cgls_iter" -s 1 -c 1 -o gpurun_out/${R}_full_c1_iter python bench.py --workload c1 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_full3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${R}_launches_c2.csv python bench.py --workload c2 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_launch2.log 2>&1
ls gpurun_out
