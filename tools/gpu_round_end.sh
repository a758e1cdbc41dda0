# final evidence: full GPU suite, smoke, bench lines of every config (with the
# CPU baseline) + variants + reference arm + ncu launch lists / full captures.
# usage (GPU box): bash tools/gpu_round_end.sh r02f
set -x
R=${1:-r02f}
timeout 3000 python -m pytest tests -m gpu -q -s > gpurun_out/${R}_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err
for w in c1 c2 c3 c4; do python bench.py --workload $w > gpurun_out/${R}_bench_$w.json 2> gpurun_out/${R}_bench_$w.err; done
python bench.py --workload c2 --exact-ndft --no-cpu-baseline > gpurun_out/${R}_bench_c2_ndft.json 2> /dev/null
python bench.py --workload c3 --tensor-route --no-cpu-baseline > gpurun_out/${R}_bench_c3_tensor.json 2> /dev/null
python bench.py --workload c4 --shard-samples > gpurun_out/${R}_bench_c4_sharded.json 2> /dev/null
for w in c5 c1 c2 c3 c4; do python bench.py --impl reference --workload $w --steps 2 --warmup 3 > gpurun_out/${R}_bench_reference_$w.json 2> gpurun_out/${R}_ref_$w.err; done
python tools/ndft_bench.py 5 > gpurun_out/${R}_ndft_bench.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_c5_16problems.csv python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2f_ -s 2 -c 2 -o gpurun_out/${R}_full_k2f python tools/prof_pair.py --problems 16 --reps 3 --cgls > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2f_ -s 2 -c 2 -o gpurun_out/${R}_full_k2f_c4 python tools/prof_pair.py --workload c4 --problems 1 --reps 3 --cgls > gpurun_out/ncu_full_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${R}_launches_c4.csv python tools/prof_pair.py --workload c4 --problems 1 --reps 3 --cgls > gpurun_out/ncu_launch4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${R}_launches_c2.csv python bench.py --workload c2 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_launch2.log 2>&1
tail -n 3 gpurun_out/${R}_pytest_gpu.log; tail -n 1 gpurun_out/${R}_smoke.log
for f in gpurun_out/${R}_bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('cpu_baseline') or {}).get('value'), (d.get('cpu_baseline') or {}).get('kind'), (d.get('clocks') or {}).get('sm_mhz'))"; done
