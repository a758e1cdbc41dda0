# small-config check: GPU suite, FP64 peak probe, C1-C3 bench lines (fused and generic iteration), launch lists
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c12_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 bash tools/micro/fp64_peak.sh > gpurun_out/fp64_peak.log 2>&1; echo fp64=$?; cp profiles/fp64_peak.json gpurun_out/ 2>/dev/null
for w in c1 c2 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/c12_bench_$w.json 2> gpurun_out/c12_bench_$w.err; echo bench_$w=$?; done
for w in c1 c2; do GS_B200_CG_FUSED=0 timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/c12_bench_${w}_generic.json 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c12_launches_c2.csv python bench.py --workload c2 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/c12_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/c12_pytest.log
for f in gpurun_out/c12_bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('kernel_ms_per_pair'))"; done
