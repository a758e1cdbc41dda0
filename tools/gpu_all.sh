# GPU suite + bench lines of every config (no CPU legs) + the generic-iteration A/B for C3/C4
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/all_pytest.log 2>&1; echo pytest_rc=$?
for w in c1 c2 c3 c4 c5; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/all_bench_$w.json 2> gpurun_out/all_bench_$w.err; echo bench_$w=$?; done
for w in c3 c4; do GS_B200_CG_FUSED=0 timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/all_bench_${w}_generic.json 2>&1; done
tail -3 gpurun_out/all_pytest.log
for f in gpurun_out/all_bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('kernel_ms_per_pair'))"; done
