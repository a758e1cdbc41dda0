# 2D check: GPU suite, C4/C5 bench lines
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c45_pytest.log 2>&1; echo pytest_rc=$?
for w in c4 c5 c3; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/c45_bench_$w.json 2> gpurun_out/c45_bench_$w.err; echo bench_$w=$?; done
tail -3 gpurun_out/c45_pytest.log
for f in gpurun_out/c45_bench_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('kernel_ms_per_pair'), d.get('roofline_fp64'))"; done
