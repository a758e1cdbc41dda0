# quick A/B: selected GPU tests + bench lines of the given workloads
# usage: bash tools/gpu_quick.sh "<pytest -k expr>" c3 c1 ...
set -x
K="$1"; shift
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/quick_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/quick_pytest.log
for w in "$@"; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/quick_bench_$w.json 2> gpurun_out/quick_bench_$w.err; echo bench_$w=$?
python -c "import json; d=json.loads(open('gpurun_out/quick_bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('kernel_ms_per_pair'))"; done
