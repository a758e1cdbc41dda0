# final evidence: full GPU suite, smoke, bench lines of every config + reference arm
set -x
R=${1:-r01i}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${R}_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err
for w in c1 c2 c3 c4; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/${R}_bench_$w.json 2> gpurun_out/${R}_bench_$w.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_ref.err
tail -2 gpurun_out/${R}_pytest_gpu.log; tail -1 gpurun_out/${R}_smoke.log
for w in c1 c2 c3 c4 c5 reference; do python -c "import json; d=json.loads(open('gpurun_out/${R}_bench_$w.json').read().strip().splitlines()[-1]); print('$w', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))"; done
