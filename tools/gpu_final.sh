# round-end style check: full GPU suite + smoke + C1/C2 bench lines
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke_rc=$?
for w in c1 c2; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r01h_bench_$w.json 2> gpurun_out/r01h_bench_$w.err; done
tail -3 gpurun_out/final_pytest.log; grep -E "FAILED|Error" gpurun_out/final_pytest.log | head; cat gpurun_out/final_smoke.log | tail -2
for w in c1 c2; do python -c "import json; d=json.loads(open('gpurun_out/r01h_bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
