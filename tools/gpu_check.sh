set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01f_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01f_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/r01f_bench_c5.json 2> gpurun_out/r01f_bench_c5.err; echo bench_rc=$?
tail -3 gpurun_out/r01f_pytest_gpu.log
cat gpurun_out/r01f_bench_c5.json
