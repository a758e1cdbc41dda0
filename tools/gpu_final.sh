# round-end style check: full GPU suite + smoke
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/final_pytest.log; cat gpurun_out/final_smoke.log | tail -2
