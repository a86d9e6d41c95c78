# re-entry validation: GPU tests, smoke, default bench on the restored checkpoint
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2v_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2v_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2v_smoke.log
timeout 900 python bench.py > gpurun_out/r2v_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2v_bench.log | cut -c1-400
