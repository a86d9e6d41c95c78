# HEAD check: build, GPU tests, smoke, default bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -q -rs -x > gpurun_out/chk_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/chk_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/chk_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/chk_smoke.log
timeout 900 python bench.py > gpurun_out/chk_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/chk_bench.log
