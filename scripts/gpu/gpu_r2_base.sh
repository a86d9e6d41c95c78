set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py --skip-cpu-baseline > gpurun_out/r2_bench_base.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_bench_base.log
