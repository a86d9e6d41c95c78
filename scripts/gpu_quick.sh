# quick GPU validation: build, gpu tests, smoke, bench (no ncu)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 4 --warmup 3 --skip-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
timeout 300 python tests/diag_sweeps.py > gpurun_out/diag.log 2>&1; tail -20 gpurun_out/diag.log
timeout 300 python scripts/k1_only.py --reps 5 > gpurun_out/k1_plain.log 2>&1; cat gpurun_out/k1_plain.log
