# iteration loop: build, gpu tests, smoke, short bench, launch list of the same short bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 8 --warmup 3 --skip-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
timeout 600 python bench.py --steps 4 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/plain_b.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv python bench.py --steps 4 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_b.log 2>&1; echo "ncu rc=$?"
