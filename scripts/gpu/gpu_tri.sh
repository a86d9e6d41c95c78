set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python scripts/tri_timeline.py 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 8 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["breakdown_ms_per_step"], d["last_estimate"])'
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv python bench.py --steps 4 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_b.log 2>&1; echo "ncu rc=$?"
