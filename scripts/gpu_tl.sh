python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/timeline.py --start 20 > gpurun_out/tl2.log 2>&1; echo rc=$?
timeout 900 python bench.py --skip-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["breakdown_ms_per_step"], d["e2e"]["value"], d["last_estimate"])'
