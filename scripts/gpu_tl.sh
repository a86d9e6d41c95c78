python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/timeline.py > gpurun_out/tl2.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 8 --warmup 3 --skip-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["breakdown_ms_per_step"], d["e2e"]["value"])'
timeout 300 python scripts/gram_only.py > gpurun_out/gram_only.log 2>&1; echo "gram_only rc=$?"; tail -2 gpurun_out/gram_only.log
timeout 900 ncu --set full --import-source on -k regex:basis_gram_tc -s 1 -c 1 -o gpurun_out/prof_bgtc2 python scripts/gram_only.py > gpurun_out/ncu_bg.log 2>&1; echo "ncu rc=$?"
