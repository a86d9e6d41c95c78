python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for cfg in "X=0"; do
  env $cfg timeout 900 python bench.py --skip-cpu-baseline > gpurun_out/bench.log 2>&1
  echo "$cfg: $(tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1), round(d["roofline"]["frac"],3), d["breakdown_ms_per_step"]["k1"], d["e2e"]["value"])')"
done
