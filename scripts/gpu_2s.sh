set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for a in "" "--one-stream" "WAVES=4" "WAVES=2"; do
  case $a in WAVES=*) export OID_BG_WAVES=${a#WAVES=}; arg="";; *) arg=$a;; esac
  timeout 600 python bench.py --steps 8 --warmup 3 --skip-cpu-baseline $arg > gpurun_out/bench.log 2>&1; echo "bench $a rc=$?"
  tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["breakdown_ms_per_step"], d["e2e"]["value"])'
done
