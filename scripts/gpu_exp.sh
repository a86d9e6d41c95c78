set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --steps 8 --warmup 3 --skip-cpu-baseline --e2e-steps 0"
for cfg in "OID_NO_SIDE=0" "OID_NO_SIDE=1" "OID_BG_FREE=0" "OID_BG_FREE=12" "OID_BG_FREE=20"; do
  env $cfg timeout 600 $B > gpurun_out/exp.log 2>&1; echo "$cfg: $(tail -1 gpurun_out/exp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["breakdown_ms_per_step"])')"
done
timeout 300 python scripts/tri_timeline.py 2>&1 | tail -4
timeout 600 python scripts/bg_compare.py 4 2>&1 | tail -6
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
