python -c "import __graft_entry__ as g; g.build()" || exit 1
for fl in "--no-estimate" "--one-stream" ""; do
  timeout 900 python bench.py --skip-cpu-baseline --e2e-steps 0 $fl > gpurun_out/bench.log 2>&1
  echo "$fl: $(tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1), round(d["roofline"]["frac"],3), d["breakdown_ms_per_step"])')"
done
timeout 300 python scripts/timeline.py --start 20 --one-stream > gpurun_out/tl1.log 2>&1; echo rc=$?
