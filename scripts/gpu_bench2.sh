# build, then the default bench twice (run-to-run spread)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for r in 1 2; do
timeout 900 python bench.py --skip-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1
echo "$(tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1), round(d["roofline"]["frac"],3), d["breakdown_ms_per_step"])')"
done
