# bench under env knob variations (diagnostics)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for cfg in "X=0" "OID_BENCH_INGEST_PRIO=-5" "OID_BENCH_INGEST_PRIO=-3" "OID_BENCH_INGEST_PRIO=-5 OID_GS_GATE=1" "X=1"; do
  env $cfg timeout 900 python bench.py --skip-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1
  echo "$cfg: $(tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1), round(d["roofline"]["frac"],3), d["breakdown_ms_per_step"]["k1"])')"
done
