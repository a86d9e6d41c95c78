python -c "import __graft_entry__ as g; g.build()" || exit 1
for ov in 0 1; do OID_A9Q_OVERLAP=$ov timeout 600 python bench.py --skip-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap', $ov, round(d['value'],1), round(d['ms_per_step'],3), 'k1', round(d['roofline']['k1_ms'],3), 'a9', round(d['a9']['ms_per_launch'],3), d['block_latency'])"; done
timeout 300 python scripts/timeline.py --start 22 2>&1 | tail -1
