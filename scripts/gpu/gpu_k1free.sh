python -c "import __graft_entry__ as g; g.build()" || exit 1
for f in 0 1 2 4; do OID_K1_FREE=$f timeout 600 python bench.py --skip-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('free', $f, round(d['value'],1), round(d['ms_per_step'],3), 'k1', round(d['roofline']['k1_ms'],3), 'a9', round(d['a9']['ms_per_launch'],3))"; done
