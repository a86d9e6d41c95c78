# C3 step with K1 leaving 0 / 1 / 2 SMs to the single-SM core SVD and the chain
python -c "import __graft_entry__ as g; g.build()" || exit 1
for f in 0 1 2 0; do
  OID_K1_FREE=$f timeout 600 python bench.py --steps 12 --warmup 3 --skip-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('free', $f, round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()}, d['a9']['ms_per_launch'])"
done
