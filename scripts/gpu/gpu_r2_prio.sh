# side-stream priorities in the pipelined schedule; K1F alone baseline
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 300 python scripts/k1_only.py --reps 10 --mode 4 2>&1 | tail -1
for cfg in "x x" "0 0" "0 -1" "-1 0" "x x"; do
  set -- $cfg
  env_args=""
  [ "$1" != "x" ] && env_args="OID_SIDE_PRIO=$1 OID_SIDE2_PRIO=$2"
  env $env_args timeout 300 python bench.py --steps 20 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/prio.log 2>&1
  tail -1 gpurun_out/prio.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('side=$1 side2=$2', round(d['value'],1), round(d['ms_per_step'],3), 'k1', round(d['breakdown_ms_per_step']['k1'],3), 'a9', round(d['a9']['ms_per_launch'],3), 'post', round(d['breakdown_ms_per_step']['post'],3), 'est', round(d['breakdown_ms_per_step']['estimate'],3))"
done
