# K1F slicer A-stage wait: test_wait + nanosleep(N) vs try_wait loop
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for n in 0 32 100 300 1000 0; do
  echo -n "sleep=$n "; OID_K1F_SLEEP=$n timeout 300 python scripts/k1_only.py --reps 12 --mode 4 2>&1 | tail -1
done
for n in 0 100 300; do
  OID_K1F_SLEEP=$n timeout 300 python bench.py --steps 20 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/sleep.log 2>&1
  tail -1 gpurun_out/sleep.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('bench sleep=$n', round(d['value'],1), round(d['ms_per_step'],3), 'k1', round(d['breakdown_ms_per_step']['k1'],3))"
done
