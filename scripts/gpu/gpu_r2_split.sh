# pipelined estimates, A9Q <= 6 clusters: K1F grid 148 - OID_K1_FREE
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for f in 0 1 2 16; do
  OID_K1_FREE=$f OID_A9Q_CL=6 timeout 300 python bench.py --steps 20 --warmup 3 --skip-cpu-baseline --e2e-steps 0 --pipeline > gpurun_out/free_$f.log 2>&1
  tail -1 gpurun_out/free_$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K1_FREE=$f', round(d['value'],1), round(d['ms_per_step'],3), 'k1', round(d['breakdown_ms_per_step']['k1'],3), 'a9', round(d['a9']['ms_per_launch'],3), 'post', round(d['breakdown_ms_per_step']['post'],3), 'lat', round(d['block_latency']['median_ms'],3))"
done
OID_A9Q_CL=6 timeout 300 python scripts/timeline.py --pipeline > gpurun_out/timeline_pipe6.log 2>&1; echo "timeline rc=$?"; tail -40 gpurun_out/timeline_pipe6.log
