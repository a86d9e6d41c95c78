# copy kernel with 32-bit item indices: A9Q tests, bench x2, steady-state timeline
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_k1fast.py -q -x > gpurun_out/bq_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bq_pytest.log
for i in 1 2; do timeout 600 python bench.py --skip-cpu-baseline --e2e-steps 0 > gpurun_out/bq_bench$i.log 2>&1; tail -1 gpurun_out/bq_bench$i.log | cut -c150-260; done
timeout 300 python scripts/timeline.py --pipeline --start 20 > gpurun_out/timeline_ss.log 2>&1; echo "timeline rc=$?"
