# K1F: one polling slicer warp on a_empty; tests, K1 alone, bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_k1fast.py -q -x > gpurun_out/k1w_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/k1w_pytest.log
timeout 300 python scripts/k1_only.py --reps 10 --mode 4 > gpurun_out/k1w_k1.log 2>&1; tail -4 gpurun_out/k1w_k1.log
for i in 1 2; do timeout 600 python bench.py --skip-cpu-baseline --e2e-steps 0 > gpurun_out/k1w_bench$i.log 2>&1; tail -1 gpurun_out/k1w_bench$i.log | cut -c150-260; done
