set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python scripts/k1_only.py --reps 5 > gpurun_out/k1v2_plain.log 2>&1; echo "k1 rc=$?"; cat gpurun_out/k1v2_plain.log | tail -5
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch" > gpurun_out/k1v2_sketch.log 2>&1; echo "sketch rc=$?"; tail -30 gpurun_out/k1v2_sketch.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/k1v2_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/k1v2_pytest.log
timeout 300 python bench.py --skip-cpu-baseline --e2e-steps 0 > gpurun_out/k1v2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/k1v2_bench.log | cut -c1-1500
