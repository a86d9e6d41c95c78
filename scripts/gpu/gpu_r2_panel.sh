# panel tridiagonalisation (512 < n <= 1024): parity tests, then C5r post-pass timing
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rs -x -k "panel or maximum_sizes or large_basis or c5r" > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2e_pytest.log
timeout 600 python bench.py --workload C5r --steps 8 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2e_c5r.log 2>&1; echo "c5r rc=$?"; tail -1 gpurun_out/r2e_c5r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['breakdown_ms_per_step'], d['block_latency'])"
