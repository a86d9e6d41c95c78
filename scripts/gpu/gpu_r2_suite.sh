# full GPU suite, small-config benches (C1, C2 latency-bound; C5r), both coefficient modes end to end
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2j_pytest.log
timeout 300 python scripts/sanitize_c1.py; timeout 300 python scripts/sanitize_c1.py --argmin
for w in C1 C2; do timeout 900 python bench.py --workload $w --steps 24 --warmup 3 --e2e-steps 2 --cpu-sample-rows 100000000 > gpurun_out/r2j_bench_$w.log 2>&1; echo "$w rc=$?"; tail -1 gpurun_out/r2j_bench_$w.log | cut -c1-900; done
