# round-2 final measurement (after the sharded gradient variant): GPU tests, smoke, bench, exact bench, reference arm,
# launch list, K1F / A9Q / fp64 A9 ncu --set full
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2k_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2k_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2k_smoke.log
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2k_bench.log | cut -c1-300
timeout 900 python bench.py --k1-mode 2 --a9 fp64 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2k_bench_exact.log 2>&1; echo "bench exact rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2k_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r2k_bench_ref.log | cut -c1-200
timeout 600 python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2k_plain_b.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2k_ncu_b.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python scripts/k1_only.py --reps 3 --mode 4 > gpurun_out/r2k_k1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1f_kernel -s 1 -c 1 -o gpurun_out/prof_k1f_r02k python scripts/k1_only.py --reps 3 --mode 4 > gpurun_out/r2k_ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 300 python scripts/a9q_check.py --full > gpurun_out/r2k_a9q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:gram_q_kernel -s 2 -c 1 -o gpurun_out/prof_a9q_r02k python scripts/a9q_check.py --full > gpurun_out/r2k_ncu_a9q.log 2>&1; echo "ncu a9q rc=$?"
timeout 600 python bench.py --workload C2 --steps 10 --warmup 3 --skip-cpu-baseline > gpurun_out/r2k_bench_C2.log 2>&1; echo "bench C2 rc=$?"
