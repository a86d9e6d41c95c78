# round-2 final measurement: GPU tests, smoke, bench (default = C3 with K1F), launch list, K1F and A9 ncu --set full
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/r2f_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2f_smoke.log
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2f_bench.log
timeout 900 python bench.py --k1-mode 2 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2f_bench_exact.log 2>&1; echo "bench exact rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2f_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r2f_bench_ref.log
timeout 600 python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2f_plain_b.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2f_ncu_b.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python scripts/k1_only.py --reps 3 --mode 4 > gpurun_out/r2f_k1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1f_kernel -s 1 -c 1 -o gpurun_out/prof_k1f_r02f python scripts/k1_only.py --reps 3 --mode 4 > gpurun_out/r2f_ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 300 python scripts/gram_only.py > gpurun_out/r2f_gram_only.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:basis_gram_tc -s 1 -c 1 -o gpurun_out/prof_bgtc_r02f python scripts/gram_only.py > gpurun_out/r2f_ncu_bg.log 2>&1; echo "ncu bg rc=$?"
