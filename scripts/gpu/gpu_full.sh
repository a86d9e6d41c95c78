# round measurement: full bench, launch list, K1 ncu --set full
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log
timeout 600 python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/plain_b.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_b.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python scripts/k1_only.py --reps 5 > gpurun_out/k1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tc_kernel -s 3 -c 1 -o gpurun_out/prof_k1tc_r01 python scripts/k1_only.py --reps 5 > gpurun_out/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 300 python scripts/gram_only.py > gpurun_out/gram_only.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:basis_gram_tc -s 1 -c 1 -o gpurun_out/prof_bgtc_r01 python scripts/gram_only.py > gpurun_out/ncu_bg.log 2>&1; echo "ncu bg rc=$?"
