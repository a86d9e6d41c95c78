# full bench (default steps) + launch list of a short bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log
timeout 600 python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/plain_b.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_b.log 2>&1; echo "ncu rc=$?"
