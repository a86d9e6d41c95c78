# build, gpu tests, default bench, launch list of a short bench
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --skip-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1
echo "$(tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["value"],1), round(d["roofline"]["frac"],3), d["breakdown_ms_per_step"])')"
timeout 600 python bench.py --steps 4 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/plain_b.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv -k "regex:^(?!.*elementwise).*_kernel$" python bench.py --steps 4 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_b.log 2>&1; echo "ncu rc=$?"
