set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 4 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench.log
timeout 300 python bench.py --steps 2 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tc_kernel -s 2 -c 1 -o gpurun_out/prof_k1tc python bench.py --steps 2 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
