# defaults changed (pipelined bench, A9Q <= 6 clusters, K1 grid 146): suite, bench, basis_quant ncu
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2i_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2i_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2i_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2i_bench.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:basis_quant -s 12 -c 1 -o gpurun_out/prof_bq_r02i python bench.py --steps 6 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2i_ncu_bq.log 2>&1; echo "ncu bq rc=$?"
