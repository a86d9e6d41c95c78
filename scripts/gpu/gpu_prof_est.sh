set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py --steps 1 --warmup 4 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/plain_est.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"basis_gram_dirty_kernel" -s 3 -c 1 -o gpurun_out/prof_bg python bench.py --steps 1 --warmup 4 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_est.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_est.log
