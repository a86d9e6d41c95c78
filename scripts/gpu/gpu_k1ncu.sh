python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_tc_kernel -s 3 -c 1 -o gpurun_out/prof_k1v2g python scripts/k1_only.py --reps 5 > gpurun_out/ncu_k1v2c.log 2>&1; echo "ncu rc=$?"
