set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python scripts/k1_timeline.py > gpurun_out/k1v2_tl.log 2>&1; echo "tl rc=$?"; cat gpurun_out/k1v2_tl.log | tail -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_tc_kernel -s 3 -c 1 -o gpurun_out/prof_k1v2 python scripts/k1_only.py --reps 5 > gpurun_out/ncu_k1v2.log 2>&1; echo "ncu rc=$?"
