set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python scripts/k1_only.py --reps 5 > gpurun_out/k1_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/k1_plain.log
timeout 300 python scripts/k1_only.py --reps 5 > gpurun_out/k1_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tc_kernel -s 3 -c 1 -o gpurun_out/prof_k1tc_v5 python scripts/k1_only.py --reps 5 > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?"
