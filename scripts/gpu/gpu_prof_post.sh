set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tests/diag_sweeps.py > gpurun_out/diag_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tridiag_cluster_kernel|small_svd_kernel|tri_scores_multi_kernel|multisect_kernel" -s 8 -c 4 -o gpurun_out/prof_post python tests/diag_sweeps.py > gpurun_out/ncu_post.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_post.log
