set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tests/diag_sweeps.py > gpurun_out/diag_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_diag.csv python tests/diag_sweeps.py > gpurun_out/ncu_diag.log 2>&1; echo "ncu rc=$?"
