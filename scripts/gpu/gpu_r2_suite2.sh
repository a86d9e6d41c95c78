# full GPU suite twice (flake check), smoke
python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2k_pytest_$i.log 2>&1; echo "pytest $i rc=$?"; tail -3 gpurun_out/r2k_pytest_$i.log; grep -E "^FAILED" gpurun_out/r2k_pytest_$i.log; done
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
