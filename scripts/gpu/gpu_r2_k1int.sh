# K1 integer-slicer + stored-omega check: GPU tests, K1 timings per variant, one ncu capture
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2b_pytest_gpu.log
for oc in 0 1; do timeout 300 python scripts/k1_only.py --reps 8 --mode 2 --omega-cache $oc; done
timeout 300 python scripts/k1_only.py --reps 8 --mode 2 --b 64 --grid 256,128,256
timeout 300 python scripts/k1_only.py --reps 5 --mode 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tc_kernel -s 3 -c 1 -o gpurun_out/prof_k1tc_r02b python scripts/k1_only.py --reps 5 --mode 2 > gpurun_out/r2b_ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
