# re-run the GPU tests after the fixes, K1 timings (generated vs stored omega), DMMA co-issue micro
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2c_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2c_pytest_gpu.log
for oc in 0 1; do timeout 300 python scripts/k1_only.py --reps 8 --mode 2 --omega-cache $oc; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_dfma scripts/micro/mma_dfma.cu && timeout 120 /tmp/mma_dfma
