# sharded gradient variant: the gradient GPU tests (old + virtual-shard) and the sharded CUDA-engine gloo test
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_gradient.py tests/test_gpu_sharded.py -m gpu -q -rs -x > gpurun_out/r2gs_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2gs_pytest.log
