python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
( time timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "whole_stream" -rs ) > gpurun_out/c3r_whole.log 2>&1; tail -8 gpurun_out/c3r_whole.log
