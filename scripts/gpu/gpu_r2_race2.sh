#!/bin/bash
# two-stream estimate race repro + the A9Q grid change tests
set -x
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/race2_build.log 2>&1
timeout 900 python scripts/race_two_stream.py --reps 6 > gpurun_out/race2.log 2>&1
echo "race rc=$?"
timeout 900 python -m pytest tests/test_gpu_k1fast.py -q -x > gpurun_out/race2_k1fast.log 2>&1
echo "k1fast rc=$?"; tail -3 gpurun_out/race2_k1fast.log
