#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
RACE_K1=2 RACE_MODES=def+hilo,noside2,hi+hilo timeout 600 python scripts/race_two_stream.py --reps 12 > gpurun_out/race7.log 2>&1; echo "rc=$?"
grep VARIANT gpurun_out/race7.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "two_stream or side_streams" > gpurun_out/race7_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/race7_pytest.log
