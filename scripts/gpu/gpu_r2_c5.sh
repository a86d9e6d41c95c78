# C5 measurements: K1 on the per-GPU C5 slab at N=8 (m_loc=2^24, b=64, l=1024, fp32), C5r bench, C5 at N=1
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python scripts/k1_only.py --reps 5 --mode 2 --lowrank-m 16777216 --b 64 --ell 1024
timeout 300 python scripts/k1_only.py --reps 5 --mode 2 --lowrank-m 16777216 --b 32 --ell 1024
timeout 600 python bench.py --workload C5r --steps 8 --warmup 3 --skip-cpu-baseline --e2e-steps 0 > gpurun_out/r2_c5r.log 2>&1; echo "c5r rc=$?"; tail -1 gpurun_out/r2_c5r.log
timeout 600 python bench.py --workload C5r --steps 8 --warmup 3 --skip-cpu-baseline --e2e-steps 0 --no-estimate > gpurun_out/r2_c5r_noest.log 2>&1; tail -1 gpurun_out/r2_c5r_noest.log | cut -c1-600
timeout 300 python bench.py --workload C5 --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/r2_c5.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/r2_c5.log
