# ncu --set full of one warm-started two-sided block Jacobi launch on the C2 stream (n = 256)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_bjacobi_kernel -s 3 -c 1 \
  -o gpurun_out/prof_symjac_c2 python scripts/jacobi_sweep_counts.py > gpurun_out/r2jp_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2jp_ncu.log
