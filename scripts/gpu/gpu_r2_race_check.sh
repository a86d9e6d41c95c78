python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "two_stream" 2>&1 | tail -1; done
echo "--- without the fix"
python - <<'PY'
p='paper_2405_16076_b200/csrc/oid.cu'
s=open(p).read()
s=s.replace("  est_kappa_kernel<<<1, 1, 0, cs2>>>(ctx->d(L.scal), par);\n  CKL();\n","")
open(p,'w').write(s)
p='paper_2405_16076_b200/csrc/path.cuh'
s=open(p).read()
s=s.replace("  scal[SC_FROB2_EST] = scal[SC_FROB2_SNAP + par];\n}","  scal[SC_FROB2_EST] = scal[SC_FROB2_SNAP + par];\n  scal[SC_KAPPA_EST] = scal[SC_KAPPA_SNAP + par];\n}",1)
open(p,'w').write(s)
PY
python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "two_stream" 2>&1 | tail -1; done
