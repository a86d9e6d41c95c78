python -c "import __graft_entry__ as g; g.build()" || exit 1
for e in 0 7; do echo "exp=$e"; OID_K1_EXP=$e timeout 120 python scripts/k1_timeline.py 2>&1 | sed -n 2,9p; done
