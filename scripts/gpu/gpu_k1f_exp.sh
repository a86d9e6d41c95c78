python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 200 python scripts/k1f_check.py --full --reps 5 2>&1 | grep -v "^m=" | tail -9
timeout 200 python scripts/k1f_race.py 300000 30
