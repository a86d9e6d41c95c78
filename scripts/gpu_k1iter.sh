python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python scripts/k1_timeline.py 2>&1 | sed -n 2,9p
timeout 120 python scripts/k1_only.py --reps 5 2>&1 | tail -1
timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
