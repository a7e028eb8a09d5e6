python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | head -c 300; echo
