# final evidence: full GPU suite, smoke, default bench, ncu launch list
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash tools/scripts/final_bench.sh
