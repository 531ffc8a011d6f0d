# round-end evidence with graph replay on by default (capture on the 24th sighting)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r25_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r25_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash tools/scripts/final_bench.sh
