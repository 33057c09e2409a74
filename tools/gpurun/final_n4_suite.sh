mkdir -p gpurun_out/s4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/s4/suite.txt 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/s4/suite.txt; grep FAILED gpurun_out/s4/suite.txt | head
