timeout 600 python -m pytest tests/test_cpp_shim.py -q -x --timeout=300 2>&1 | tail -3
tests/cpp/_bin/shim_test | tail -5
