# tc/metric.hpp on the device: C-ABI tests + the C++ device suite
python -m pytest tests/test_metric.py tests/test_cpp_suites.py tests/test_abi.py -m gpu -x -q 2>&1 | tail -15
