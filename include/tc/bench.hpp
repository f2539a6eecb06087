// Drop-in header name of the reference API (proj/include/tc/bench.hpp); the
// declarations (BenchConfig / run_bench / write_bench_csv) live in tc/contract.hpp.
#pragma once
#include "tc/contract.hpp"
