// Drop-in header name of the reference API (proj/include/tc/tensor_io.hpp); the
// declarations (write_tensor / read_tensor) live in tc/contract.hpp.
#pragma once
#include "tc/contract.hpp"
