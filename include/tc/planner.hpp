// Drop-in header name of the reference API (proj/include/tc/planner.hpp); the
// declarations live in tc/contract.hpp.
#pragma once
#include "tc/contract.hpp"
