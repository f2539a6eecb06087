// Drop-in header name of the reference API (proj/include/tc/oracle.hpp):
// resource_limit_error, OracleStats and contract_naive. The declarations live
// in tc/contract.hpp.
#pragma once
#include "tc/contract.hpp"
