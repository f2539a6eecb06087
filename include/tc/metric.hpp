// Drop-in header name of the reference API (proj/include/tc/metric.hpp):
// MetricTensor, invert_metric, spherical_metric, lower_index, raise_index.
// The declarations live in tc/contract.hpp.
#pragma once
#include "tc/contract.hpp"
