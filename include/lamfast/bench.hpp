// Drop-in header name of the reference's lamfast/bench.hpp; the B200 edition
// declares the whole API in one place.
#pragma once
#include "lamfast/lamfast_b200.hpp"
