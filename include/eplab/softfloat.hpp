// eplab/softfloat.hpp -- the reference header's name (/root/reference/proj/src/eplab/softfloat.hpp:10-28), so callers
// written against the reference -- including its own unit tests, compiled against this library in
// tests/test_reference_suite.py -- include it unchanged. Every declaration lives in eplab.hpp.
#pragma once
#include "eplab/eplab.hpp"
