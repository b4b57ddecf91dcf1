// Reference-named forwarding header: code written against the reference's
//   proj/include/taskmap/common.hpp:1-46 (Error, fail, DType, floordiv/floormod)
// includes "taskmap/common.hpp" and compiles unchanged against this library; the
// declarations live in taskmap/ir.hpp (one header for the whole IR layer).
#pragma once
#include "taskmap/ir.hpp"
