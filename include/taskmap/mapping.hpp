// Reference-named forwarding header: code written against the reference's
//   proj/include/taskmap/mapping.hpp:1-92 (TaskShape, TaskMapping, operator*, parse_mapping)
// includes "taskmap/mapping.hpp" and compiles unchanged against this library; the
// declarations live in taskmap/ir.hpp (one header for the whole IR layer).
#pragma once
#include "taskmap/ir.hpp"
