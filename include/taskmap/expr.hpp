// Reference-named forwarding header: code written against the reference's
//   proj/include/taskmap/expr.hpp:1-96 (Expr builders, substitute, rewrite_loads, fold, expr_to_text)
// includes "taskmap/expr.hpp" and compiles unchanged against this library; the
// declarations live in taskmap/ir.hpp (one header for the whole IR layer).
#pragma once
#include "taskmap/ir.hpp"
