// Reference-named forwarding header: code written against the reference's
//   proj/include/taskmap/compute_ir.hpp:1-121 (ComputeDAG, classify, affine analysis, builders)
// includes "taskmap/compute_ir.hpp" and compiles unchanged against this library; the
// declarations live in taskmap/ir.hpp (one header for the whole IR layer).
//
// Not provided here: reference_eval, Tensor / TensorMap, fold_batchnorm_params
// and reduce_dag (proj/include/taskmap/tensor.hpp, compute_ir.hpp:60,:108-113).
// They are the reference's CPU oracle; this library ships the device
// interpreter tm_dag_eval (taskmap_b200.h) instead, and the oracle itself is
// test infrastructure under oracle/.
#pragma once
#include "taskmap/ir.hpp"
#include "taskmap/schedule.hpp"
