// A program written against the reference's C++ API (proj/include/taskmap/
// {common,mapping,expr,compute_ir}.hpp).  tests/test_boundary_cpp.py compiles it
// twice -- against the reference headers + sources (when /root/reference is
// present) and against this repo's headers + libtaskmap_b200.so -- and requires
// identical output: the drop-in boundary of SURVEY §8(b) for the IR layer.
// The part under TASKMAP_B200 uses the spec-only API the reference never
// implemented (schedule_space, partition) and the C ABI.
#include <iostream>
#include <string>
#include <vector>

#include "taskmap/common.hpp"
#include "taskmap/compute_ir.hpp"
#include "taskmap/expr.hpp"
#include "taskmap/mapping.hpp"
#ifdef TASKMAP_B200
#include "taskmap/schedule.hpp"
#include "taskmap_b200.h"
#endif

using namespace taskmap;

static void print_tasks(const char* what, const std::vector<Task>& ts) {
  std::cout << what << ":";
  for (const auto& t : ts) {
    std::cout << " (";
    for (size_t i = 0; i < t.size(); ++i) std::cout << (i ? "," : "") << t[i];
    std::cout << ")";
  }
  std::cout << "\n";
}

int main() {
  // Fig. 5 cooperative load
  TaskMapping fig5 = TaskMapping::repeat({4, 1}) * TaskMapping::spatial({16, 8});
  std::cout << "fig5 " << fig5.to_text() << " workers=" << fig5.num_workers() << " shape=" << fig5.task_shape()[0]
            << "x" << fig5.task_shape()[1] << " tpw=" << fig5.tasks_per_worker() << "\n";
  print_tasks("fig5 w0", fig5.assign(0));
  print_tasks("fig5 w9", fig5.assign(9));
  // the paper's CUDA-core matmul mapping
  TaskMapping mm = parse_mapping("spatial(4, 2) * repeat(2, 2) * spatial(4, 8) * repeat(4, 4)");
  std::cout << "mm " << mm.to_text() << " workers=" << mm.num_workers() << " tpw=" << mm.tasks_per_worker() << "\n";
  std::vector<Task> w33 = mm.assign(33);
  w33.resize(4);
  print_tasks("mm w33", w33);
  std::cout << "visualize\n" << (TaskMapping::spatial({2, 1}) * TaskMapping::repeat({1, 2})).visualize();
  std::cout << "equal " << (parse_mapping(fig5.to_text()) == fig5) << "\n";
  try {
    TaskMapping::compose(TaskMapping::repeat({2}), TaskMapping::spatial({2, 2}));
  } catch (const Error& e) {
    std::cout << "error " << e.what() << "\n";
  }
  try {
    TaskMapping::spatial({2, 2}).assign(4);
  } catch (const Error& e) {
    std::cout << "error " << e.what() << "\n";
  }
  // expressions: construction, folding, substitution, printing (expr.hpp)
  Expr e = add(mul(var("x"), imm(1)), mul(imm(2), imm(3)));
  std::cout << "fold " << expr_to_text(fold(e)) << "\n";
  std::cout << "subst " << expr_to_text(substitute(e, {{"x", add(var("y"), imm(4))}})) << "\n";
  Expr r = rewrite_loads(load("A", {var("i")}), [](const ExprNode& n) -> std::optional<Expr> {
    return mul(load("C", {sub(imm(99), n.args[0])}), fimm(2.0));  // Fig. 11 prologue splice
  });
  std::cout << "rewrite " << expr_to_text(r) << "\n";
  // builders + classify (compute_ir.hpp)
  ComputeDAG conv = conv2d_im2col_dag(1, 4, 8, 8, 8, 3, 3, 1, 1, DType::F32);
  for (const char* n : {"Col", "Wf", "Y", "Out"}) std::cout << "classify " << n << " " << opclass_name(classify(conv, conv.at(n))) << "\n";
  std::cout << "col " << expr_to_text(conv.at("Col").value) << "\n";
  ComputeDAG mmd = matmul_dag(2, 3, 4, DType::I32);
  std::cout << "matmul C " << opclass_name(classify(mmd, mmd.at("C"))) << " shape " << mmd.at("C").shape[0] << "x"
            << mmd.at("C").shape[1] << "\n";
  ComputeDAG tr = transpose_dag({2, 3, 4, 5}, {0, 2, 1, 3}, DType::F32);
  std::cout << "transpose " << opclass_name(classify(tr, tr.nodes.back())) << "\n";
  ComputeDAG rs = reshape_dag({100}, {2, 50}, DType::F32);
  ComputeDAG rm = reshape_dag({2, 50}, {100}, DType::F32);
  std::cout << "reshape split " << opclass_name(classify(rs, rs.nodes.back())) << " merge "
            << opclass_name(classify(rm, rm.nodes.back())) << "\n";
  auto aff = analyze_affine_access(load("Y", {var("p"), add(mul(var("n"), imm(64)), var("q"))}),
                                   {{"n", 2}, {"p", 8}, {"q", 64}});
  std::cout << "affine " << (aff ? aff->size() : 0) << " " << (aff ? (*aff)[1].terms.size() : 0) << "\n";
  ComputeDAG bad = matmul_dag(2, 2, 2, DType::F32);
  bad.nodes.back().axes[0].extent = 3;
  try {
    bad.validate();
  } catch (const Error& e) {
    std::cout << "validate " << e.what() << "\n";
  }
  std::cout << "conv_out " << conv_out_extent(224, 7, 2, 3) << " floordiv " << floordiv(-7, 2) << " floormod "
            << floormod(-7, 2) << "\n";
#ifdef TASKMAP_B200
  // spec-only API of the B200 build
  auto space = schedule_space("matmul");
  std::cout << "b200 schedule_space " << space.size() << " first " << space[0].key() << "\n";
  ComputeDAG cbr = conv2d_im2col_dag(1, 4, 8, 8, 8, 3, 3, 1, 1, DType::F32);
  for (const auto& sg : partition(cbr))
    std::cout << "b200 partition anchor=" << sg.anchor << " prologue=" << sg.prologue.size()
              << " epilogue=" << sg.epilogue.size() << " output=" << sg.output << "\n";
  std::cout << "b200 " << tm_version() << "\n";
#endif
  return 0;
}
