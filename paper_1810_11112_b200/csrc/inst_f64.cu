// Kernel instantiations for element type F64 (one translation unit per type so
// nvcc compiles them in parallel; see csrc/kernels.cuh).
#include "kernels.cuh"

namespace cm {
namespace dev {
CM_KERNEL_TABLE(F64)
}  // namespace dev
}  // namespace cm

cm_kfn_t cm_kernels_f64(int kind, int op, int p, bool tree) {
  using namespace cm::dev;
  void* f = op == CM_SUM ? cm_table_op_F64<CM_SUM>(kind, p, tree) : cm_table_op_F64<CM_MAX>(kind, p, tree);
  return reinterpret_cast<cm_kfn_t>(f);
}
