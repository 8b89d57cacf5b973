// Kernel instantiations for ONE (element type, reduce op) pair. _build.py
// compiles this file once per pair (-DCM_INST_T=F32 -DCM_INST_OP=CM_SUM ...)
// so the ten kernel tables compile in parallel; see csrc/kernels.cuh.
#include "kernels.cuh"

#if !defined(CM_INST_T) || !defined(CM_INST_OP) || !defined(CM_INST_FN)
#error "compile with -DCM_INST_T=<type> -DCM_INST_OP=<op> -DCM_INST_FN=<entry>"
#endif

#define CM_CAT2(a, b) a##b
#define CM_CAT(a, b) CM_CAT2(a, b)
#define CM_TABLE_OF(T) CM_KERNEL_TABLE(T)   // expands CM_INST_T before pasting

namespace cm {
namespace dev {
CM_TABLE_OF(CM_INST_T)
}  // namespace dev
}  // namespace cm

cm_kfn_t CM_INST_FN(int kind, int p, bool tree) {
  using namespace cm::dev;
  return reinterpret_cast<cm_kfn_t>(CM_CAT(cm_table_op_, CM_INST_T)<CM_INST_OP>(kind, p, tree));
}
