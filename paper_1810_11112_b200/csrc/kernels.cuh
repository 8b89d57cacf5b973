// sm_100a device code for the CUDA-aware allreduce: the single include point
// for the per-dtype translation units (inst_*.cu) and the host code (comm.cu).
//
//   dev_common.cuh        heap layout, CollParams, folds, reduce/copy loops
//   kernel_collective.cuh one-/two-shot pull collectives (+ RS/AG, multi-buffer)
//   kernel_ll.cuh         LL one-shot / two-shot (small and medium messages)
//   kernel_rhd.cuh        literal log2(p)-step recursive halving/doubling
//   kernel_copy.cuh       fusion pack (SM and TMA bulk copy), NVLink diagnostics
//   kernel_ps.cuh         parameter-server step (owner update + pull)
//   kernels.cuh           local_reduce and the per-dtype kernel tables
#pragma once

#include "dev_common.cuh"
#include "kernel_collective.cuh"
#include "kernel_ll.cuh"
#include "kernel_rhd.cuh"
#include "kernel_copy.cuh"
#include "kernel_ps.cuh"

namespace cm {
namespace dev {

// ---- local_reduce (core.py:94-110) -------------------------------------------------
template <class D, int OP>
__global__ void __launch_bounds__(THREADS, 1) local_reduce_kernel(const char* a, const char* b, char* out,
                                                              long long n, int vec) {
  using S = typename D::S;
  using A = typename D::A;
  constexpr int W = 16 / sizeof(S);
  const long long nvec = vec ? n / W : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < nvec; j += stride) {
    A u[2][W];
    load_vec<D, W>(a, j * W, u[0]);
    load_vec<D, W>(b, j * W, u[1]);
#pragma unroll
    for (int w = 0; w < W; ++w) u[0][w] = op2<OP>(u[0][w], u[1][w]);
    store_vec<D, W>(out, j * W, u[0]);
  }
  for (long long i = nvec * W + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    A u[2][1];
    load_vec<D, 1>(a, i, u[0]);
    load_vec<D, 1>(b, i, u[1]);
    u[0][0] = op2<OP>(u[0][0], u[1][0]);
    store_vec<D, 1>(out, i, u[0]);
  }
}

// kernel table of one element type: kind 0 collective, 1 pipelined two-shot,
// 2 LL one-shot, 3 LL two-shot, 4 log-p recursive halving/doubling, 5 multi-buffer collective (defined in csrc/inst_<type>.cu)
#define CM_KERNEL_TABLE(D)                                                          \
  template <int OP, int MP>                                                         \
  static void* cm_table_coll_##D(int kind, bool tree) {                             \
    if (kind == 1) return tree ? (void*)collective_kernel<D, OP, MP, true, true, false>    \
                               : (void*)collective_kernel<D, OP, MP, false, true, false>;  \
    if (kind == 5) {                     /* aggregate only: SUM */                 \
      if constexpr (OP == CM_SUM)                                                   \
        return tree ? (void*)collective_kernel<D, OP, MP, true, false, true>        \
                    : (void*)collective_kernel<D, OP, MP, false, false, true>;      \
      return nullptr;                                                               \
    }                                                                               \
    return tree ? (void*)collective_kernel<D, OP, MP, true, false, false>                  \
                : (void*)collective_kernel<D, OP, MP, false, false, false>;                \
  }                                                                                 \
  template <int OP, int MP>                                                         \
  static void* cm_table_ll_##D(int kind, bool tree) {                               \
    if (kind == 2) return tree ? (void*)ll_kernel<D, OP, MP, true> : (void*)ll_kernel<D, OP, MP, false>; \
    return tree ? (void*)ll2_kernel<D, OP, MP, true> : (void*)ll2_kernel<D, OP, MP, false>;              \
  }                                                                                 \
  template <int OP>                                                                 \
  static void* cm_table_op_##D(int kind, int p, bool tree) {                        \
    if (kind == 4) return (void*)rhd_kernel<D, OP>;                                 \
    if (kind == 2 || kind == 3) return p <= 8 ? cm_table_ll_##D<OP, 8>(kind, tree) : cm_table_ll_##D<OP, 16>(kind, tree); \
    if (p <= 2) return cm_table_coll_##D<OP, 2>(kind, tree);                        \
    if (p <= 4) return cm_table_coll_##D<OP, 4>(kind, tree);                        \
    if (p <= 8) return cm_table_coll_##D<OP, 8>(kind, tree);                        \
    return cm_table_coll_##D<OP, 16>(kind, tree);                                   \
  }

}  // namespace dev
}  // namespace cm

using cm_kfn_t = void (*)(cm::dev::CollParams);
// one entry per (type, op) translation unit of csrc/inst.cu
#define CM_INST_DECL(T)                              \
  cm_kfn_t cm_kernels_##T##_sum(int kind, int p, bool tree); \
  cm_kfn_t cm_kernels_##T##_max(int kind, int p, bool tree);
CM_INST_DECL(f32)
CM_INST_DECL(f64)
CM_INST_DECL(bf16)
CM_INST_DECL(i32)
CM_INST_DECL(i64)
#undef CM_INST_DECL
