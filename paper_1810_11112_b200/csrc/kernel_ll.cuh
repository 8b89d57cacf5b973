// LL (flag-in-data) one-shot and two-shot kernels for small and medium messages
// (part of the sm_100a device code; see kernels.cuh for the overview)
#pragma once

#include "dev_common.cuh"

namespace cm {
namespace dev {
// ---- LL one-shot (small messages) ------------------------------------------------
// Rank r writes every 8-byte unit of its input into slot [par][r][u] of EVERY
// rank's heap as {w0, flag, w1, flag} with one 16-byte volatile store; readers
// poll their own heap until both flags equal the call's epoch tag, then fold
// the p sources in the reference order. No fence, no separate flag round trip:
// latency = launch + one NVLink store + local polls. Header units carry the
// call signature so mismatched peers raise ShapeError.
#define LLSLOT(heap, par, phase, src, u) \
  ((heap) + LL_OFF + ((((size_t)(par) * 2 + (phase)) * P.p + (src)) * (size_t)P.ll_units + (size_t)(u)) * 16)
__device__ __forceinline__ char* llh_slot(char* heap, int par, int blk, int src) {
  return heap + LLH_OFF + (((size_t)par * MAXBLK + blk) * MAXP + src) * 16;
}

template <class D, int OP, int MP, bool TREE>
__global__ void __launch_bounds__(THREADS, 1) ll_kernel(const __grid_constant__ CollParams P) {
  pdl_begin();
  using S = typename D::S;
  using A = typename D::A;
  constexpr int E = 8 / sizeof(S);                    // elements per unit
  const int lr = P.virt ? blockIdx.y : 0;
  const int rank = P.virt ? (int)blockIdx.y : P.rank;
  const int b = blockIdx.x, nb = gridDim.x, p = P.p, tid = threadIdx.x;
  char* myheap = P.heap[rank];
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(myheap + CTRL_OFF);
  if (gated_out(P, ctrl)) return;
  __shared__ unsigned long long s_epoch;
  __shared__ int s_err;
  __shared__ int s_seq[MAXP];
  __shared__ int s_disagree;
  if (tid == 0) {
    s_epoch = epoch_read(myheap, b) + 1;
    s_err = 0;
    s_disagree = 0;
  }
  int m = 1;
  while ((m << 1) <= p) m <<= 1;
  const int excess = p - m;
  if (tid < p) {                                      // fold sequence (see collective_kernel)
    int src;
    if (P.order == ORD_TREE) src = tid < m ? (tid < excess ? 2 * tid : tid + excess) : 2 * (tid - m) + 1;
    else src = tid;
    s_seq[tid] = src;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int par = (int)(e & 1);
  const unsigned flag = (unsigned)(e & 0x7fffffffu) | 0x80000000u;
  const long long nbytes = P.n * (long long)sizeof(S);
  const long long nunits = (nbytes + 7) / 8;
  const long long u0 = nunits * b / nb, u1 = nunits * (b + 1) / nb;
  CM_CHECK(nunits <= P.ll_units, P.herr);
  // prestaged input (fused pack) lives in staging[parity]
  CM_TRACE(P, lr, b, 0);
  const char* in = P.srcmode == SRC_PRESTAGED
                       ? myheap + P.staging_off + (long long)par * P.staging_bytes
                       : P.srcmode == SRC_INLINE ? reinterpret_cast<const char*>(P.inl) : P.in[lr];
  char* out = P.out[lr];

  // header units: this CTA's call signature to every rank
  if (tid < p) {
    st_ll(llh_slot(P.heap[tid], par, b, rank), (unsigned)P.hdr, (unsigned)(P.hdr >> 32), flag);
  }
  // write phase: my units into every rank's slot [par][rank][u]
  for (long long u = u0 + tid; u < u1; u += blockDim.x) {
    unsigned w0 = 0, w1 = 0;
    const long long boff = u * 8;
    if (boff + 8 <= nbytes && ((((uintptr_t)in) & 7u) == 0)) {
      const uint2 v = *reinterpret_cast<const uint2*>(in + boff);
      w0 = v.x;
      w1 = v.y;
    } else {
      unsigned char bytes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int k = 0; k < 8 && boff + k < nbytes; ++k) bytes[k] = (unsigned char)in[boff + k];
      memcpy(&w0, bytes, 4);
      memcpy(&w1, bytes + 4, 4);
    }
#pragma unroll
    for (int q = 0; q < MP; ++q)
      if (q < p) st_ll(LLSLOT(P.heap[q], par, 0, rank, u), w0, w1, flag);
  }
  // header check before trusting the unit count
  if (tid < p) {
    uint4 h;
    if (!ll_wait(llh_slot(myheap, par, b, tid), flag, P.timeout_cycles, &h)) {
      atomicExch(&s_err, ERR_TRANSPORT);
    } else if (((unsigned long long)h.z << 32 | h.x) != P.hdr) {
      atomicExch(&s_err, ERR_SHAPE);
    }
  }
  __syncthreads();
  CM_TRACE(P, lr, b, 2);
  if (s_err) goto ll_finish;
  // read + fold phase
  for (long long u = u0 + tid; u < u1; u += blockDim.x) {
    A v[MP][E];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < MP; ++k) {
      if (k < p) {
        uint4 x;
        if (!ll_wait(LLSLOT(myheap, par, 0, s_seq[k], u), flag, P.timeout_cycles, &x)) {
          ok = false;
          x = make_uint4(0, 0, 0, 0);
        }
        union { uint2 u; S s[E]; } w;
        w.u = make_uint2(x.x, x.z);
#pragma unroll
        for (int t = 0; t < E; ++t) v[k][t] = to_acc<D>(w.s[t]);
      }
    }
    if (!ok) {
      atomicExch(&s_err, ERR_TRANSPORT);
      break;
    }
    fold<OP, MP, E, TREE>(v, p, m, excess);
    union { uint2 u; S s[E]; unsigned char c[8]; } res;
#pragma unroll
    for (int t = 0; t < E; ++t) res.s[t] = from_acc<D>(P.average ? div_p<A>(v[0][t], p) : v[0][t]);
    // agreement check (cm_agree): the MAX of every rank's values equals mine
    // for all values on every rank iff all ranks hold the same values
    if (P.done_flag && u < 8 &&
        (long long)(((unsigned long long)res.u.y << 32) | res.u.x) != reinterpret_cast<const long long*>(in)[u])
      s_disagree = 1;
    const long long boff = u * 8;
    if (boff + 8 <= nbytes && ((((uintptr_t)out) & 7u) == 0)) {
      *reinterpret_cast<uint2*>(out + boff) = res.u;
    } else {
      for (int k = 0; k < 8 && boff + k < nbytes; ++k) out[boff + k] = (char)res.c[k];
    }
  }
ll_finish:
  __syncthreads();
  CM_TRACE(P, lr, b, 5);
  if (tid == 0) {
    if (s_err) *reinterpret_cast<volatile unsigned*>(P.herr) = (unsigned)s_err;
    if (P.done_flag) {                   // host spins on this (cm_agree): after every CTA's output
      __threadfence();
      const unsigned old = atomicAdd(&ctrl->done, 1u);
      if (old == (unsigned)nb - 1) {
        ctrl->done = 0;
        ctrl->agree_ok = s_disagree ? 0 : 1;   // read by gated collectives queued behind
        ctrl->agree_tag = P.done_value;
        __threadfence_system();
        reinterpret_cast<volatile unsigned long long*>(P.done_flag)[lr] = P.done_value;
      }
    }
  }
  epoch_publish(myheap, b, nb, e);
}

// ---- LL two-shot (medium messages) ----------------------------------------------
// reduce-scatter by PUSH: every rank writes unit u of segment q of its input
// into the owner q's LL slot [par][0][src][u]; the owner polls its own heap,
// folds the p sources in the reference order (ring rotation or RHD tree) and
// pushes the reduced unit to every peer's slot [par][1][owner][u]; readers
// poll locally and write their output. No barriers and no fences: every
// 16-byte unit carries its own epoch flags, so each hop costs one posted
// NVLink store plus a local poll.
template <class D>
__device__ __forceinline__ uint2 pack_elems(const char* base, long long i, int cnt) {
  using S = typename D::S;
  constexpr int E = 8 / sizeof(S);
  union { uint2 u; S s[E]; } w;
  w.u = make_uint2(0, 0);
  const S* src = reinterpret_cast<const S*>(base) + i;
#pragma unroll
  for (int t = 0; t < E; ++t)
    if (t < cnt) w.s[t] = src[t];
  return w.u;
}

template <class D>
__device__ __forceinline__ void unpack_elems(char* base, long long i, int cnt, uint2 v) {
  using S = typename D::S;
  constexpr int E = 8 / sizeof(S);
  union { uint2 u; S s[E]; } w;
  w.u = v;
  S* dst = reinterpret_cast<S*>(base) + i;
#pragma unroll
  for (int t = 0; t < E; ++t)
    if (t < cnt) dst[t] = w.s[t];
}

template <class D, int OP, int MP, bool TREE>
__global__ void __launch_bounds__(THREADS, 1) ll2_kernel(const __grid_constant__ CollParams P) {
  pdl_begin();
  using S = typename D::S;
  using A = typename D::A;
  constexpr int E = 8 / sizeof(S);
  const int lr = P.virt ? blockIdx.y : 0;
  const int rank = P.virt ? (int)blockIdx.y : P.rank;
  const int b = blockIdx.x, nb = gridDim.x, p = P.p, tid = threadIdx.x, bd = blockDim.x;
  char* myheap = P.heap[rank];
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(myheap + CTRL_OFF);
  if (gated_out(P, ctrl)) return;
  __shared__ unsigned long long s_epoch;
  __shared__ int s_err;
  __shared__ int s_seq[MAXP];
  CM_TRACE(P, lr, b, 0);
  if (tid == 0) {
    s_epoch = epoch_read(myheap, b) + 1;
    s_err = 0;
  }
  int m = 1;
  while ((m << 1) <= p) m <<= 1;
  const int excess = p - m;
  if (tid < p) {
    int src;
    if (P.order == ORD_TREE) src = tid < m ? (tid < excess ? 2 * tid : tid + excess) : 2 * (tid - m) + 1;
    else if (P.order == ORD_RING) src = ((rank - 1 - tid) % p + p) % p;   // x_{r-1}, ..., x_r
    else src = tid;
    s_seq[tid] = src;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int par = (int)(e & 1);
  const unsigned flag = (unsigned)(e & 0x7fffffffu) | 0x80000000u;
  const char* in = P.srcmode == SRC_PRESTAGED
                       ? myheap + P.staging_off + (long long)par * P.staging_bytes
                       : P.in[lr];
  char* out = P.out[lr];

  if (tid < p) st_ll(llh_slot(P.heap[tid], par, b, rank), (unsigned)P.hdr, (unsigned)(P.hdr >> 32), flag);
  // 1. push slice b of every segment to its owner
  for (int i = 0; i < p; ++i) {
    const int q = (rank + 1 + i) % p;               // spread the first stores over peers
    const long long so = P.seg_off[q], sl = P.seg_len[q];
    const long long nu = (sl + E - 1) / E;
    const long long u0 = nu * b / nb, u1 = nu * (b + 1) / nb;
    CM_CHECK(nu <= P.ll_units, P.herr);
    char* dst = P.heap[q];
    for (long long u = u0 + tid; u < u1; u += bd) {
      const long long el = u * E;
      const int cnt = (int)((sl - el) < E ? (sl - el) : E);
      const uint2 w = pack_elems<D>(in, so + el, cnt);
      st_ll(LLSLOT(dst, par, 0, rank, u), w.x, w.y, flag);
    }
  }
  if (tid < p) {
    uint4 h;
    if (!ll_wait(llh_slot(myheap, par, b, tid), flag, P.timeout_cycles, &h)) atomicExch(&s_err, ERR_TRANSPORT);
    else if (((unsigned long long)h.z << 32 | h.x) != P.hdr) atomicExch(&s_err, ERR_SHAPE);
  }
  __syncthreads();
  CM_TRACE(P, lr, b, 2);
  if (s_err) goto ll2_finish;
  {
    // 2. reduce my segment, write it and push it to every peer
    const long long so = P.seg_off[rank], sl = P.seg_len[rank];
    const long long nu = (sl + E - 1) / E;
    const long long u0 = nu * b / nb, u1 = nu * (b + 1) / nb;
    for (long long u = u0 + tid; u < u1; u += bd) {
      A v[MP][E];
      bool ok = true;
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        if (k < p) {
          uint4 x;
          if (!ll_wait(LLSLOT(myheap, par, 0, s_seq[k], u), flag, P.timeout_cycles, &x)) {
            ok = false;
            x = make_uint4(0, 0, 0, 0);
          }
          union { uint2 u; S s[E]; } w;
          w.u = make_uint2(x.x, x.z);
#pragma unroll
          for (int t = 0; t < E; ++t) v[k][t] = to_acc<D>(w.s[t]);
        }
      }
      if (!ok) {
        atomicExch(&s_err, ERR_TRANSPORT);
        break;
      }
      fold<OP, MP, E, TREE>(v, p, m, excess);
      union { uint2 u; S s[E]; } r;
#pragma unroll
      for (int t = 0; t < E; ++t) r.s[t] = from_acc<D>(P.average ? div_p<A>(v[0][t], p) : v[0][t]);
      const long long el = u * E;
      const int cnt = (int)((sl - el) < E ? (sl - el) : E);
      for (int i = 1; i < p; ++i) {
        const int q = (rank + i) % p;
        st_ll(LLSLOT(P.heap[q], par, 1, rank, u), r.u.x, r.u.y, flag);
      }
      unpack_elems<D>(out, so + el, cnt, r.u);
    }
    CM_TRACE(P, lr, b, 3);
    // 3. collect every other segment
    for (int i = 1; i < p; ++i) {
      const int q = (rank + i) % p;
      const long long qo = P.seg_off[q], ql = P.seg_len[q];
      const long long qn = (ql + E - 1) / E;
      const long long q0 = qn * b / nb, q1 = qn * (b + 1) / nb;
      for (long long u = q0 + tid; u < q1; u += bd) {
        uint4 x;
        if (!ll_wait(LLSLOT(myheap, par, 1, q, u), flag, P.timeout_cycles, &x)) {
          atomicExch(&s_err, ERR_TRANSPORT);
          break;
        }
        const long long el = u * E;
        const int cnt = (int)((ql - el) < E ? (ql - el) : E);
        unpack_elems<D>(out, qo + el, cnt, make_uint2(x.x, x.z));
      }
    }
  }
ll2_finish:
  __syncthreads();
  CM_TRACE(P, lr, b, 5);
  if (tid == 0 && s_err) *reinterpret_cast<volatile unsigned*>(P.herr) = (unsigned)s_err;
  epoch_publish(myheap, b, nb, e);
}

}  // namespace dev
}  // namespace cm
