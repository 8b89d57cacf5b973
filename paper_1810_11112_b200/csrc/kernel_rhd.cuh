// literal log2(p)-step recursive halving/doubling kernel (rhd_logp)
// (part of the sm_100a device code; see kernels.cuh for the overview)
#pragma once

#include "dev_common.cuh"

namespace cm {
namespace dev {
// ---- recursive halving / doubling in log2(p) pairwise steps ---------------------
// The reference's rhd_rsa schedule (collectives.py:155-236) executed literally
// over NVLink: fold of the excess odd ranks into their even neighbours, log2(m)
// halving steps (partner vrank ^ 2^k, lower vrank keeps [lo, mid)), log2(m)
// doubling steps in reverse, unfold. Each step pulls the partner's half from
// its staging buffer and is ordered by ONE pairwise flag per CTA: every CTA
// owns the same slice of [0, n) in every phase, so CTA b only ever depends on
// CTA b of its partner (no grid-wide barrier). Element results equal the
// balanced vrank tree (Appendix A.3) bit for bit; the direct kernels compute
// the same tree in one or two exchanges, which is why they are the default.
struct RFlag {
  unsigned long long v;
  unsigned long long hdr;
};

__device__ __forceinline__ RFlag* rflag_slot(char* heap, int src, int blk) {
  return reinterpret_cast<RFlag*>(heap + RHDF_OFF) + ((size_t)src * MAXBLK + blk);
}

// dst_raw[i] = a[i] (op) b[i] (b == nullptr: a[i]); dst_out[i] = the same value,
// divided by p when averaging. Either destination may be null. i in [lo, hi).
template <class D, int OP>
__device__ void pair_pass(const char* a, const char* b, char* dst_raw, char* dst_out, long long lo,
                          long long hi, int average, int p) {
  using S = typename D::S;
  using A = typename D::A;
  constexpr int W = 16 / sizeof(S);
  constexpr int U = 4;
  if (lo >= hi) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool vec = al16(a) && (!b || al16(b)) && (!dst_raw || al16(dst_raw)) && (!dst_out || al16(dst_out));
  long long blo = hi, bhi = hi;
  if (vec) {
    blo = ((lo + W - 1) / W) * W;
    bhi = (hi / W) * W;
    if (bhi < blo) blo = bhi = hi;
  }
  auto one = [&](long long i) {
    A u[1], t[1];
    load_vec<D, 1>(a, i, u);
    if (b) {
      load_vec<D, 1>(b, i, t);
      u[0] = op2<OP>(u[0], t[0]);
    }
    if (dst_raw) store_vec<D, 1>(dst_raw, i, u);
    if (dst_out) {
      if (average) u[0] = div_p<A>(u[0], p);
      store_vec<D, 1>(dst_out, i, u);
    }
  };
  for (long long i = lo + tid; i < blo; i += nthr) one(i);
  for (long long i = bhi + tid; i < hi; i += nthr) one(i);
  const long long v0 = blo / W, v1 = bhi / W;
  for (long long j = v0 + tid; j < v1; j += U * (long long)nthr) {
    A u[U][W], t[U][W];
#pragma unroll
    for (int g = 0; g < U; ++g) {
      const long long jj = j + g * (long long)nthr;
      if (jj < v1) {
        load_vec<D, W>(a, jj * W, u[g]);
        if (b) load_vec<D, W>(b, jj * W, t[g]);
      }
    }
#pragma unroll
    for (int g = 0; g < U; ++g) {
      const long long jj = j + g * (long long)nthr;
      if (jj >= v1) break;
      if (b) {
#pragma unroll
        for (int w = 0; w < W; ++w) u[g][w] = op2<OP>(u[g][w], t[g][w]);
      }
      if (dst_raw) store_vec<D, W>(dst_raw, jj * W, u[g]);
      if (dst_out) {
        if (average) {
#pragma unroll
          for (int w = 0; w < W; ++w) u[g][w] = div_p<A>(u[g][w], p);
        }
        store_vec<D, W>(dst_out, jj * W, u[g]);
      }
    }
  }
}

template <class D, int OP>
__global__ void __launch_bounds__(THREADS, 1) rhd_kernel(const __grid_constant__ CollParams P) {
  pdl_begin();
  const int lr = P.virt ? blockIdx.y : 0;
  const int rank = P.virt ? (int)blockIdx.y : P.rank;
  const int b = blockIdx.x, nb = gridDim.x, p = P.p, tid = threadIdx.x;
  char* myheap = P.heap[rank];
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(myheap + CTRL_OFF);
  if (gated_out(P, ctrl)) return;
  __shared__ unsigned long long s_epoch;
  __shared__ int s_err;
  CM_TRACE(P, lr, b, 0);
  if (tid == 0) {
    s_epoch = epoch_read(myheap, b) + 1;
    s_err = 0;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const long long stage_off = P.staging_off + (long long)(e & 1) * P.staging_bytes;
  char* buf = myheap + stage_off;
  char* out = P.out[lr];
  const long long n = P.n;
  const long long lo_b = slice_bound(0, n, b, nb), hi_b = slice_bound(0, n, b + 1, nb);
  int m = 1;
  while ((m << 1) <= p) m <<= 1;
  const int excess = p - m;
  int steps = 0;
  while ((1 << steps) < m) ++steps;
  const bool folded_odd = rank < 2 * excess && (rank & 1);
  const int v = rank < 2 * excess ? rank / 2 : rank - excess;
  const unsigned long long base = e << 8;
  const int ph_fold = excess > 0 ? 1 : 0;
  long long los[MAXP], his[MAXP];        // range after halving step k-1 (level k)

  auto real = [&](int w) { return w < excess ? 2 * w : w + excess; };
  auto peer_buf = [&](int q) -> const char* { return P.heap[q] + stage_off; };
  auto signal = [&](int ph) {
    __syncthreads();                     // this CTA's writes of the phase precede the flag
    if (tid < p) {
      RFlag* f = rflag_slot(P.heap[tid], rank, b);
      st_relaxed_sys(&f->hdr, P.hdr);
      st_release_sys(&f->v, base | (unsigned long long)ph);
    }
  };
  auto wait = [&](int src, int ph) -> bool {
    if (tid == 0) {
      RFlag* f = rflag_slot(myheap, src, b);
      const unsigned long long want = base | (unsigned long long)ph;
      if (!wait_geq(&f->v, want, P.timeout_cycles)) {
        s_err = ERR_TRANSPORT;
      } else if ((ld_acquire_sys(&f->v) >> 8) == e && ld_relaxed_sys(&f->hdr) != P.hdr) {
        s_err = ERR_SHAPE;               // (a flag of a later call means src passed this one)
      }
    }
    __syncthreads();
    return s_err == 0;
  };

  // phase 0: my slice of the input into my staging buffer
  pair_pass<D, OP>(P.in[lr], nullptr, buf, nullptr, lo_b, hi_b, 0, p);
  signal(0);
  CM_TRACE(P, lr, b, 1);
  // phase 1 (non-power-of-two p): L_v = x_{2v} + x_{2v+1} on the even rank
  if (excess > 0) {
    if (rank < 2 * excess && !(rank & 1)) {
      if (!wait(rank + 1, 0)) goto finish;
      pair_pass<D, OP>(buf, peer_buf(rank + 1), buf, nullptr, lo_b, hi_b, 0, p);
    }
    signal(1);
  }
  CM_TRACE(P, lr, b, 2);
  if (!folded_odd) {
    long long lo = 0, hi = n;
    los[0] = 0;
    his[0] = n;
    for (int k = 0; k < steps; ++k) {            // halving
      const int q = real(v ^ (1 << k));
      const long long mid = lo + (hi - lo) / 2;
      const int bit = (v >> k) & 1;               // 0: lower vrank, keeps [lo, mid)
      const long long klo = bit ? mid : lo, khi = bit ? hi : mid;
      if (!wait(q, ph_fold + k)) goto finish;
      const char* pb = peer_buf(q);
      const bool last = k == steps - 1;
      pair_pass<D, OP>(bit ? pb : buf, bit ? buf : pb, buf, last ? out : nullptr, klo > lo_b ? klo : lo_b,
                       khi < hi_b ? khi : hi_b, P.average, p);
      lo = klo;
      hi = khi;
      los[k + 1] = lo;
      his[k + 1] = hi;
      signal(ph_fold + 1 + k);
    }
    CM_TRACE(P, lr, b, 3);
    for (int t = 0; t < steps; ++t) {            // doubling, reverse order
      const int j = steps - 1 - t;
      const int q = real(v ^ (1 << j));
      if (!wait(q, ph_fold + steps + t)) goto finish;
      const long long ulo = los[j], uhi = his[j], rlo = los[j + 1], rhi = his[j + 1];
      const long long slo = rlo == ulo ? rhi : ulo, shi = rlo == ulo ? uhi : rlo;   // partner's part
      pair_pass<D, OP>(peer_buf(q), nullptr, buf, out, slo > lo_b ? slo : lo_b, shi < hi_b ? shi : hi_b,
                       P.average, p);
      signal(ph_fold + steps + 1 + t);
    }
  } else {                                       // unfold: the result from rank - 1
    if (!wait(rank - 1, ph_fold + 2 * steps)) goto finish;
    pair_pass<D, OP>(peer_buf(rank - 1), nullptr, nullptr, out, lo_b, hi_b, P.average, p);
  }
  CM_TRACE(P, lr, b, 4);

finish:
  __syncthreads();
  CM_TRACE(P, lr, b, 5);
  if (tid == 0 && s_err) *reinterpret_cast<volatile unsigned*>(P.herr) = (unsigned)s_err;
  epoch_publish(myheap, b, nb, e);
}

}  // namespace dev
}  // namespace cm
