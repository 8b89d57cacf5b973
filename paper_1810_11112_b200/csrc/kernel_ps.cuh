// Parameter-server step over NVLink (paramserver.py:171-271, the pull model's
// synchronous training step) as one kernel per rank.
//
// Tensors are laid out in sorted-name order (global element offsets). Every
// worker has packed its gradients at staging[e&1] + 0; PS rank q owns the
// tensors the round-robin shard map gives it (paramserver.py:159-165).
//   1. start barrier (per-CTA records, as in collective_kernel)
//   2. owner phase: CTA b takes slice b of the rank's owned elements; per
//      element: acc = (double)g_w0 + g_w1 + ... in worker-rank order, read from
//      every worker's staging over NVLink (PS_U = 8 f32 / 4 f64 elements per thread in
//      flight); mean = acc / W; updated =
//      (T)((double)param - lr * mean) with separately rounded multiply and
//      subtract (no FMA contraction, as numpy evaluates it). The result goes
//      to the rank's parameter buffer and to its "served" area (staging +
//      Gtot elements, same global offsets).
//   3. per-CTA mid flag, then pull phase (workers): slice b of every other
//      owner's owned elements is copied from that owner's served area
//      (16-byte vectors where the offsets allow).
#pragma once

#include "dev_common.cuh"

namespace cm {
namespace dev {
// the served area follows the staged gradients, rounded up to 16 bytes so that
// it shares the 16-byte alignment of the parameter buffers (element offsets
// are equal): the pull phase's vector copies then apply to every piece
__host__ __device__ constexpr long long served_off(long long gtot, long long sz) {
  return (gtot * sz + 127) / 128 * 128;    // own cache lines: no line shared with the staged gradients
}

struct PsParams {
  char* heap[MAXP];
  char* params[MAXP];         // per local rank: fused parameters (in/out), sorted-name layout
  const long long* table;     // device: for each rank q: own_first[q], then entries {prefix, goff, len}
  int p, rank, virt;
  int nworkers;
  int workers[MAXP];          // worker ranks, ascending (the accumulation order)
  unsigned int worker_mask;   // bit q: rank q is a worker
  long long gtot;             // total elements of the schema
  double lr;
  unsigned long long hdr;
  unsigned long long timeout_cycles;
  long long staging_off, staging_bytes;
  unsigned int* herr;
};

// table layout: own_first[0..p] (entry index ranges per rank), then entries of
// 3 long longs {prefix in the owner's space, global offset, length}
__device__ __forceinline__ const long long* ps_entry(const long long* table, int p, long long e) {
  return table + (p + 1) + e * 3;
}

// visit the pieces of [lo, hi) of rank q's owned space as (global offset, count)
template <class F>
__device__ __forceinline__ void ps_pieces(const long long* table, int p, int q, long long lo, long long hi, F&& f) {
  long long a = table[q], z = table[q + 1];           // entries [a, z)
  if (hi <= lo || z <= a) return;
  while (z - a > 1) {                                 // last entry with prefix <= lo
    const long long mid = (a + z) >> 1;
    if (ps_entry(table, p, mid)[0] <= lo) a = mid; else z = mid;
  }
  for (long long e = a; e < table[q + 1]; ++e) {
    const long long* en = ps_entry(table, p, e);
    const long long pre = en[0], goff = en[1], len = en[2];
    if (pre >= hi) break;
    const long long s = lo > pre ? lo : pre, t = hi < pre + len ? hi : pre + len;
    if (t > s) f(goff + (s - pre), t - s);
  }
}



template <class D>
__global__ void __launch_bounds__(THREADS, 1) ps_kernel(const __grid_constant__ PsParams P) {
  using S = typename D::S;
  constexpr int SZ = sizeof(S);
  constexpr int PS_U = SZ == 8 ? 4 : 8;   // elements in flight per thread (f64: keeps 2 CTAs/SM)
  const int lr_ = P.virt ? blockIdx.y : 0;
  const int rank = P.virt ? (int)blockIdx.y : P.rank;
  const int b = blockIdx.x, nb = gridDim.x, p = P.p, tid = threadIdx.x;
  char* myheap = P.heap[rank];
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(myheap + CTRL_OFF);
  __shared__ unsigned long long s_epoch;
  __shared__ int s_err;
  if (tid == 0) {
    s_epoch = epoch_read(myheap, b) + 1;
    s_err = 0;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int par = (int)(e & 1);
  const long long stage_off = P.staging_off + (long long)par * P.staging_bytes;
  S* prm = reinterpret_cast<S*>(P.params[lr_]);

  // 1. start barrier: every worker's gradients are staged (pack kernels ran
  // before this launch on each rank's stream)
  const unsigned tag = ll_tag(e);
  if (tid < p) {
    const long long rv[REC_UNITS] = {(long long)P.hdr, 0, 0, 0, 0, 0};
    rec_put(rec_slot(P.heap[tid], par, b, rank), tag, rv, 1);
  }
  if (tid < p) {
    long long rv[REC_UNITS];
    if (!rec_get(rec_slot(myheap, par, b, tid), tag, rv, 1, P.timeout_cycles)) atomicExch(&s_err, ERR_TRANSPORT);
    else if ((unsigned long long)rv[RF_HDR] != P.hdr) atomicExch(&s_err, ERR_SHAPE);
    __threadfence();
  }
  __syncthreads();
  if (s_err) goto finish;

  {
    // 2. owner phase over slice b of my owned elements
    const long long own = P.table[rank + 1] > P.table[rank]
                              ? ps_entry(P.table, p, P.table[rank + 1] - 1)[0] +
                                    ps_entry(P.table, p, P.table[rank + 1] - 1)[2]
                              : 0;
    const long long lo = slice_bound(0, own, b, nb), hi = slice_bound(0, own, b + 1, nb);
    S* served = reinterpret_cast<S*>(myheap + stage_off + served_off(P.gtot, SZ));
    const double wcount = (double)P.nworkers;
    ps_pieces(P.table, p, rank, lo, hi, [&](long long g0, long long cnt) {
      // PS_U independent elements per thread (strided by THREADS so every
      // load stays coalesced): the NVLink loads of one worker are issued
      // together before the adds; each element keeps its own fold in
      // worker-rank order, so the result is unchanged.
      long long i = tid;
      for (; i + (PS_U - 1) * THREADS < cnt; i += PS_U * THREADS) {
        const long long g = g0 + i;
        double acc[PS_U];
        const S* s0 = reinterpret_cast<const S*>(P.heap[P.workers[0]] + stage_off) + g;
#pragma unroll
        for (int u = 0; u < PS_U; ++u) acc[u] = (double)s0[u * THREADS];
        for (int w = 1; w < P.nworkers; ++w) {
          const S* sw = reinterpret_cast<const S*>(P.heap[P.workers[w]] + stage_off) + g;
          S v[PS_U];
#pragma unroll
          for (int u = 0; u < PS_U; ++u) v[u] = sw[u * THREADS];
#pragma unroll
          for (int u = 0; u < PS_U; ++u) acc[u] = __dadd_rn(acc[u], (double)v[u]);
        }
        S pv[PS_U];
#pragma unroll
        for (int u = 0; u < PS_U; ++u) pv[u] = prm[g + u * THREADS];
#pragma unroll
        for (int u = 0; u < PS_U; ++u) {
          const double mean = __ddiv_rn(acc[u], wcount);
          const S v = (S)__dsub_rn((double)pv[u], __dmul_rn(P.lr, mean));
          prm[g + u * THREADS] = v;
          served[g + u * THREADS] = v;
        }
      }
      for (; i < cnt; i += THREADS) {
        const long long g = g0 + i;
        double acc = (double)reinterpret_cast<const S*>(P.heap[P.workers[0]] + stage_off)[g];
        for (int w = 1; w < P.nworkers; ++w)
          acc = __dadd_rn(acc, (double)reinterpret_cast<const S*>(P.heap[P.workers[w]] + stage_off)[g]);
        const double mean = __ddiv_rn(acc, wcount);
        const double upd = __dsub_rn((double)prm[g], __dmul_rn(P.lr, mean));
        const S v = (S)upd;
        prm[g] = v;
        served[g] = v;
      }
    });
  }
  // 3. publish "slice b of my owned space is served", then pull the others'
  __syncthreads();
  if (tid < p) flag_put(mid_slot(P.heap[tid], b, rank), e);
  if ((P.worker_mask >> rank) & 1u) {
    for (int q = 0; q < p; ++q) {
      if (q == rank || P.table[q + 1] == P.table[q]) continue;
      if (tid == 0 && !flag_wait(mid_slot(myheap, b, q), e, P.timeout_cycles)) atomicExch(&s_err, ERR_TRANSPORT);
      __syncthreads();
      if (s_err) break;
      const long long own = ps_entry(P.table, p, P.table[q + 1] - 1)[0] + ps_entry(P.table, p, P.table[q + 1] - 1)[2];
      const long long lo = slice_bound(0, own, b, nb), hi = slice_bound(0, own, b + 1, nb);
      const S* src = reinterpret_cast<const S*>(P.heap[q] + stage_off + served_off(P.gtot, SZ));
      ps_pieces(P.table, p, q, lo, hi, [&](long long g0, long long cnt) {
        // served area and parameters share the element offset, so they share
        // 16-byte alignment: scalar head, uint4 body, scalar tail
        constexpr long long VE = 16 / SZ;
        const long long head = ((VE - ((reinterpret_cast<uintptr_t>(prm + g0) & 15) / SZ)) % VE);
        const bool vec = ((reinterpret_cast<uintptr_t>(src + g0) ^ reinterpret_cast<uintptr_t>(prm + g0)) & 15) == 0;
        const long long h = vec ? (head < cnt ? head : cnt) : cnt;
        // (peer data: L1-bypassing loads)
        for (long long i = tid; i < h; i += THREADS) prm[g0 + i] = ld_cg_elem(src + g0 + i);
        if (vec) {
          const long long nv = (cnt - h) / VE;
          const uint4* vs = reinterpret_cast<const uint4*>(src + g0 + h);
          uint4* vd = reinterpret_cast<uint4*>(prm + g0 + h);
          long long i = tid;
          for (; i + 3 * THREADS < nv; i += 4 * THREADS) {
            const uint4 a = __ldcg(vs + i), b2 = __ldcg(vs + i + THREADS), c = __ldcg(vs + i + 2 * THREADS),
                        d = __ldcg(vs + i + 3 * THREADS);
            vd[i] = a; vd[i + THREADS] = b2; vd[i + 2 * THREADS] = c; vd[i + 3 * THREADS] = d;
          }
          for (; i < nv; i += THREADS) vd[i] = __ldcg(vs + i);
          for (long long j = h + nv * VE + tid; j < cnt; j += THREADS) prm[g0 + j] = ld_cg_elem(src + g0 + j);
        }
      });
    }
  }

finish:
  __syncthreads();
  if (tid == 0 && s_err) *reinterpret_cast<volatile unsigned*>(P.herr) = (unsigned)s_err;
  epoch_publish(myheap, b, nb, e);
}

}  // namespace dev
}  // namespace cm
