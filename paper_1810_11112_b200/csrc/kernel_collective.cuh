// collective_kernel: one-/two-shot pull allreduce, reduce-scatter, allgather, multi-buffer and gather variants, pipelined (STREAM) variant
// (part of the sm_100a device code; see kernels.cuh for the overview)
#pragma once

#include "dev_common.cuh"

namespace cm {
namespace dev {
// ---- the collective kernel -------------------------------------------------------
constexpr int RS_WARPS = 8;                      // reducer warps of the pipelined two-shot
__device__ __forceinline__ unsigned long long* wmid_slot(char* heap, int blk, int src, int warp) {
  return reinterpret_cast<unsigned long long*>(heap + WMID_OFF +
                                               (((size_t)blk * MAXP + src) * RS_WARPS + warp) * 8);
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// chunk k of slice [lo, hi): the first chunk ends at the first 64-aligned
// boundary + C, later chunks are C elements on 64-aligned boundaries
__device__ __forceinline__ void chunk_of(long long lo, long long hi, long long C, long long k,
                                         long long* a, long long* z) {
  const long long base = ((lo + SLICE_ALIGN - 1) / SLICE_ALIGN) * SLICE_ALIGN;
  long long x = k == 0 ? lo : base + k * C;
  long long y = base + (k + 1) * C;
  if (x > hi) x = hi;
  if (y > hi) y = hi;
  if (y < x) y = x;
  *a = x;
  *z = y;
}
__device__ __forceinline__ long long chunks_of(long long lo, long long hi, long long C) {
  const long long base = ((lo + SLICE_ALIGN - 1) / SLICE_ALIGN) * SLICE_ALIGN;
  return hi <= base ? 1 : (hi - base + C - 1) / C;
}

template <class D, int OP, int MP, bool TREE>
__device__ void stream_body(const CollParams& P, int rank, int b, int nb, unsigned long long e,
                            const char* const* s_src, char* const* s_red, const char* const* s_seq,
                            int* s_err, char* out, char* myheap) {
  using S = typename D::S;
  constexpr int SZ = sizeof(S);
  constexpr int W = 16 / SZ;
  constexpr int NR = RS_WARPS * 32;                // threads per role
  const int p = P.p, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long C = P.stream_chunk;
  // common chunk count (identical on every rank and for every segment)
  long long K = 1;
  for (int q = 0; q < p; ++q) {
    const long long lo = slice_bound(P.seg_off[q], P.seg_len[q], b, nb);
    const long long hi = slice_bound(P.seg_off[q], P.seg_len[q], b + 1, nb);
    const long long kq = chunks_of(lo, hi, C);
    K = kq > K ? kq : K;
  }
  const unsigned long long tag0 = e << 20;
  if (warp < RS_WARPS) {
    // ---------------- reducer warps
    int m = 1;
    while ((m << 1) <= p) m <<= 1;
    const int excess = p - m;
    const long long so = P.seg_off[rank], sl = P.seg_len[rank];
    const long long lo = slice_bound(so, sl, b, nb), hi = slice_bound(so, sl, b + 1, nb);
    bool vec = true;
    for (int q = 0; q < p; ++q) vec = vec && al16(s_src[q]);
    char* red = s_red[rank];
    vec = vec && al16(out) && al16s(red, so, SZ);
    for (long long k = 0; k < K; ++k) {
      long long a, z;
      chunk_of(lo, hi, C, k, &a, &z);
      reduce_range<D, OP, MP, TREE>(s_seq, p, m, excess, a, z, vec, P.average, out, 0, red, so, tid, NR);
      __syncwarp();
      if (lane == 0) {
        fence_acq_rel_sys();
        for (int q = 0; q < p; ++q)
          if (q != rank) st_relaxed_sys(wmid_slot(P.heap[q], b, rank, warp), tag0 | (unsigned long long)(k + 1));
      }
    }
  } else {
    // ---------------- gather warps
    const int rt = tid - NR;
    __shared__ VecRange s_av[MAXP];
    for (long long k = 0; k < K; ++k) {
      const unsigned long long want = tag0 | (unsigned long long)(k + 1);
      if (rt < p * RS_WARPS) {
        const int q = rt / RS_WARPS, w = rt % RS_WARPS;
        if (q != rank && !wait_geq(wmid_slot(myheap, b, q, w), want, P.timeout_cycles))
          atomicExch(s_err, ERR_TRANSPORT);
      }
      named_sync(1, NR);
      if (*s_err) break;
      if (rt < p) {                                  // ranges + scalar head/tail of peer rt
        const int q = rt;
        VecRange v{nullptr, nullptr, 0};
        if (q != rank) {
          const long long qo = P.seg_off[q], ql = P.seg_len[q];
          long long a, z;
          chunk_of(slice_bound(qo, ql, b, nb), slice_bound(qo, ql, b + 1, nb), C, k, &a, &z);
          const S* src = reinterpret_cast<const S*>(s_red[q]) - qo;
          S* dst = reinterpret_cast<S*>(out);
          long long blo = z, bhi = z;
          if (((((uintptr_t)src) | ((uintptr_t)dst)) & 15u) == 0) {
            blo = ((a + W - 1) / W) * W;
            bhi = (z / W) * W;
            if (bhi < blo) blo = bhi = z;
          }
          for (long long i = a; i < blo; ++i) dst[i] = src[i];
          for (long long i = bhi; i < z; ++i) dst[i] = src[i];
          v.src = reinterpret_cast<const uint4*>(src + blo);
          v.dst = reinterpret_cast<uint4*>(dst + blo);
          v.nv = (bhi - blo) / W;
        }
        s_av[q] = v;
      }
      named_sync(1, NR);
      long long nvmax = 0;
      for (int q = 0; q < p; ++q) nvmax = s_av[q].nv > nvmax ? s_av[q].nv : nvmax;
      for (long long j = rt; j < nvmax; j += NR) {
        uint4 v[MP];
#pragma unroll
        for (int q = 0; q < MP; ++q)
          if (q < p && j < s_av[q].nv) v[q] = s_av[q].src[j];
#pragma unroll
        for (int q = 0; q < MP; ++q)
          if (q < p && j < s_av[q].nv) s_av[q].dst[j] = v[q];
      }
      named_sync(1, NR);                             // s_av reuse
    }
  }
}

// Allgather as a task queue: after its reduce-scatter slice, every CTA takes
// (slice s, peer q) tasks in order from a per-rank counter, waits for peer q's
// CTA s to have published its reduced slice, and pulls it. CTAs that finish
// their reduce early start pulling whatever is ready instead of waiting for
// the peers' CTA of their own index (no per-index RS->AG barrier skew).
template <class D, int MP>
__device__ void dynamic_allgather(const CollParams& P, int rank, int nb, unsigned long long e, char* myheap,
                                  Ctrl* ctrl, const char* const* s_src, char* const* s_red, char* out, bool multi,
                                  CopyRange* s_cr, VecRange* s_vr, int* s_ncr, int* s_err) {
  constexpr int SZ = sizeof(typename D::S);
  __shared__ long long s_task;
  const int tid = threadIdx.x, p = P.p, np1 = p - 1;
  const long long ntask = (long long)nb * np1;
  while (true) {
    if (tid == 0) s_task = (long long)atomicAdd(&ctrl->ag_next, 1ull);
    __syncthreads();
    const long long t = s_task;
    if (t >= ntask) break;
    const int s = (int)(t / np1);
    const int q = (rank + 1 + (int)(t % np1)) % p;
    if (tid == 0) {
      if (!wait_geq(mid_slot(myheap, s, q), e, P.timeout_cycles)) atomicExch(s_err, ERR_TRANSPORT);
      int r = 0;
      if (multi) {
        for (int k = 0; k < P.nbuf; ++k) {
          const long long so = P.bseg_off[k][q], sl = P.bseg_len[k][q];
          const long long lo = slice_bound(so, sl, s, nb), hi = slice_bound(so, sl, s + 1, nb);
          if (hi > lo) s_cr[r++] = CopyRange{s_src[q] + P.bboff[k] * SZ, out + P.bout_off[k] * SZ, 0, 0, lo, hi};
        }
      } else {
        const long long so = P.seg_off[q], sl = P.seg_len[q];
        const long long lo = slice_bound(so, sl, s, nb), hi = slice_bound(so, sl, s + 1, nb);
        if (hi > lo) s_cr[r++] = CopyRange{s_red[q], out, so, 0, lo, hi};
      }
      *s_ncr = r;
    }
    __syncthreads();
    if (*s_err) break;
    multi_copy<D, MP>(s_cr, *s_ncr, s_vr);
    __syncthreads();
  }
}

// MULTI: the multi-buffer / gathered-member aggregate launch (nbuf >= 1 or
// SRC_GATHER); otherwise every single-buffer mode. Separate instantiations keep
// each kernel's register footprint to its own mode.
template <class D, int OP, int MP, bool TREE, bool STREAM, bool MULTI>
__global__ void __launch_bounds__(THREADS, 1) collective_kernel(const __grid_constant__ CollParams P) {
  pdl_begin();
  using S = typename D::S;
  constexpr int SZ = sizeof(S);
  const int lr = P.virt ? blockIdx.y : 0;       // index into in/out
  const int rank = P.virt ? (int)blockIdx.y : P.rank;
  const int b = blockIdx.x, nb = gridDim.x, p = P.p, tid = threadIdx.x;
  char* myheap = P.heap[rank];
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(myheap + CTRL_OFF);

  __shared__ unsigned long long s_epoch;
  __shared__ const char* s_src[MAXP];   // element 0 of rank q's input
  __shared__ char* s_red[MAXP];         // element seg_off[q] of q's segment
  __shared__ const char* s_seq[MAXP];   // fold sequence
  __shared__ int s_rord[MAXP];          // fold sequence as source ranks
  __shared__ int s_err;
  __shared__ int s_skip;                // 2: inline agreement failed, the call moves no data

  if (gated_out(P, ctrl)) return;       // agreement failed earlier in this call
  CM_TRACE(P, lr, b, 0);
  if (!STREAM && P.bulk_rs)
    bulk_rs_setup(P.bulk_rs, P.bulk_stage, tid, (MULTI && P.ws) ? team_ws_rs().ncons : RS_CONSUMERS);
  if (tid == 0) {
    s_epoch = epoch_read(myheap, b) + 1;
    s_err = 0;
    s_skip = 0;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int par = (int)(e & 1);
  const long long stage_off = P.staging_off + (long long)par * P.staging_bytes;
  const char* in = P.in[lr];
  char* out = P.out[lr];
  const bool ag_only = !(P.phases & PH_RS);
  const bool two_shot = !P.oneshot;

  CM_CHECK(stage_off + P.staging_bytes <= P.heap_bytes, P.herr);
  CM_CHECK(MULTI || P.srcmode == SRC_ZEROCOPY || P.srcmode == SRC_REGISTERED || P.n * SZ <= P.staging_bytes, P.herr);
  // my own src/red offsets (published to peers)
  long long my_srcoff, my_redoff;
  const long long mso = P.seg_off[rank];
  if (P.srcmode == SRC_ZEROCOPY || P.srcmode == SRC_REGISTERED) {
    my_srcoff = P.zc_srcoff[lr];           // heap offset, or REG_FLAG | id | delta
    if (!ag_only)            // reduced segment goes to staging, vector-aligned like the source
      my_redoff = stage_off + (mso % SLICE_ALIGN) * SZ;
    else if (P.ag_in_rel)    // allgather: `in` holds only my segment
      my_redoff = my_srcoff;
    else
      my_redoff = my_srcoff + mso * SZ;
  } else {
    my_srcoff = stage_off;
    my_redoff = stage_off + mso * SZ;
  }

  // 1. copy-in: this CTA's slice of every segment peers will read from me
  __shared__ CopyRange s_cr[MAXBUF * MAXP + 1];
  __shared__ VecRange s_vr[MAXBUF * MAXP + 1];
  __shared__ int s_ncr;
  if (!MULTI && P.srcmode == SRC_COPYIN && !s_skip) {
    char* stage = myheap + stage_off;
    if (ag_only) {
      if (tid == 0) {
        const long long lo = slice_bound(mso, P.seg_len[rank], b, nb);
        const long long hi = slice_bound(mso, P.seg_len[rank], b + 1, nb);
        const long long ish = P.ag_in_rel ? mso : 0;
        s_cr[0] = CopyRange{in, stage, ish, 0, lo, hi};
        s_cr[1] = CopyRange{in, out, ish, 0, lo, hi};
        s_ncr = 2;
      }
    } else {
      const int nseg = P.oneshot ? 1 : p;
      if (tid < nseg) {
        const long long so = P.oneshot ? 0 : P.seg_off[tid];
        const long long sl = P.oneshot ? P.n : P.seg_len[tid];
        s_cr[tid] = CopyRange{in, stage, 0, 0, slice_bound(so, sl, b, nb), slice_bound(so, sl, b + 1, nb)};
      }
      if (tid == 0) s_ncr = nseg;
    }
    __syncthreads();
    multi_copy<D, MP>(s_cr, s_ncr, s_vr);
  }
  __syncthreads();
  CM_TRACE(P, lr, b, 1);

  // 2. publish my record to every peer (LL units, no release fence: only the
  // copy-in above wrote data peers are about to read, and a gpu-scope fence
  // puts it in my L2 first), then collect theirs
  const unsigned tag = ll_tag(e);
  if (tid < p && !s_skip) {
    if (P.srcmode == SRC_COPYIN) __threadfence();
    const long long rv[REC_UNITS] = {(long long)P.hdr, my_srcoff, my_redoff, P.akey[lr], P.acnt[lr], P.reg_seq};
    rec_put(rec_slot(P.heap[tid], par, b, rank), tag, rv, REC_UNITS);
  }
  if (tid < p && !s_skip) {
    long long rv[REC_UNITS];
    if (!rec_get(rec_slot(myheap, par, b, tid), tag, rv, REC_UNITS, P.timeout_cycles)) {
      atomicExch(&s_err, ERR_TRANSPORT);
    } else {
      __threadfence();                     // the peer's data is read after its record
      if (P.agree_inline && (rv[RF_AKEY] != P.akey[lr] || rv[RF_ACNT] != P.acnt[lr]))
        atomicExch(&s_skip, 2);            // ready sets differ: nobody moves data
      if ((unsigned long long)rv[RF_HDR] != P.hdr) atomicExch(&s_err, ERR_SHAPE);
      // peer's staging / symmetric pool, or its registered buffer mapped here
      s_src[tid] = resolve_src(P.heap, myheap, tid, rv[RF_SRCOFF], P.heap_bytes, P.herr);
      s_red[tid] = const_cast<char*>(resolve_src(P.heap, myheap, tid, rv[RF_REDOFF], P.heap_bytes, P.herr));
      if (b == 0) autoreg_report(P, myheap, rank, tid, rv[RF_REGSEQ]);
    }
  }
  __syncthreads();                       // s_src / s_red / s_err complete
  if (P.agree_inline && s_err != ERR_TRANSPORT) {
    // every rank compared every peer: a disagreement is seen by all ranks, so
    // all skip; the plans (and headers) of disagreeing ranks may differ, which
    // is then not an error
    const bool agreed = s_skip != 2;
    __syncthreads();
    if (tid == 0 && !agreed) s_err = 0;
    if (tid == 0 && b == 0 && P.agree_out) {
      volatile unsigned long long* ao = P.agree_out + 2 * lr;
      ao[1] = agreed ? 1ull : 0ull;
      __threadfence_system();
      ao[0] = P.agree_ticket;
    }
    __syncthreads();
  }
  // fold sequence of my segment's sources (reference order)
  if (tid == 0 && (P.phases & PH_RS)) {
    int m = 1;
    while ((m << 1) <= p) m <<= 1;
    const int excess = p - m;
    if (P.order == ORD_RING) {            // chunk c folds x_{c-1}, x_{c-2}, ..., x_c
      for (int k = 0; k < p; ++k) s_rord[k] = ((rank - 1 - k) % p + p) % p;
    } else if (P.order == ORD_TREE) {     // leaves real(v), partners 2v+1 at M+v
      for (int v = 0; v < m; ++v) s_rord[v] = v < excess ? 2 * v : v + excess;
      for (int v = 0; v < excess; ++v) s_rord[m + v] = 2 * v + 1;
    } else {
      for (int k = 0; k < p; ++k) s_rord[k] = k;
    }
    for (int k = 0; k < p; ++k) s_seq[k] = s_src[s_rord[k]];
  }
  __syncthreads();
  CM_TRACE(P, lr, b, 2);
  if (s_err || s_skip) goto finish;

  if constexpr (STREAM) {
    // Pipelined two-shot: warps 0..7 reduce chunk after chunk of my segment
    // slice and publish per-warp progress to every peer; warps 8..15 pull
    // chunk k of every other segment as soon as all peers' reducer warps have
    // published it. Reduce-scatter of chunk k+1 overlaps allgather of chunk k,
    // so there is no CTA-wide mid barrier and no idle link between phases.
    stream_body<D, OP, MP, TREE>(P, rank, b, nb, e, s_src, s_red, s_seq, &s_err, out, myheap);
    goto finish;
  }

  if constexpr (MULTI) {
    // ---- several fused buffers, one launch: RS of every buffer, then AG of
    // every buffer. Input prestaged in staging, or (SRC_GATHER) read in place
    // from every rank's registered member tensors. The CTA walks its slice of
    // every buffer as a sequence of pieces (a piece never crosses a member of
    // a gathered buffer); thread 0 prepares each piece's source table in
    // shared memory, so ONE reduce call site serves both input modes and no
    // per-piece state lives in registers.
    //
    // overlap: CTAs [0, nrs) reduce-scatter slice b and push their progress
    // after every chunk; CTAs [nrs, 2 nrs) allgather slice b - nrs of every
    // peer chunk by chunk as soon as that peer has reduced it. Otherwise every
    // CTA reduces its slice, then one RS->AG barrier per CTA index, then AG.
    __shared__ const char* s_seqk[MAXP];
    __shared__ char* s_bo;
    __shared__ char* s_rd;
    __shared__ long long s_i, s_pe, s_hi, s_pos;
    __shared__ int s_k, s_vec;
    __shared__ Prog s_prog;
    int m = 1;
    while ((m << 1) <= p) m <<= 1;
    const int excess = p - m;
    char* mystage = myheap + stage_off;
    const bool ovl = P.overlap != 0;
    // warp-specialised two-shot: warps 0..8 reduce-scatter (8 consumer warps
    // + the bulk-engine producer) and push per-chunk progress; warps 9..15 of
    // the same CTA allgather each peer's chunks as soon as they are reduced
    const bool ws = P.ws != 0 && !ovl;
    const Team T = ws ? team_ws_rs() : team_all();
    const int nrs = ovl ? P.nrs : nb;
    if (ovl && b >= nrs) {
      // ---- allgather role: slice j of every peer's segment, chunk by chunk
      const int j = b - nrs;
      // elements per allgather block: the reduce chunk times the report interval
      const long long G = (long long)((P.bulk_stage / p) & ~15) / SZ * P.ovl_chunks;
      __shared__ long long s_tot[MAXP];
      if (tid < p) {
        long long t = 0;
        for (int k = 0; k < P.nbuf; ++k) {
          const long long so = P.bseg_off[k][tid], sl = P.bseg_len[k][tid];
          t += slice_bound(so, sl, j + 1, nrs) - slice_bound(so, sl, j, nrs);
        }
        s_tot[tid] = tid == rank ? 0 : t;
      }
      __syncthreads();
      long long tmax = 0;
      for (int q = 0; q < p; ++q) tmax = s_tot[q] > tmax ? s_tot[q] : tmax;
      const unsigned long long ptag = e << 32;
#pragma unroll 1
      for (long long pos = 0; pos < tmax; pos += G) {
        if (tid < p && pos < s_tot[tid]) {
          const long long need = pos + G < s_tot[tid] ? pos + G : s_tot[tid];
          const unsigned long long* f =
              reinterpret_cast<const unsigned long long*>(myheap + PROG_OFF + ((size_t)j * MAXP + tid) * 8);
          if (!flag_wait(f, ptag | (unsigned long long)need, P.timeout_cycles)) atomicExch(&s_err, ERR_TRANSPORT);
        }
        __syncthreads();
        if (s_err) break;
        if (tid == 0) {                               // [pos, pos + G) of each peer's slice sequence
          int r = 0;
          for (int q = 0; q < p; ++q) {
            if (pos >= s_tot[q]) continue;
            const long long end = pos + G < s_tot[q] ? pos + G : s_tot[q];
            long long base = 0;
            for (int k = 0; k < P.nbuf && base < end; ++k) {
              const long long so = P.bseg_off[k][q], sl = P.bseg_len[k][q];
              const long long lo = slice_bound(so, sl, j, nrs), hi = slice_bound(so, sl, j + 1, nrs);
              const long long a = pos > base ? pos : base, z = end < base + hi - lo ? end : base + hi - lo;
              if (z > a) {
                CM_CHECK(lo + (z - base) <= hi && (P.bboff[k] + hi) * SZ <= P.staging_bytes, P.herr);
                s_cr[r++] = CopyRange{P.heap[q] + stage_off + P.bboff[k] * SZ, out + P.bout_off[k] * SZ, 0, 0,
                                      lo + (a - base), lo + (z - base)};
              }
              base += hi - lo;
            }
          }
          s_ncr = r;
        }
        __syncthreads();
        multi_copy<D, MP>(s_cr, s_ncr, s_vr);
        __syncthreads();
      }
      goto finish;
    }
    if (ws && tid >= T.grp) {
      // ---- allgather team: slice b of every peer's segment, block by block
      const int at = tid - WS_AG_T0;
      const long long G = (long long)((P.bulk_stage / p) & ~15) / SZ * P.ovl_chunks;
      __shared__ long long s_tot2[MAXP];
      __shared__ CopyRange s_cr2[MAXBUF * MAXP + 1];
      __shared__ VecRange s_vr2[MAXBUF * MAXP + 1];
      __shared__ int s_ncr2;
      if (at < p) {
        long long t = 0;
        for (int k = 0; k < P.nbuf; ++k) {
          const long long so = P.bseg_off[k][at], sl = P.bseg_len[k][at];
          t += slice_bound(so, sl, b + 1, nb) - slice_bound(so, sl, b, nb);
        }
        s_tot2[at] = at == rank ? 0 : t;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(WS_AG_BAR), "r"(WS_AG_N) : "memory");
      long long tmax = 0;
      for (int q = 0; q < p; ++q) tmax = s_tot2[q] > tmax ? s_tot2[q] : tmax;
      const unsigned long long ptag = e << 32;
#pragma unroll 1
      for (long long pos = 0; pos < tmax; pos += G) {
        if (at < p && pos < s_tot2[at]) {
          const long long need = pos + G < s_tot2[at] ? pos + G : s_tot2[at];
          const unsigned long long* f =
              reinterpret_cast<const unsigned long long*>(myheap + PROG_OFF + ((size_t)b * MAXP + at) * 8);
          if (!flag_wait(f, ptag | (unsigned long long)need, P.timeout_cycles)) atomicExch(&s_err, ERR_TRANSPORT);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(WS_AG_BAR), "r"(WS_AG_N) : "memory");
        if (s_err) break;
        if (at == 0) {
          int r = 0;
          for (int q = 0; q < p; ++q) {
            if (pos >= s_tot2[q]) continue;
            const long long end = pos + G < s_tot2[q] ? pos + G : s_tot2[q];
            long long base = 0;
            for (int k = 0; k < P.nbuf && base < end; ++k) {
              const long long so = P.bseg_off[k][q], sl = P.bseg_len[k][q];
              const long long lo = slice_bound(so, sl, b, nb), hi = slice_bound(so, sl, b + 1, nb);
              const long long a = pos > base ? pos : base, z = end < base + hi - lo ? end : base + hi - lo;
              if (z > a)
                s_cr2[r++] = CopyRange{P.heap[q] + stage_off + P.bboff[k] * SZ, out + P.bout_off[k] * SZ, 0, 0,
                                       lo + (a - base), lo + (z - base)};
              base += hi - lo;
            }
          }
          s_ncr2 = r;
        }
        asm volatile("bar.sync %0, %1;" ::"r"(WS_AG_BAR), "r"(WS_AG_N) : "memory");
        multi_copy<D, MP>(s_cr2, s_ncr2, s_vr2, WS_AG_T0, WS_AG_N, WS_AG_BAR);
        asm volatile("bar.sync %0, %1;" ::"r"(WS_AG_BAR), "r"(WS_AG_N) : "memory");
      }
      goto finish;
    }
    // piece iterator, advanced by thread 0 only (the loop state lives in
    // shared memory, not in every thread's registers)
    if (tid == 0) {
      s_k = -1;
      s_i = s_hi = 0;
      s_pos = 0;
      s_prog.tag = e << 32;
      s_prog.p = p;
      s_prog.every = P.ovl_chunks;
      for (int q = 0; q < p; ++q)
        s_prog.dst[q] = ((ovl || ws) && q != rank)
                            ? reinterpret_cast<unsigned long long*>(P.heap[q] + PROG_OFF + ((size_t)b * MAXP + rank) * 8)
                            : nullptr;
    }
#pragma unroll 1
    while (true) {
      if (tid == 0) {
        while (s_i >= s_hi && ++s_k < P.nbuf) {        // next buffer with a non-empty slice
          const long long so = P.bseg_off[s_k][rank], sl = P.bseg_len[s_k][rank];
          s_i = slice_bound(so, sl, b, nrs);
          s_hi = slice_bound(so, sl, b + 1, nrs);
        }
        if (s_k < P.nbuf) {
          const int k = s_k;
          const long long i = s_i, hi = s_hi;
          char* bo = out + P.bout_off[k] * SZ;
          char* red = mystage + P.bboff[k] * SZ;       // element 0 of buffer k (AG source)
          long long pe = hi;
          if (P.srcmode == SRC_GATHER) {               // member holding global index bboff + i
            const long long* gstart = P.gtab;
            const long long* gid = P.gtab + P.gmem + 1;
            const long long g = P.bboff[k] + i;
            int a = 0, z = P.gmem;                     // gstart[a] <= g < gstart[z]
            while (z - a > 1) {
              const int mid = (a + z) >> 1;
              if (gstart[mid] <= g) a = mid; else z = mid;
            }
            const long long mend = gstart[a + 1] - P.bboff[k];
            pe = mend < hi ? mend : hi;
            for (int q = 0; q < p; ++q) {
              const char* base = *reinterpret_cast<char* const*>(
                  myheap + REG_OFF + ((size_t)gid[a] * MAXP + s_rord[q]) * 8);
              s_seqk[q] = base - (gstart[a] - P.bboff[k]) * SZ;   // element i of buffer k
            }
          } else {
            for (int q = 0; q < p; ++q) s_seqk[q] = s_seq[q] + P.bboff[k] * SZ;
          }
          bool vec = al16(bo) && al16(red);
          for (int q = 0; q < p; ++q) vec = vec && al16(s_seqk[q]);
          s_bo = bo;
          s_rd = red;
          s_pe = pe;
          s_vec = vec ? 1 : 0;
          s_prog.base = s_pos;
        }
      }
      team_sync(T);
      if (s_k >= P.nbuf) break;
      CM_CHECK(s_i <= s_pe && s_pe <= s_hi && s_hi <= P.bseg_off[s_k][rank] + P.bseg_len[s_k][rank] &&
                   (P.bboff[s_k] + s_pe) * SZ <= P.staging_bytes && s_pe <= P.bn[s_k],
               P.herr);
      if (P.bulk_rs && s_vec) {
        reduce_range_bulk<D, OP, MP, TREE>(P.bulk_rs, P.bulk_stage, s_seqk, p, m, excess, s_i, s_pe, P.average,
                                           s_bo, 0, s_rd, 0, tid, (ovl || ws) ? &s_prog : nullptr, T);
      } else {
        reduce_range<D, OP, MP, TREE>(s_seqk, p, m, excess, s_i, s_pe, s_vec != 0, P.average, s_bo, 0, s_rd, 0,
                                      tid, T.grp);
        if (ovl || ws) {
          team_sync(T);
          if (tid == 0) prog_publish(&s_prog, s_pos + (s_pe - s_i));
        }
      }
      team_sync(T);
      if (tid == 0) {
        s_pos += s_pe - s_i;
        s_i = s_pe;
      }
    }
    CM_TRACE(P, lr, b, 3);
    if (ovl || ws) goto finish;
    if (tid < p) flag_put(mid_slot(P.heap[tid], b, rank), e);
    if (P.dyn_ag) {
      dynamic_allgather<D, MP>(P, rank, nb, e, myheap, ctrl, s_src, s_red, out, true, s_cr, s_vr, &s_ncr, &s_err);
      goto finish;
    }
    if (tid < p && !flag_wait(mid_slot(myheap, b, tid), e, P.timeout_cycles)) atomicExch(&s_err, ERR_TRANSPORT);
    __syncthreads();
    CM_TRACE(P, lr, b, 4);
    if (s_err) goto finish;
    if (tid == 0) {
      int r = 0;
      for (int k = 0; k < P.nbuf; ++k)
        for (int q = 0; q < p; ++q) {
          if (q == rank) continue;
          const long long so = P.bseg_off[k][q], sl = P.bseg_len[k][q];
          const long long lo = slice_bound(so, sl, b, nb), hi = slice_bound(so, sl, b + 1, nb);
          if (hi <= lo) continue;
          s_cr[r++] = CopyRange{s_src[q] + P.bboff[k] * SZ, out + P.bout_off[k] * SZ, 0, 0, lo, hi};
        }
      s_ncr = r;
    }
    __syncthreads();
    multi_copy<D, MP>(s_cr, s_ncr, s_vr);
    goto finish;
  }

  if constexpr (!MULTI) {
  // 3. reduce my segment (RS) — or the whole vector (one-shot)
  if (P.phases & PH_RS) {
    const long long so = P.oneshot ? 0 : mso;
    const long long sl = P.oneshot ? P.n : P.seg_len[rank];
    int m = 1;
    while ((m << 1) <= p) m <<= 1;
    const int excess = p - m;
    bool vec = true;
    for (int q = 0; q < p; ++q) vec = vec && al16(s_src[q]);
    const long long out_shift = P.out_rel ? so : 0;
    vec = vec && al16s(out, out_shift, SZ);
    char* red = nullptr;
    long long red_shift = 0;
    if (two_shot && (P.phases & PH_AG)) {
      red = s_red[rank];
      red_shift = so;
      vec = vec && al16s(red, red_shift, SZ);
    }
    const long long lo = slice_bound(so, sl, b, nb), hi = slice_bound(so, sl, b + 1, nb);
    if (P.bulk_rs && vec)
      reduce_range_bulk<D, OP, MP, TREE>(P.bulk_rs, P.bulk_stage, s_seq, p, m, excess, lo, hi, P.average, out, out_shift, red,
                                         red_shift, tid);
    else
      reduce_range<D, OP, MP, TREE>(s_seq, p, m, excess, lo, hi, vec, P.average, out, out_shift,
                                    red, red_shift, tid, blockDim.x);
  }

  // 4. RS -> AG barrier (per CTA index) and 5. allgather
  CM_TRACE(P, lr, b, 3);
  if (P.phases & PH_AG) {
    if (!ag_only) {
      __syncthreads();
      if (tid < p) flag_put(mid_slot(P.heap[tid], b, rank), e);
      if (P.dyn_ag) {
        dynamic_allgather<D, MP>(P, rank, nb, e, myheap, ctrl, s_src, s_red, out, false, s_cr, s_vr, &s_ncr,
                                 &s_err);
        goto finish;
      }
      if (tid < p && !flag_wait(mid_slot(myheap, b, tid), e, P.timeout_cycles))
        atomicExch(&s_err, ERR_TRANSPORT);
      __syncthreads();
      CM_TRACE(P, lr, b, 4);
      if (s_err) goto finish;
    }
    // pull slice b of every other segment from all peers concurrently
    if (tid == 0) {
      int k = 0;
      for (int q = 0; q < p; ++q) {
        // (allgather with my segment read in place: copy my own part too)
        if (q == rank && !(ag_only && (P.srcmode == SRC_ZEROCOPY || P.srcmode == SRC_REGISTERED))) continue;
        const long long so = P.seg_off[q], sl = P.seg_len[q];
        const long long lo = slice_bound(so, sl, b, nb), hi = slice_bound(so, sl, b + 1, nb);
        if (hi <= lo) continue;
        s_cr[k++] = CopyRange{s_red[q], out, so, 0, lo, hi};
      }
      s_ncr = k;
    }
    __syncthreads();
    multi_copy<D, MP>(s_cr, s_ncr, s_vr);
  }

  }

finish:
  __syncthreads();
  CM_TRACE(P, lr, b, 5);
  if (tid == 0) {
    if (s_err) *reinterpret_cast<volatile unsigned*>(P.herr) = (unsigned)s_err;
    // outcome for the gated launches queued behind (every CTA compared the
    // same records, so CTA 0's verdict is the grid's)
    if (P.agree_inline && b == 0) {
      ctrl->agree_ok = s_skip == 2 ? 0 : 1;
      ctrl->agree_tag = P.agree_ticket;
    }
    if (P.dyn_ag) {                       // the allgather task counter is reset by the last CTA
      __threadfence();
      const unsigned old = atomicAdd(&ctrl->done, 1u);
      if (old == (unsigned)nb - 1) {
        ctrl->done = 0;
        ctrl->ag_next = 0;
      }
    }
  }
  epoch_publish(myheap, b, nb, e);
  CM_TRACE(P, lr, b, 6);
}

}  // namespace dev
}  // namespace cm
