// sm_100a device code for the CUDA-aware allreduce: heap layout, parameters,
// element types, memory-model helpers, vector I/O, reference-order folds,
// SM and bulk-engine reduce loops and the concurrent range copy shared by the
// kernels (kernel_*.cuh). Overview of the kernel family:
//
// One kernel family (`collective_kernel`) implements every collective of the
// reference allreduce suite over a CUDA-IPC peer-mapped symmetric heap:
//
//   one-shot  : every rank reduces the whole vector from all p peers' staged
//               copies (small messages; RHD tree order or flat order)
//   two-shot  : reduce-scatter (rank r reduces its layout segment from all p
//               peers, in the reference fold order) -> per-CTA flag barrier ->
//               allgather (rank r pulls every other segment). This is the ring
//               RSA (collectives.py:107-152) / RHD RSA (:155-236) data movement
//               collapsed onto NVSwitch's full crossbar: the same 2(p-1)/p*S
//               bytes per GPU per direction, two sync points instead of 2(p-1),
//               and the per-element fold order of the reference replayed
//               exactly so results are bit-identical.
//   RS-only / AG-only : the public reduce_scatter / allgather.
//
// Synchronisation is flag based over NVLink: CTA b of rank r publishes a
// record {epoch, header, src offset, reduced offset} into slot [parity][b][r]
// of every peer's heap with st.release.sys, and waits on its own heap with
// ld.acquire.sys. The epoch lives in device memory and is advanced by the last
// CTA of each launch, so launches can be captured into CUDA graphs. Staging is
// double-buffered by epoch parity: a rank rewrites staging[e&1] only in call
// e+2, after every peer has entered call e+1 (and therefore left call e).
// Waits are bounded (timeout -> CM_ERR_TRANSPORT in the host-mapped error word).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cm.h"

namespace cm {
namespace dev {

constexpr int MAXP = CM_MAX_RANKS;
constexpr int MAXBLK = 1024;
constexpr int THREADS = 512;
constexpr int SLICE_ALIGN = 64;  // elements; slice boundaries are multiples of this
constexpr int MAXBUF = 4;        // fused buffers per multi-buffer launch

// ---- heap layout (identical on every rank) ---------------------------------
constexpr size_t CTRL_OFF = 0;
constexpr size_t REC_OFF = 4096;
constexpr size_t REC_BYTES = 64;
constexpr size_t REC_SIZE = 2ull * MAXBLK * MAXP * REC_BYTES;
constexpr size_t MID_OFF = REC_OFF + REC_SIZE;
constexpr size_t MID_SIZE = (size_t)MAXBLK * MAXP * 8;
// LL (low-latency) slots: every 16-byte unit carries 8 payload bytes and two
// copies of the epoch flag, so data and "ready" arrive in one store. Layout
// [parity][phase][src < p][unit < ll_units] starting at LL_OFF; its size
// depends on p and is chosen at communicator creation, so staging starts at a
// runtime offset (CollParams::staging_off).
constexpr size_t WMID_OFF = MID_OFF + MID_SIZE;         // per-warp progress of the pipelined two-shot
constexpr size_t WMID_SIZE = (size_t)MAXBLK * MAXP * 8 * 8;
constexpr size_t LLH_OFF = WMID_OFF + WMID_SIZE;        // per-CTA LL header units
constexpr size_t LLH_SIZE = 2ull * MAXBLK * MAXP * 16;
// registered-buffer table: REGTAB[id][q] = rank q's registered buffer start,
// mapped in THIS process (cm_comm_register, the IPC side of the pointer cache)
constexpr int MAXREG = 4096;
constexpr size_t REG_OFF = LLH_OFF + LLH_SIZE;
constexpr size_t REG_SIZE = (size_t)MAXREG * MAXP * 8;
// pairwise phase flags of the log-p recursive halving/doubling kernel:
// RFLAG[src][cta] = {(epoch << 8) | phase, call header}, pushed by src
constexpr size_t RHDF_OFF = REG_OFF + REG_SIZE;
constexpr size_t RHDF_SIZE = (size_t)MAXP * MAXBLK * 16;
constexpr size_t HEAP_ALIGN = 2ull << 20;
constexpr size_t LL_OFF = ((RHDF_OFF + RHDF_SIZE + HEAP_ALIGN - 1) / HEAP_ALIGN) * HEAP_ALIGN;
// record source encoding for registered inputs: bit 62 | id << 40 | byte delta
constexpr unsigned long long REG_FLAG = 1ull << 62;
constexpr size_t CTRL_REGION = LL_OFF;                  // zeroed at creation

struct Ctrl {
  unsigned long long epoch;      // calls completed by this rank
  unsigned int done;             // CTAs finished in the current call
  unsigned int pad;
  unsigned long long agree_tag;  // ticket of the last agreement check (cm_agree)
  long long agree_ok;            // its outcome: every rank held the same values
  unsigned long long ag_next;    // next allgather task of the current call (dynamic allgather)
};

struct Rec {
  unsigned long long epoch;
  unsigned long long hdr;
  long long srcoff;  // element i of the sender's input at heap + srcoff + i*sz
  long long redoff;  // element i of the sender's segment at heap + redoff + (i-seg_off)*sz
  long long akey;    // inline agreement (aggregate's ready-set hash and count)
  long long acnt;
  long long pad[2];
};

enum SrcMode { SRC_COPYIN = 0, SRC_PRESTAGED = 1, SRC_ZEROCOPY = 2, SRC_INLINE = 3, SRC_REGISTERED = 4,
               SRC_GATHER = 5 };
enum Order { ORD_SEQ = 0, ORD_RING = 1, ORD_TREE = 2 };
enum Phase { PH_RS = 1, PH_AG = 2 };
enum Err { ERR_SHAPE = 1, ERR_TRANSPORT = 4 };

struct CollParams {
  char* heap[MAXP];          // every rank's heap, mapped in this process
  const char* in[MAXP];      // per local rank (real mode: [0])
  char* out[MAXP];
  long long seg_off[MAXP];   // layout segment per rank (elements)
  long long seg_len[MAXP];
  long long n;               // full vector length (elements)
  long long zc_srcoff[MAXP]; // ZEROCOPY: byte offset of `in` within own heap (per local rank)
  unsigned long long hdr;    // call signature checked against every peer
  unsigned long long timeout_cycles;
  long long staging_bytes;   // per parity half
  unsigned int* herr;        // host-mapped error word
  int p;
  int rank;                  // real mode
  int virt;                  // 1: blockIdx.y is the rank (single-GPU emulation)
  int srcmode;
  int order;                 // Order
  int phases;                // Phase bits
  int oneshot;               // every segment is [0, n)
  int out_rel;               // RS writes out[i - seg_off] (reduce_scatter API)
  int ag_in_rel;             // AG-only: `in` holds only my segment (in[i - seg_off])
  int average;               // divide the reduced value by p (aggregate mean)
  long long staging_off;     // heap offset of staging[0]
  long long stream_chunk;    // elements per chunk of the pipelined two-shot
  long long ll_units;        // LL units per (parity, phase, source)
  unsigned long long* trace; // optional: per-CTA phase timestamps (globaltimer ns)
  int trace_ctas;
  // several fused buffers in ONE launch (aggregate): buffer k holds bn[k]
  // elements at staging element offset bboff[k] and is written to bout[k];
  // each keeps its own reduce-scatter layout (so ring chunking, and therefore
  // the fold order, is exactly that of one allreduce per buffer)
  int nbuf;
  long long bn[MAXBUF];
  long long bboff[MAXBUF];
  char* bout[MAXBUF];
  long long bseg_off[MAXBUF][MAXP];
  long long bseg_len[MAXBUF][MAXP];
  // SRC_GATHER (aggregate on registered gradients): the fused buffers are the
  // concatenation of registered member tensors; gtab = {gstart[0..gmem],
  // id[0..gmem)} in device memory; peers' members are read in place through
  // REGTAB[id][q] (no pack, no staging copy)
  const long long* gtab;
  int gmem;
  long long inl[8];          // SRC_INLINE: the input travels in the parameters (cm_agree)
  unsigned long long* done_flag;  // optional: written with done_value when the call completes
  unsigned long long done_value;
  int bulk_rs;               // >0: reduce through the bulk-copy engine with this many smem stages
  int bulk_local;            // the reduce's own-rank source is loaded directly, not staged
  int bulk_stage;            // bytes per shared-memory stage of the bulk reduce
  // >0: run only if the agreement check with this ticket (queued before on the
  // same stream) succeeded; otherwise every rank skips the call identically
  unsigned long long agree_gate;
  // inline agreement: every rank publishes {akey, acnt} in its records; if any
  // peer's differ, every rank skips the call identically and CTA 0 reports
  // it through agree_out = {ok, ticket} (host-mapped)
  int agree_inline;
  long long akey, acnt;
  unsigned long long* agree_out;
  unsigned long long agree_ticket;
  int dyn_ag;                // allgather as a queue of (slice, peer) tasks shared by the CTAs
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// phase stamp k (0 start, 1 copied-in, 2 start barrier, 3 reduced, 4 mid barrier, 5 end)
#define CM_TRACE(P, lr, b, k)                                                   \
  do {                                                                          \
    if ((P).trace && threadIdx.x == 0 && (b) < (P).trace_ctas)                  \
      (P).trace[((size_t)(lr) * (P).trace_ctas + (b)) * 8 + (k)] = gtimer();    \
  } while (0)

// ---- element types ----------------------------------------------------------
struct F32 { using S = float;    using A = float; };
struct F64 { using S = double;   using A = double; };
struct BF16 { using S = uint16_t; using A = float; };
struct I32 { using S = int32_t;  using A = int32_t; };
struct I64 { using S = int64_t;  using A = int64_t; };

__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float(((unsigned)h) << 16);
}
// round-to-nearest-even, NaN -> 0x7FC0 (matches oracle/collectives.f32_to_bf16)
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  const unsigned u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7FC0;
  return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

template <class D> __device__ __forceinline__ typename D::A to_acc(typename D::S s) { return s; }
template <> __device__ __forceinline__ float to_acc<BF16>(uint16_t s) { return bf16_to_f32(s); }
template <class D> __device__ __forceinline__ typename D::S from_acc(typename D::A a) { return a; }
template <> __device__ __forceinline__ uint16_t from_acc<BF16>(float a) { return f32_to_bf16(a); }

// _reduce_arrays (collectives.py:57-64): `a` is the accumulator (first operand).
// MAX is numpy.maximum bit for bit: (a > b || isnan(a)) ? a : b.
template <int OP, typename A> __device__ __forceinline__ A op2(A a, A b);
template <> __device__ __forceinline__ float op2<CM_SUM, float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double op2<CM_SUM, double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ int32_t op2<CM_SUM, int32_t>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}
template <> __device__ __forceinline__ int64_t op2<CM_SUM, int64_t>(int64_t a, int64_t b) {
  return (int64_t)((uint64_t)a + (uint64_t)b);
}
template <> __device__ __forceinline__ float op2<CM_MAX, float>(float a, float b) { return (a > b || a != a) ? a : b; }
template <> __device__ __forceinline__ double op2<CM_MAX, double>(double a, double b) { return (a > b || a != a) ? a : b; }
template <> __device__ __forceinline__ int32_t op2<CM_MAX, int32_t>(int32_t a, int32_t b) { return a > b ? a : b; }
template <> __device__ __forceinline__ int64_t op2<CM_MAX, int64_t>(int64_t a, int64_t b) { return a > b ? a : b; }

// IEEE division by p (aggregation.py:167-172: float32(float64(s)/p) == s/(float)p)
template <typename A> __device__ __forceinline__ A div_p(A a, int p);
template <> __device__ __forceinline__ float div_p<float>(float a, int p) { return __fdiv_rn(a, (float)p); }
template <> __device__ __forceinline__ double div_p<double>(double a, int p) { return __ddiv_rn(a, (double)p); }
template <> __device__ __forceinline__ int32_t div_p<int32_t>(int32_t a, int) { return a; }
template <> __device__ __forceinline__ int64_t div_p<int64_t>(int64_t a, int) { return a; }

// ---- memory-model helpers -----------------------------------------------------
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_s64(long long* p, long long v) {
  asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_relaxed_sys_s64(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ Rec* rec_slot(char* heap, int par, int blk, int src) {
  return reinterpret_cast<Rec*>(heap + REC_OFF +
                                ((size_t)(par * MAXBLK + blk) * MAXP + src) * REC_BYTES);
}
__device__ __forceinline__ unsigned long long* mid_slot(char* heap, int blk, int src) {
  return reinterpret_cast<unsigned long long*>(heap + MID_OFF + ((size_t)blk * MAXP + src) * 8);
}

// bounded spin: returns false on timeout
__device__ __forceinline__ bool wait_geq(const unsigned long long* f, unsigned long long e,
                                         unsigned long long timeout) {
  if (ld_acquire_sys(f) >= e) return true;
  const long long t0 = clock64();
  while (true) {
    for (int i = 0; i < 64; ++i)
      if (ld_acquire_sys(f) >= e) return true;
    if ((unsigned long long)(clock64() - t0) > timeout) return false;
  }
}

// Slice b of segment [off, off+len) split over nb CTAs; interior boundaries
// are multiples of SLICE_ALIGN (absolute element index) so they are vector
// aligned and independent of the vector width.
__device__ __forceinline__ long long slice_bound(long long off, long long len, int k, int nb) {
  if (k <= 0) return off;
  if (k >= nb) return off + len;
  long long x = off + (long long)(((__int128)len * k) / nb);
  x = (x / SLICE_ALIGN) * SLICE_ALIGN;
  if (x < off) x = off;
  if (x > off + len) x = off + len;
  return x;
}

// ---- vector load/store of W elements (16 B when W*sizeof(S)==16) ---------------
template <class D, int W>
__device__ __forceinline__ void load_vec(const char* base, long long i, typename D::A (&v)[W]) {
  using S = typename D::S;
  const S* p = reinterpret_cast<const S*>(base) + i;
  if constexpr (W * sizeof(S) == 16) {
    uint4 raw = *reinterpret_cast<const uint4*>(p);
    const S* s = reinterpret_cast<const S*>(&raw);
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = to_acc<D>(s[w]);
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = to_acc<D>(p[w]);
  }
}

template <class D, int W>
__device__ __forceinline__ void store_vec(char* base, long long i, const typename D::A (&v)[W]) {
  using S = typename D::S;
  S* p = reinterpret_cast<S*>(base) + i;
  if constexpr (W * sizeof(S) == 16) {
    uint4 raw;
    S* s = reinterpret_cast<S*>(&raw);
#pragma unroll
    for (int w = 0; w < W; ++w) s[w] = from_acc<D>(v[w]);
    *reinterpret_cast<uint4*>(p) = raw;
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) p[w] = from_acc<D>(v[w]);
  }
}

// ---- fold of p loaded operands in the reference order -------------------------
// u[k] was loaded from seq[k]. LEFT: ((u0 op u1) op u2) ... (ring & flat).
// TREE (collectives.py:178-229): leaves L_v = u[v] op u[M+v] for v < excess,
// else u[v]; then a balanced tree, lower subtree first.
template <int OP, int MP, int W, int M, typename A>
__device__ __forceinline__ void tree_fold(A (&u)[MP][W], int excess) {
#pragma unroll
  for (int v = 0; v < M; ++v) {
    constexpr int dummy = 0;
    (void)dummy;
    const int hi = (M + v < MP) ? M + v : MP - 1;
    if (v < excess) {
#pragma unroll
      for (int w = 0; w < W; ++w) u[v][w] = op2<OP>(u[v][w], u[hi][w]);
    }
  }
#pragma unroll
  for (int s = 1; s < M; s *= 2) {
#pragma unroll
    for (int v = 0; v + s < M; v += 2 * s) {
#pragma unroll
      for (int w = 0; w < W; ++w) u[v][w] = op2<OP>(u[v][w], u[v + s][w]);
    }
  }
}

template <int OP, int MP, int W, bool TREE, typename A>
__device__ __forceinline__ void fold(A (&u)[MP][W], int p, int m, int excess) {
  if constexpr (!TREE) {
#pragma unroll
    for (int k = 1; k < MP; ++k)
      if (k < p) {
#pragma unroll
        for (int w = 0; w < W; ++w) u[0][w] = op2<OP>(u[0][w], u[k][w]);
      }
  } else {
    switch (m) {
      case 1: tree_fold<OP, MP, W, 1>(u, excess); break;
      case 2: tree_fold<OP, MP, W, 2>(u, excess); break;
      case 4: tree_fold<OP, MP, W, (4 <= MP ? 4 : 1)>(u, excess); break;
      case 8: tree_fold<OP, MP, W, (8 <= MP ? 8 : 1)>(u, excess); break;
      default: tree_fold<OP, MP, W, (16 <= MP ? 16 : 1)>(u, excess); break;
    }
  }
}

// reduce U groups of W elements starting at element indices i0 + g*stride
template <class D, int OP, int MP, int W, bool TREE>
__device__ __forceinline__ void reduce_one(const char* const* seq, int p, int m, int excess,
                                           long long i, int average, char* out,
                                           long long out_shift, char* red, long long red_shift) {
  using A = typename D::A;
  A u[MP][W];
#pragma unroll
  for (int k = 0; k < MP; ++k)
    if (k < p) load_vec<D, W>(seq[k], i, u[k]);
  fold<OP, MP, W, TREE>(u, p, m, excess);
  if (average) {
#pragma unroll
    for (int w = 0; w < W; ++w) u[0][w] = div_p<A>(u[0][w], p);
  }
  store_vec<D, W>(out, i - out_shift, u[0]);
  if (red) store_vec<D, W>(red, i - red_shift, u[0]);
}

// Process [lo, hi) of one segment: scalar head/tail, W-wide body with 2-way
// unrolling for memory-level parallelism over NVLink.
template <class D, int OP, int MP, bool TREE>
__device__ void reduce_range(const char* const* seq, int p, int m, int excess, long long lo,
                             long long hi, bool vec, int average, char* out, long long out_shift,
                             char* red, long long red_shift, int tid, int nthr) {
  using S = typename D::S;
  constexpr int W = 16 / sizeof(S);
  long long body_lo = lo, body_hi = lo;
  if (vec) {
    body_lo = ((lo + W - 1) / W) * W;
    body_hi = (hi / W) * W;
    if (body_hi < body_lo) body_hi = body_lo = hi;
  }
  // scalar head and tail
  for (long long i = lo + tid; i < body_lo; i += nthr)
    reduce_one<D, OP, MP, 1, TREE>(seq, p, m, excess, i, average, out, out_shift, red, red_shift);
  for (long long i = body_hi + tid; i < hi; i += nthr)
    reduce_one<D, OP, MP, 1, TREE>(seq, p, m, excess, i, average, out, out_shift, red, red_shift);
  // vector body: vectors j in [body_lo/W, body_hi/W)
  const long long v0 = body_lo / W, v1 = body_hi / W;
  using A = typename D::A;
  // vector groups in flight per thread: ~32 operand registers whatever MP is (the
  // bulk-engine path carries the large-message traffic; this one stays spill-free)
  constexpr int OPR = MP * W * (int)(sizeof(A) / 4);
  constexpr int U = OPR >= 32 ? 1 : 32 / OPR;
  // Groups are predicated rather than peeled: the last partial round still
  // keeps every remaining load in flight at once (a peeled one-group tail
  // would pay one NVLink round trip per group).
  for (long long j = v0 + tid; j < v1; j += U * (long long)nthr) {
    A u[U][MP][W];
#pragma unroll
    for (int g = 0; g < U; ++g)
      if (j + g * (long long)nthr < v1) {
#pragma unroll
        for (int k = 0; k < MP; ++k)
          if (k < p) load_vec<D, W>(seq[k], (j + g * (long long)nthr) * W, u[g][k]);
      }
#pragma unroll
    for (int g = 0; g < U; ++g) {
      if (j + g * (long long)nthr >= v1) break;
      fold<OP, MP, W, TREE>(u[g], p, m, excess);
      if (average) {
#pragma unroll
        for (int w = 0; w < W; ++w) u[g][0][w] = div_p<A>(u[g][0][w], p);
      }
      const long long i = (j + g * (long long)nthr) * W;
      store_vec<D, W>(out, i - out_shift, u[g][0]);
      if (red) store_vec<D, W>(red, i - red_shift, u[g][0]);
    }
  }
}

// Several element ranges copied CONCURRENTLY: range r moves elements
// [lo, hi) with dst[i - dshift] = src[i - sshift]. Every thread issues the
// loads of all ranges before any store, so the allgather pulls from all
// peers at once (balanced NVLink traffic, one round trip per iteration).
struct CopyRange {
  const char* src;
  char* dst;
  long long sshift, dshift, lo, hi;
};

struct VecRange {
  const uint4* src;
  uint4* dst;
  long long nv;
};

// R[0..nr) in shared memory; V is shared scratch of the same size.
template <class D, int MP>
__device__ void multi_copy(const CopyRange* R, int nr, VecRange* V) {
  using S = typename D::S;
  constexpr int W = 16 / sizeof(S);
  const int tid = threadIdx.x, bd = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = bd >> 5;
  // scalar heads/tails (and misaligned ranges): one warp per range
  for (int r = warp; r < nr; r += nwarps) {
    const CopyRange c = R[r];
    const S* s = reinterpret_cast<const S*>(c.src) - c.sshift;
    S* d = reinterpret_cast<S*>(c.dst) - c.dshift;
    long long blo = c.hi, bhi = c.hi;
    if (((((uintptr_t)s) | ((uintptr_t)d)) & 15u) == 0) {
      blo = ((c.lo + W - 1) / W) * W;
      bhi = (c.hi / W) * W;
      if (bhi < blo) blo = bhi = c.hi;
    }
    for (long long i = c.lo + lane; i < blo; i += 32) d[i] = s[i];
    for (long long i = bhi + lane; i < c.hi; i += 32) d[i] = s[i];
    if (lane == 0) {
      V[r].src = reinterpret_cast<const uint4*>(s + blo);
      V[r].dst = reinterpret_cast<uint4*>(d + blo);
      V[r].nv = (bhi - blo) / W;
    }
  }
  __syncthreads();
  long long nvmax = 0;
  for (int r = 0; r < nr; ++r) nvmax = V[r].nv > nvmax ? V[r].nv : nvmax;
  // NS 16-byte loads in flight per thread whatever the number of ranges:
  // slot s copies range s % nr at vector offset (s / nr) * bd
  constexpr int NS = MP > 8 ? MP : 8;
  if (nr < 1) return;
  // ranges are processed in blocks of at most NS (multi-buffer launches have
  // up to MAXBUF * (p - 1) ranges)
  for (int r0 = 0; r0 < nr; r0 += NS) {
    const int nrb = nr - r0 < NS ? nr - r0 : NS;
    const VecRange* VB = V + r0;
    long long nvb = 0;
    for (int r = 0; r < nrb; ++r) nvb = VB[r].nv > nvb ? VB[r].nv : nvb;
    const int G = NS / nrb > 1 ? NS / nrb : 1;
    const int act = nrb * G < NS ? nrb * G : NS;
    int sr[NS], sg[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      sr[k] = k % nrb;
      sg[k] = k / nrb;
    }
    for (long long j0 = tid; j0 < nvb; j0 += (long long)bd * G) {
      uint4 v[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const long long j = j0 + (long long)sg[k] * bd;
        if (k < act && j < VB[sr[k]].nv) v[k] = VB[sr[k]].src[j];
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const long long j = j0 + (long long)sg[k] * bd;
        if (k < act && j < VB[sr[k]].nv) VB[sr[k]].dst[j] = v[k];
      }
    }
  }
  (void)nvmax;
}

__device__ __forceinline__ bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}

// ---- reduce through the bulk-copy engine ----------------------------------------
// The reduce-scatter's sources (p - 1 of them across NVLink) are streamed into
// a ring of shared-memory stages by ONE producer thread with cp.async.bulk
// (completion counted on a `full` mbarrier per stage), so the bytes in flight
// no longer depend on registers: stages x 32 KiB per SM. Warps 0..14 fold
// each stage (sources in the reference order) and write out / staging; each
// warp then arrives on the stage's `empty` mbarrier so the producer can refill.
constexpr int RS_MAX_STAGES = 6;
constexpr int RS_STAGE_BYTES = 32768;         // default stage size (knob bulk_stage_kb)
constexpr int RS_CONSUMERS = THREADS - 32;
__host__ __device__ constexpr size_t rs_smem_bytes(int stages, int stage_bytes = RS_STAGE_BYTES) {
  return (size_t)stages * stage_bytes + (2 * (size_t)stages + 2) * 8;
}

struct BulkRS {
  unsigned char* smem;        // stages x stage_bytes
  unsigned long long* full;   // [stages], 1 arrival + tx bytes
  unsigned long long* empty;  // [stages], RS_CONSUMERS / 32 arrivals
  unsigned long long* seqno;  // stage uses so far in this launch
  int stages;
  int stage_bytes;
};

__device__ __forceinline__ BulkRS bulk_rs_setup(unsigned char* dyn, int stages, int stage_bytes, int tid) {
  BulkRS B;
  B.stages = stages;
  B.stage_bytes = stage_bytes;
  B.smem = dyn;
  B.full = reinterpret_cast<unsigned long long*>(dyn + (size_t)stages * stage_bytes);
  B.empty = B.full + stages;
  B.seqno = B.empty + stages;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&B.full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&B.empty[s])), "r"(RS_CONSUMERS / 32));
    }
    *B.seqno = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  return B;
}

// Same contract as reduce_range (sources 16-byte aligned at vector boundaries).
template <class D, int OP, int MP, bool TREE>
__device__ void reduce_range_bulk(const BulkRS& B, const char* const* seq, int p, int m, int excess,
                                  long long lo, long long hi, int average, char* out, long long out_shift,
                                  char* red, long long red_shift, int tid, int local_k = -1) {
  // local_k >= 0: source local_k is this rank's own (HBM) buffer; the
  // consumers load it directly, so every stage byte carries NVLink traffic
  using S = typename D::S;
  using A = typename D::A;
  constexpr int W = 16 / sizeof(S);
  constexpr int SZ = sizeof(S);
  long long body_lo = ((lo + W - 1) / W) * W, body_hi = (hi / W) * W;
  if (body_hi < body_lo) body_lo = body_hi = hi;
  for (long long i = lo + tid; i < body_lo; i += THREADS)
    reduce_one<D, OP, MP, 1, TREE>(seq, p, m, excess, i, average, out, out_shift, red, red_shift);
  for (long long i = body_hi + tid; i < hi; i += THREADS)
    reduce_one<D, OP, MP, 1, TREE>(seq, p, m, excess, i, average, out, out_shift, red, red_shift);
  const long long nbytes = (body_hi - body_lo) * SZ;
  if (nbytes <= 0) return;
  const int nstaged = local_k >= 0 ? p - 1 : p;
  const int ch = (B.stage_bytes / nstaged) & ~15;       // bytes per staged source per stage
  const long long C = (nbytes + ch - 1) / ch;
  const unsigned long long base = *B.seqno;
  if (tid == RS_CONSUMERS) {                            // producer: warp 15, lane 0
    asm volatile("fence.proxy.async;" ::: "memory");
    for (long long c = 0; c < C; ++c) {
      const unsigned long long g = base + (unsigned long long)c;
      const int s = (int)(g % B.stages);
      if (g >= (unsigned long long)B.stages) mbar_wait(&B.empty[s], (unsigned)(((g / B.stages) - 1) & 1));
      const long long off = body_lo * SZ + c * ch;
      const int len = (int)((nbytes - c * ch) < ch ? (nbytes - c * ch) : ch);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&B.full[s])),
                   "r"(len * nstaged)
                   : "memory");
      for (int k = 0; k < p; ++k) {
        if (k == local_k) continue;
        const int slot = (local_k >= 0 && k > local_k) ? k - 1 : k;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(B.smem + (size_t)s * B.stage_bytes + (size_t)slot * ch)),
            "l"(seq[k] + off), "r"(len), "r"(smem_u32(&B.full[s]))
            : "memory");
      }
    }
  } else if (tid < RS_CONSUMERS) {
    for (long long c = 0; c < C; ++c) {
      const unsigned long long g = base + (unsigned long long)c;
      const int s = (int)(g % B.stages);
      mbar_wait(&B.full[s], (unsigned)((g / B.stages) & 1));
      const int len = (int)((nbytes - c * ch) < ch ? (nbytes - c * ch) : ch);
      const int nv = len / 16;
      const char* st = reinterpret_cast<const char*>(B.smem + (size_t)s * B.stage_bytes);
      const long long e0 = body_lo + c * (ch / SZ);
      for (int v = tid; v < nv; v += RS_CONSUMERS) {
        A u[MP][W];
#pragma unroll
        for (int k = 0; k < MP; ++k) {
          if (k >= p) continue;
          if (k == local_k) {
            load_vec<D, W>(seq[k], e0 + (long long)v * W, u[k]);
          } else {
            const int slot = (local_k >= 0 && k > local_k) ? k - 1 : k;
            load_vec<D, W>(st + (size_t)slot * ch, (long long)v * W, u[k]);
          }
        }
        fold<OP, MP, W, TREE>(u, p, m, excess);
        if (average) {
#pragma unroll
          for (int w = 0; w < W; ++w) u[0][w] = div_p<A>(u[0][w], p);
        }
        const long long i = e0 + (long long)v * W;
        store_vec<D, W>(out, i - out_shift, u[0]);
        if (red) store_vec<D, W>(red, i - red_shift, u[0]);
      }
      __syncwarp();
      if ((tid & 31) == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&B.empty[s])) : "memory");
    }
  }
  __syncthreads();
  if (tid == 0) *B.seqno = base + (unsigned long long)C;
  __syncthreads();
}
__device__ __forceinline__ bool al16s(const char* base, long long shift_elems, int sz) {
  return (((uintptr_t)base - (uintptr_t)(shift_elems * sz)) & 15u) == 0;
}

}  // namespace dev
}  // namespace cm
