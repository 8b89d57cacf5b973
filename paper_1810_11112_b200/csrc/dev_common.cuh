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
// record {header, src offset, reduced offset, ...} into slot [parity][b][r]
// of every peer's heap as LL units tagged with the epoch (rec_put), and polls
// its own heap (rec_get); later phase flags are a gpu-scope fence + relaxed
// store (flag_put / flag_wait). The epoch lives in device memory and is advanced by the last
// CTA of each launch, so launches can be captured into CUDA graphs. Staging is
// double-buffered by epoch parity: a rank rewrites staging[e&1] only in call
// e+2, after every peer has entered call e+1 (and therefore left call e).
// Waits are bounded (timeout -> CM_ERR_TRANSPORT in the host-mapped error word).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

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
constexpr size_t REC_BYTES = 128;             // REC_UNITS LL units (see rec_put)
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
// Automatic registration of user allocations (the pointer cache's IPC side,
// no host collective): rank r publishes allocation slot s in its own heap at
// MAILBOX[s] = {IPC handle, allocation bytes}; every peer q maps it when its
// kernels report r's new slot count, stores the mapping at AUTOTAB[s][r] in
// its own heap and acknowledges by writing ACK[q] in r's heap.
constexpr int MAXAUTO = 2048;
constexpr size_t MAILBOX_BYTES = 128;
constexpr size_t AUTOTAB_OFF = RHDF_OFF + RHDF_SIZE;
constexpr size_t AUTOTAB_SIZE = (size_t)MAXAUTO * MAXP * 8;
constexpr size_t MAILBOX_OFF = AUTOTAB_OFF + AUTOTAB_SIZE;
constexpr size_t MAILBOX_SIZE = (size_t)MAXAUTO * MAILBOX_BYTES;
constexpr size_t ACK_OFF = MAILBOX_OFF + MAILBOX_SIZE;
constexpr size_t ACK_SIZE = (size_t)MAXP * 8;
// reduce-scatter progress of the overlapped two-shot: PROG[slice][src] =
// (epoch << 32) | elements of slice `slice` (of every fused buffer, in order)
// that rank `src` has reduced, pushed by src's reduce-scatter CTA
constexpr size_t PROG_OFF = ACK_OFF + ACK_SIZE;
constexpr size_t PROG_SIZE = (size_t)MAXBLK * MAXP * 8;
// epoch slots: ESLOT[j] = epoch of the last completed call, for every j (see
// epoch_read / epoch_publish)
constexpr size_t ESLOT_OFF = PROG_OFF + PROG_SIZE;
constexpr size_t ESLOT_SIZE = (size_t)MAXBLK * 8;
constexpr size_t HEAP_ALIGN = 2ull << 20;
constexpr size_t LL_OFF = ((ESLOT_OFF + ESLOT_SIZE + HEAP_ALIGN - 1) / HEAP_ALIGN) * HEAP_ALIGN;
// record source encoding for registered inputs: bit 62 | id << 40 | byte delta
// (collective registration id), bit 62 | bit 61 | slot << 40 | delta (the
// sender's automatically registered allocation slot)
constexpr unsigned long long REG_FLAG = 1ull << 62;
constexpr unsigned long long AUTO_FLAG = 1ull << 61;
constexpr size_t CTRL_REGION = LL_OFF;                  // zeroed at creation

struct Ctrl {
  unsigned long long epoch;      // (unused: the epoch lives in the ESLOT region)
  unsigned int done;             // CTAs finished in the current call
  unsigned int pad;
  unsigned long long agree_tag;  // ticket of the last agreement check (cm_agree)
  long long agree_ok;            // its outcome: every rank held the same values
  unsigned long long ag_next;    // next allgather task of the current call (dynamic allgather)
};

// The start-barrier record a rank publishes to every peer (one per CTA and
// epoch parity), as REC_UNITS LL units (rec_put / rec_get)
enum RecField {
  RF_HDR = 0,     // call signature
  RF_SRCOFF = 1,  // element i of the sender's input at heap + srcoff + i*sz (or a REG_FLAG encoding)
  RF_REDOFF = 2,  // element i of the sender's segment at heap + redoff + (i-seg_off)*sz
  RF_AKEY = 3,    // inline agreement (aggregate's ready-set hash and count)
  RF_ACNT = 4,
  RF_REGSEQ = 5,  // allocation slots the sender has published in its mailbox
  REC_UNITS = 6
};

enum SrcMode { SRC_COPYIN = 0, SRC_PRESTAGED = 1, SRC_ZEROCOPY = 2, SRC_INLINE = 3, SRC_REGISTERED = 4,
               SRC_GATHER = 5 };
enum Order { ORD_SEQ = 0, ORD_RING = 1, ORD_TREE = 2 };
enum Phase { PH_RS = 1, PH_AG = 2 };
enum Err { ERR_SHAPE = 1, ERR_TRANSPORT = 4, ERR_CHECK = 8 };

// Checked build (-DCM_CHECKED, python paper_1810_11112_b200/_build.py --checked
// -> libcm_checked.so, loaded with CM_LIB=...): device-side bounds checks on
// every computed range, staging offset, peer address and pipeline index —
// the substitute for compute-sanitizer, which this pool does not run. A failed
// check prints its location, raises CM_ERR_CHECK in the host-mapped error
// word and traps the kernel (the host sees a launch failure).
#ifdef CM_CHECKED
static __device__ __noinline__ void cm_check_fail(const char* what, int line, unsigned* herr, long long v0 = 0,
                                                  long long v1 = 0) {
  printf("libcm checked build: '%s' failed at line %d (block %d,%d thread %d; values %lld %lld)\n", what, line,
         blockIdx.x, blockIdx.y, threadIdx.x, v0, v1);
  if (herr) *reinterpret_cast<volatile unsigned*>(herr) = ERR_CHECK;
  __threadfence_system();
  __trap();
}
#define CM_CHECK(cond, herr)                                  \
  do {                                                        \
    if (!(cond)) cm_check_fail(#cond, __LINE__, (herr));      \
  } while (0)
#define CM_CHECKV(cond, herr, v0, v1)                                                   \
  do {                                                                                  \
    if (!(cond)) cm_check_fail(#cond, __LINE__, (herr), (long long)(v0), (long long)(v1)); \
  } while (0)
#else
#define CM_CHECK(cond, herr) \
  do {                       \
  } while (0)
#define CM_CHECKV(cond, herr, v0, v1) \
  do {                                \
  } while (0)
#endif

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
  long long heap_bytes;      // size of every rank's heap (checked build)
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
  // elements at staging element offset bboff[k] and is written to
  // out[lr] + bout_off[k] elements;
  // each keeps its own reduce-scatter layout (so ring chunking, and therefore
  // the fold order, is exactly that of one allreduce per buffer)
  int nbuf;
  long long bn[MAXBUF];
  long long bboff[MAXBUF];
  long long bout_off[MAXBUF];
  long long bseg_off[MAXBUF][MAXP];
  long long bseg_len[MAXBUF][MAXP];
  // SRC_GATHER (aggregate on registered gradients): the fused buffers are the
  // concatenation of registered member tensors; gtab = {gstart[0..gmem],
  // id[0..gmem)} in device memory; peers' members are read in place through
  // REGTAB[id][q] (no pack, no staging copy)
  const long long* gtab;
  int gmem;
  long long inl[8];          // SRC_INLINE: the input travels in the parameters (cm_agree)
  unsigned long long* done_flag;  // optional: done_flag[lr] = done_value when the call completes
  unsigned long long done_value;
  int bulk_rs;               // >0: reduce through the bulk-copy engine with this many smem stages
  int bulk_stage;            // bytes per shared-memory stage of the bulk reduce
  // >0: run only if the agreement check with this ticket (queued before on the
  // same stream: the LL agreement kernel, or the inline-agreement launch)
  // succeeded; otherwise every CTA returns at once — no records, no barrier,
  // no epoch advance — so ranks whose plans (and launch counts) differ stay
  // in step
  unsigned long long agree_gate;
  // inline agreement: every rank publishes {akey, acnt} in its records; if any
  // peer's differ, every rank skips the call identically (the start barrier
  // and the epoch advance still happen: the grid is the same on every rank),
  // CTA 0 reports it through agree_out[2*lr] = {ticket, ok} (host-mapped) and
  // CTA 0 leaves {agree_tag, agree_ok} in Ctrl for the gated launches
  int agree_inline;
  long long akey[MAXP], acnt[MAXP];
  unsigned long long* agree_out;
  unsigned long long agree_ticket;
  int dyn_ag;                // allgather as a queue of (slice, peer) tasks shared by the CTAs
  // overlapped two-shot (multi-buffer kernel): CTAs [0, nrs) reduce-scatter
  // and publish per-chunk progress, CTAs [nrs, 2 nrs) allgather each peer's
  // slice chunk by chunk as soon as it is reduced (no RS->AG barrier)
  int overlap;
  int nrs;
  int ovl_chunks;            // reduce chunks per progress report / allgather block
  int ws;                    // warp-specialised two-shot (multi-buffer kernel): RS and AG warps per CTA
  // automatic registration (real communicators): my published slot count,
  // the slot counts of each peer I have mapped, and host-mapped words where
  // CTA 0 reports peers' newer slot counts (notice[q]) and the smallest
  // count every peer has acknowledged (acked)
  long long reg_seq;
  long long mapped_seq[MAXP];
  unsigned long long* notice;
  unsigned long long* acked;
};

// Programmatic dependent launch: the kernels of the collective path are
// launched with programmaticStreamSerialization, so the next launch is
// scheduled while this one drains (hides the ~2.5 us launch gap between
// back-to-back kernels). Every thread first waits for the preceding grid to
// complete and flush (a no-op without the attribute), then lets the next
// launch be scheduled.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

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

// IEEE division by p (aggregation.py:167-172: float32(float64(s)/p) == s/(float)p).
// float: RN32(RN64(s * RN64(1/p))) == RN32(s/p) for every float s and p <= 16:
// the double product is within 2^-52 relative of s/p, while s/p (a rational
// with denominator p) stays at least 2^-10 ulp away from any float rounding
// midpoint unless it lies exactly on one — so both round alike, subnormals
// included. Unlike __fdiv_rn this has no slow-path subroutine call, which
// forced the hot loops to spill their operand registers around the call site.
static __constant__ double c_rcp[MAXP + 1] = {
    0.0,      1.0,      1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,  1.0 / 6,  1.0 / 7, 1.0 / 8,
    1.0 / 9,  1.0 / 10, 1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16};
template <typename A> __device__ __forceinline__ A div_p(A a, int p);
template <> __device__ __forceinline__ float div_p<float>(float a, int p) {
  return __double2float_rn(__dmul_rn((double)a, c_rcp[p]));
}
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

__device__ __forceinline__ char* rec_slot(char* heap, int par, int blk, int src) {
  return heap + REC_OFF + ((size_t)(par * MAXBLK + blk) * MAXP + src) * REC_BYTES;
}

// ---- LL units: data and "ready" in one 16-byte store -----------------------------
// {w0, flag, w1, flag}: a reader that sees both flags equal to the expected tag
// sees the 8 payload bytes (NVLink delivers each 8-byte half whole), so no
// release/acquire fence is needed — a sys-scope release costs ~3.5 us per
// barrier on B200 (tools/flag_latency.py), a relaxed flag ~1.5 us.
__device__ __forceinline__ void st_ll(void* p, unsigned w0, unsigned w1, unsigned f) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w0), "r"(f), "r"(w1),
               "r"(f)
               : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
// poll one LL unit until both flags match; false on timeout
__device__ __forceinline__ bool ll_wait(const char* slot, unsigned f, unsigned long long timeout,
                                        uint4* out) {
  uint4 v = ld_ll(slot);
  if (v.y == f && v.w == f) { *out = v; return true; }
  const long long t0 = clock64();
  while (true) {
    for (int i = 0; i < 32; ++i) {
      v = ld_ll(slot);
      if (v.y == f && v.w == f) { *out = v; return true; }
    }
    if ((unsigned long long)(clock64() - t0) > timeout) return false;
  }
}


// the epoch's LL tag (never 0, so zeroed memory never matches)
__device__ __forceinline__ unsigned ll_tag(unsigned long long e) {
  return (unsigned)(e & 0x7fffffffu) | 0x80000000u;
}

__device__ __forceinline__ void rec_put(char* slot, unsigned tag, const long long (&v)[REC_UNITS], int nunits) {
  for (int u = 0; u < nunits; ++u)
    st_ll(slot + u * 16, (unsigned)(unsigned long long)v[u], (unsigned)((unsigned long long)v[u] >> 32), tag);
}

// All units are loaded back to back (independent loads, one L2 round trip per
// poll instead of one per unit) and the record is taken once every unit
// carries the tag.
__device__ __forceinline__ bool rec_get(const char* slot, unsigned tag, long long (&v)[REC_UNITS], int nunits,
                                        unsigned long long timeout) {
  uint4 x[REC_UNITS];
  long long t0 = -1;
  while (true) {
#pragma unroll
    for (int u = 0; u < REC_UNITS; ++u)
      if (u < nunits) x[u] = ld_ll(slot + u * 16);
    bool ok = true;
#pragma unroll
    for (int u = 0; u < REC_UNITS; ++u)
      if (u < nunits) ok = ok && x[u].y == tag && x[u].w == tag;
    if (ok) break;
    if (t0 < 0) t0 = clock64();
    else if ((unsigned long long)(clock64() - t0) > timeout) return false;
  }
#pragma unroll
  for (int u = 0; u < REC_UNITS; ++u)
    if (u < nunits) v[u] = (long long)(((unsigned long long)x[u].z << 32) | x[u].x);
  return true;
}

// Flags ordered by a gpu-scope fence instead of a sys-scope release/acquire:
// the writer's data is performed at its own L2 — where peers' NVLink loads are
// served — before the flag store leaves; the reader fences after seeing the
// flag, and reads peer data with L1-bypassing loads (ld.cg / TMA).
__device__ __forceinline__ void flag_put(unsigned long long* f, unsigned long long v) {
  __threadfence();
  st_relaxed_sys(f, v);
}
__device__ __forceinline__ bool flag_wait(const unsigned long long* f, unsigned long long e,
                                          unsigned long long timeout) {
  bool ok = true;
  if (ld_relaxed_sys(f) < e) {
    const long long t0 = clock64();
    while (ld_relaxed_sys(f) < e) {
      if ((unsigned long long)(clock64() - t0) > timeout) {
        ok = false;
        break;
      }
    }
  }
  __threadfence();
  return ok;
}
__device__ __forceinline__ unsigned long long* mid_slot(char* heap, int blk, int src) {
  return reinterpret_cast<unsigned long long*>(heap + MID_OFF + ((size_t)blk * MAXP + src) * 8);
}

// a peer's published source offset -> its address in this process
__device__ __forceinline__ const char* resolve_src(char* const* heap, char* myheap, int src, long long so,
                                                   long long heap_bytes = 0, unsigned* herr = nullptr) {
  if (!((unsigned long long)so & REG_FLAG)) {
    CM_CHECK(so >= 0 && so < heap_bytes, herr);
    return heap[src] + so;
  }
  const long long delta = so & ((1ll << 40) - 1);
  if ((unsigned long long)so & AUTO_FLAG) {       // the sender's auto-registered allocation
    const long long slot = (so >> 40) & 0x1FFFFF;
    CM_CHECK(slot < MAXAUTO, herr);
    const char* base = *reinterpret_cast<char* const*>(myheap + AUTOTAB_OFF + ((size_t)slot * MAXP + src) * 8);
    CM_CHECK(base != nullptr, herr);
    return base + delta;
  }
  const long long id = (so >> 40) & 0x1FFFFF;     // collective registration id
  CM_CHECK(id < MAXREG, herr);
  const char* base = *reinterpret_cast<char* const*>(myheap + REG_OFF + ((size_t)id * MAXP + src) * 8);
  CM_CHECK(base != nullptr, herr);
  return base + delta;
}

// CTA 0 only, after the start barrier: report peers' newer allocation slots
// and the acknowledged slot count to the host (automatic registration)
__device__ __forceinline__ void autoreg_report(const CollParams& P, char* myheap, int rank, int tid,
                                               long long peer_seq) {
  if (!P.notice) return;
  if (tid < P.p && tid != rank && peer_seq > P.mapped_seq[tid])
    reinterpret_cast<volatile unsigned long long*>(P.notice)[tid] = (unsigned long long)peer_seq;
  if (tid == 0) {
    unsigned long long lo = ~0ull;
    const volatile unsigned long long* ack = reinterpret_cast<const volatile unsigned long long*>(myheap + ACK_OFF);
    for (int q = 0; q < P.p; ++q)
      if (q != rank) lo = ack[q] < lo ? ack[q] : lo;
    *reinterpret_cast<volatile unsigned long long*>(P.acked) = lo;
  }
}

// The epoch (calls completed by this rank) without a grid-wide "last CTA"
// hand-off: CTA b of a launch reads ESLOT[b] at its start and, at its end,
// writes the new epoch to every ESLOT[j] with j = b (mod nb). After the launch
// every slot holds it, whatever the next launch's grid; no CTA of the same
// launch reads a slot another of its CTAs writes (saves the atomic + fence
// chain of the last CTA, ~1.2 us per launch).
__device__ __forceinline__ unsigned long long epoch_read(const char* heap, int b) {
  return *reinterpret_cast<const volatile unsigned long long*>(heap + ESLOT_OFF + (size_t)b * 8);
}
// every thread of the CTA, after its last use of the call's epoch-parity areas
__device__ __forceinline__ void epoch_publish(char* heap, int b, int nb, unsigned long long e) {
  unsigned long long* sl = reinterpret_cast<unsigned long long*>(heap + ESLOT_OFF);
  for (int j = b + (int)threadIdx.x * nb; j < MAXBLK; j += nb * (int)blockDim.x) sl[j] = e;
}

// a gated launch whose agreement failed is a no-op (uniform for the grid)
__device__ __forceinline__ bool gated_out(const CollParams& P, const Ctrl* ctrl) {
  return P.agree_gate && !(ctrl->agree_tag == P.agree_gate && ctrl->agree_ok);
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
// floor(a * k / d) for 0 <= a < 2^50, 0 <= k <= d <= 2^20, exactly: a double
// estimate (relative error < 2^-51, so off by at most one) corrected in
// integers — no 128-bit or 64-bit division subroutine in the kernels
__device__ __forceinline__ long long muldiv_floor(long long a, int k, int d) {
  const long long num = a * k;
  long long q = (long long)(__dmul_rn((double)num, __drcp_rn((double)d)));
  if (q * d > num) --q;
  else if ((q + 1) * d <= num) ++q;
  return q;
}

__device__ __forceinline__ long long slice_bound(long long off, long long len, int k, int nb) {
  if (k <= 0) return off;
  if (k >= nb) return off + len;
  long long x = off + muldiv_floor(len, k, nb);
  x = x & ~(long long)(SLICE_ALIGN - 1);
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
  } else if constexpr (W * sizeof(S) == 8) {
    uint2 raw = *reinterpret_cast<const uint2*>(p);
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
  } else if constexpr (W * sizeof(S) == 8) {
    uint2 raw;
    S* s = reinterpret_cast<S*>(&raw);
#pragma unroll
    for (int w = 0; w < W; ++w) s[w] = from_acc<D>(v[w]);
    *reinterpret_cast<uint2*>(p) = raw;
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) p[w] = from_acc<D>(v[w]);
  }
}

// Elements folded per thread per step: a 16-byte vector, narrowed so that the
// MP operands take at most REGS registers (bf16 accumulates in fp32, so a
// 16-byte bf16 vector would need 64 at MP = 8). The bulk-engine consumers read
// their operands from shared memory and use a 16-register budget; the SM-load
// path keeps 32 so that enough NVLink loads are in flight.
template <class D, int MP, int REGS = 32>
__host__ __device__ constexpr int fold_width() {
  constexpr int w16 = 16 / (int)sizeof(typename D::S);
  constexpr int cap = REGS / (MP * (int)(sizeof(typename D::A) / 4));
  int w = w16;
  while (w > 1 && w > cap) w /= 2;
  return w;
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

// One element, few registers: the sources are loaded one at a time. Left
// fold for ring/flat; for the rhd tree, leaves L_v (v < m) are combined by a
// binary counter (after leaf v, merge while v has trailing ones), which is the
// balanced tree with the lower subtree first — the association of tree_fold.
template <class D, int OP, int MP, bool TREE>
__device__ __forceinline__ void reduce_elem(const char* const* seq, int p, int m, int excess, long long i,
                                            int average, char* out, long long out_shift, char* red,
                                            long long red_shift) {
  using A = typename D::A;
  using S = typename D::S;
  auto ld = [&](int k) { return to_acc<D>(reinterpret_cast<const S*>(seq[k])[i]); };
  A acc;
  if constexpr (!TREE) {
    acc = ld(0);
#pragma unroll
    for (int k = 1; k < MP; ++k)
      if (k < p) acc = op2<OP>(acc, ld(k));
  } else {
    A st[5];
#pragma unroll
    for (int v = 0; v < MP; ++v) {
      if (v < m) {
        A x = ld(v);
        if (v < excess) x = op2<OP>(x, ld(m + v));
        int top = __popc(v) - 1;                       // entries on the stack before leaf v (compile time)
#pragma unroll
        for (int t = v; t & 1; t >>= 1) x = op2<OP>(st[top--], x);
        st[top + 1] = x;
      }
    }
    acc = st[0];
  }
  if (average) acc = div_p<A>(acc, p);
  reinterpret_cast<S*>(out)[i - out_shift] = from_acc<D>(acc);
  if (red) reinterpret_cast<S*>(red)[i - red_shift] = from_acc<D>(acc);
}

// Scalar head [lo, a) and tail [z, hi) of a range whose body is vectorised
template <class D, int OP, int MP, bool TREE>
__device__ __forceinline__ void reduce_scalar(const char* const* seq, int p, int m, int excess, long long lo,
                                              long long a, long long z, long long hi, int average, char* out,
                                              long long out_shift, char* red, long long red_shift, int tid,
                                              int nthr) {
#pragma unroll 1
  for (long long i = lo + tid; i < a; i += nthr)
    reduce_elem<D, OP, MP, TREE>(seq, p, m, excess, i, average, out, out_shift, red, red_shift);
#pragma unroll 1
  for (long long i = z + tid; i < hi; i += nthr)
    reduce_elem<D, OP, MP, TREE>(seq, p, m, excess, i, average, out, out_shift, red, red_shift);
}

// Process [lo, hi) of one segment: scalar head/tail, W-wide body with 2-way
// unrolling for memory-level parallelism over NVLink.
template <class D, int OP, int MP, bool TREE>
__device__ __noinline__ void reduce_range(const char* const* seq, int p, int m, int excess, long long lo,
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
  reduce_scalar<D, OP, MP, TREE>(seq, p, m, excess, lo, body_lo, body_hi, hi, average, out, out_shift, red,
                                 red_shift, tid, nthr);
  // vector body: VW-element vectors j in [body_lo/VW, body_hi/VW)
  constexpr int VW = fold_width<D, MP>();
  const long long v0 = body_lo / VW, v1 = body_hi / VW;
  using A = typename D::A;
  // vector groups in flight per thread: ~32 operand registers whatever MP is (the
  // bulk-engine path carries the large-message traffic; this one stays spill-free)
  constexpr int OPR = MP * VW * (int)(sizeof(A) / 4);
  constexpr int U = OPR >= 32 ? 1 : 32 / OPR;
  // Groups are predicated rather than peeled: the last partial round still
  // keeps every remaining load in flight at once (a peeled one-group tail
  // would pay one NVLink round trip per group).
#pragma unroll 1
  for (long long j = v0 + tid; j < v1; j += U * (long long)nthr) {
    A u[U][MP][VW];
#pragma unroll
    for (int g = 0; g < U; ++g)
      if (j + g * (long long)nthr < v1) {
#pragma unroll
        for (int k = 0; k < MP; ++k)
          if (k < p) load_vec<D, VW>(seq[k], (j + g * (long long)nthr) * VW, u[g][k]);
      }
#pragma unroll
    for (int g = 0; g < U; ++g) {
      if (j + g * (long long)nthr >= v1) break;
      fold<OP, MP, VW, TREE>(u[g], p, m, excess);
      if (average) {
#pragma unroll
        for (int w = 0; w < VW; ++w) u[g][0][w] = div_p<A>(u[g][0][w], p);
      }
      const long long i = (j + g * (long long)nthr) * VW;
      store_vec<D, VW>(out, i - out_shift, u[g][0]);
      if (red) store_vec<D, VW>(red, i - red_shift, u[g][0]);
    }
  }
}

// Several element ranges copied CONCURRENTLY: range r moves elements
// [lo, hi) with dst[i - dshift] = src[i - sshift]. The 16-byte body of every
// range is cut into 4 KiB chunks dealt round-robin over the ranges (chunk k
// belongs to range k % nr), and the warps of the CTA stride over that chunk
// sequence: at any time the CTA reads from every range (every peer of an
// allgather) at once, and each warp keeps CP_U 16-byte loads per lane in
// flight with a handful of registers (no per-range state in registers).
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

constexpr int CP_U = 8;                       // 16-byte loads in flight per lane
constexpr int CP_CHUNK = 32 * CP_U;           // vectors per warp chunk (4 KiB)

// R[0..nr) in shared memory; V is shared scratch of the same size.
template <class D, int MP>
__device__ void multi_copy(const CopyRange* R, int nr, VecRange* V, int t0 = 0, int nt = THREADS, int bar = 0) {
  auto ld_cg = [](const typename D::S* a) -> typename D::S {
    using S = typename D::S;
    if constexpr (sizeof(S) == 8) {
      const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(a));
      return *reinterpret_cast<const S*>(&v);
    } else if constexpr (sizeof(S) == 4) {
      const unsigned v = __ldcg(reinterpret_cast<const unsigned*>(a));
      return *reinterpret_cast<const S*>(&v);
    } else {
      const unsigned short v = __ldcg(reinterpret_cast<const unsigned short*>(a));
      return *reinterpret_cast<const S*>(&v);
    }
  };
  using S = typename D::S;
  constexpr int W = 16 / sizeof(S);
  const int tid = threadIdx.x - t0;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nt >> 5;
  // scalar heads/tails (and misaligned ranges): one warp per range
  for (int r = warp; r < nr; r += nwarps) {
    const CopyRange c = R[r];
    CM_CHECKV(c.lo <= c.hi, nullptr, c.lo, c.hi);
    CM_CHECKV(c.lo == c.hi || (c.src != nullptr && c.dst != nullptr), nullptr, (long long)(uintptr_t)c.src,
              (long long)(uintptr_t)c.dst);
    const S* s = reinterpret_cast<const S*>(c.src) - c.sshift;
    S* d = reinterpret_cast<S*>(c.dst) - c.dshift;
    long long blo = c.hi, bhi = c.hi;
    if (((((uintptr_t)s) | ((uintptr_t)d)) & 15u) == 0) {
      blo = ((c.lo + W - 1) / W) * W;
      bhi = (c.hi / W) * W;
      if (bhi < blo) blo = bhi = c.hi;
    }
    for (long long i = c.lo + lane; i < blo; i += 32) d[i] = ld_cg(s + i);
    for (long long i = bhi + lane; i < c.hi; i += 32) d[i] = ld_cg(s + i);
    if (lane == 0) {
      V[r].src = reinterpret_cast<const uint4*>(s + blo);
      V[r].dst = reinterpret_cast<uint4*>(d + blo);
      V[r].nv = (bhi - blo) / W;
    }
  }
  if (bar == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nt) : "memory");
  if (nr < 1) return;
  long long nvmax = 0;
  for (int r = 0; r < nr; ++r) nvmax = V[r].nv > nvmax ? V[r].nv : nvmax;
  const int nchunks = (int)((nvmax + CP_CHUNK - 1) / CP_CHUNK) * nr;   // < 2^31: slices are small
#pragma unroll 1
  for (int k = warp; k < nchunks; k += nwarps) {
    const int r = k % nr;
    const long long c0 = (long long)(k / nr) * CP_CHUNK;
    const long long nv = V[r].nv;
    if (c0 >= nv) continue;
    const uint4* src = V[r].src + c0;
    uint4* dst = V[r].dst + c0;
    const int m = (int)(nv - c0 < CP_CHUNK ? nv - c0 : CP_CHUNK);
    uint4 v[CP_U];
#pragma unroll
    for (int u = 0; u < CP_U; ++u)
      if (lane + 32 * u < m) v[u] = __ldcg(src + lane + 32 * u);   // peer data: bypass L1
#pragma unroll
    for (int u = 0; u < CP_U; ++u)
      if (lane + 32 * u < m) dst[lane + 32 * u] = v[u];
  }
}

__device__ __forceinline__ bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// one element through L2 only (peer data after a flag: no stale L1 line)
__device__ __forceinline__ float ld_cg_elem(const float* a) { return __ldcg(a); }
__device__ __forceinline__ double ld_cg_elem(const double* a) { return __ldcg(a); }

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

// The threads that run a bulk-engine reduce: `ncons` consumers (tid < ncons),
// the producer (tid == ncons, one lane of the next warp) and their group
// barrier (`bar` 0 = the whole CTA). The warp-specialised two-shot runs the
// reduce on warps 0..8 and the allgather on warps 9..15 of the same CTA.
struct Team {
  int ncons;
  int grp;
  int bar;
};
__host__ __device__ constexpr Team team_all() { return Team{RS_CONSUMERS, THREADS, 0}; }
__host__ __device__ constexpr Team team_ws_rs() { return Team{256, 288, 3}; }
constexpr int WS_AG_T0 = 288, WS_AG_N = THREADS - 288, WS_AG_BAR = 2;

__device__ __forceinline__ void team_sync(const Team T) {
  if (T.bar == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(T.bar), "r"(T.grp) : "memory");
}
__host__ __device__ constexpr size_t rs_smem_bytes(int stages, int stage_bytes = RS_STAGE_BYTES) {
  return (size_t)stages * stage_bytes + (2 * (size_t)stages + 2) * 8;
}

// The stage ring lives at the start of the launch's dynamic shared memory; its
// view is rebuilt from (stages, stage_bytes) — kernel parameters — wherever it
// is used, so no pointers to it stay live in registers across the kernel.
extern __shared__ __align__(128) unsigned char cm_dyn_smem[];

struct BulkRS {
  unsigned char* smem;        // stages x stage_bytes
  unsigned long long* full;   // [stages], 1 arrival + tx bytes
  unsigned long long* empty;  // [stages], RS_CONSUMERS / 32 arrivals
  unsigned long long* seqno;  // stage uses so far in this launch
  int stages;
  int stage_bytes;
};

__device__ __forceinline__ BulkRS bulk_view(int stages, int stage_bytes) {
  BulkRS B;
  B.stages = stages;
  B.stage_bytes = stage_bytes;
  B.smem = cm_dyn_smem;
  B.full = reinterpret_cast<unsigned long long*>(cm_dyn_smem + (size_t)stages * stage_bytes);
  B.empty = B.full + stages;
  B.seqno = B.empty + stages;
  return B;
}

__device__ __forceinline__ void bulk_rs_setup(int stages, int stage_bytes, int tid, int ncons = RS_CONSUMERS) {
  const BulkRS B = bulk_view(stages, stage_bytes);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&B.full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&B.empty[s])), "r"(ncons / 32));
    }
    *B.seqno = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// Progress publication of the overlapped two-shot: after each reduced chunk the
// consumers synchronise and one thread pushes (tag | base + elements done in
// this range) to every peer's PROG[blk][rank] (gpu-scope fence + relaxed store).
struct Prog {
  unsigned long long* dst[MAXP];   // peers' PROG slots for this CTA's slice (nullptr: self)
  unsigned long long tag;          // epoch << 32
  long long base;                  // slice-sequence position of the range start
  int p;
  int every;                       // report after every `every`-th chunk (and the last)
};

__device__ __forceinline__ void prog_publish(const Prog* pg, long long pos) {
  __threadfence();
  for (int q = 0; q < pg->p; ++q)
    if (pg->dst[q]) st_relaxed_sys(pg->dst[q], pg->tag | (unsigned long long)pos);
}

// Same contract as reduce_range (sources 16-byte aligned at vector boundaries).
template <class D, int OP, int MP, bool TREE>
__device__ void reduce_range_bulk(int stages, int stage_bytes, const char* const* seq, int p, int m, int excess,
                                  long long lo, long long hi, int average, char* out, long long out_shift,
                                  char* red, long long red_shift, int tid, const Prog* prog = nullptr,
                                  const Team T = team_all()) {
  const BulkRS B = bulk_view(stages, stage_bytes);
  using S = typename D::S;
  using A = typename D::A;
  constexpr int W = 16 / sizeof(S);
  constexpr int SZ = sizeof(S);
  long long body_lo = ((lo + W - 1) / W) * W, body_hi = (hi / W) * W;
  if (body_hi < body_lo) body_lo = body_hi = hi;
  if (body_lo > lo || body_hi < hi)
    reduce_scalar<D, OP, MP, TREE>(seq, p, m, excess, lo, body_lo, body_hi, hi, average, out, out_shift, red,
                                   red_shift, tid, T.grp);
  const long long nbytes = (body_hi - body_lo) * SZ;
  if (nbytes <= 0) return;
  if (prog) team_sync(T);         // the scalar head/tail precede every progress report
  const int ch = (B.stage_bytes / p) & ~15;             // bytes per source per stage
  const int C = (int)((nbytes + ch - 1) / ch);
  // stage uses so far in this launch (< 2^32): stage index and mbarrier phase
  // advance incrementally (no 64-bit division in the loops)
  const unsigned base = (unsigned)*B.seqno;
  if (tid == T.ncons) {                                 // producer: lane 0 of the warp after the consumers
    asm volatile("fence.proxy.async;" ::: "memory");
    int s = (int)(base % (unsigned)B.stages);
    unsigned ph = (base / (unsigned)B.stages) & 1u;
    bool wrapped = base >= (unsigned)B.stages;
    for (int c = 0; c < C; ++c) {
      if (wrapped) mbar_wait(&B.empty[s], ph ^ 1u);
      const long long off = body_lo * SZ + (long long)c * ch;
      const int len = (int)((nbytes - (long long)c * ch) < ch ? (nbytes - (long long)c * ch) : ch);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&B.full[s])),
                   "r"(len * p)
                   : "memory");
      CM_CHECK(s < B.stages && (size_t)p * ch <= (size_t)B.stage_bytes && len > 0 && len <= ch && (len & 15) == 0,
               nullptr);
      for (int k = 0; k < p; ++k) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(B.smem + (size_t)s * B.stage_bytes + (size_t)k * ch)),
            "l"(seq[k] + off), "r"(len), "r"(smem_u32(&B.full[s]))
            : "memory");
      }
      if (++s == B.stages) { s = 0; ph ^= 1u; wrapped = true; }
    }
  } else if (tid < T.ncons) {
    int s = (int)(base % (unsigned)B.stages);
    unsigned ph = (base / (unsigned)B.stages) & 1u;
    for (int c = 0; c < C; ++c) {
      mbar_wait(&B.full[s], ph);
      const int len = (int)((nbytes - (long long)c * ch) < ch ? (nbytes - (long long)c * ch) : ch);
      constexpr int VW = fold_width<D, MP, 16>();
      const int nv = len / (VW * SZ);
      const char* st = reinterpret_cast<const char*>(B.smem + (size_t)s * B.stage_bytes);
      const long long e0 = body_lo + (long long)c * (ch / SZ);
#pragma unroll 1
      for (int v = tid; v < nv; v += T.ncons) {
        A u[MP][VW];
#pragma unroll
        for (int k = 0; k < MP; ++k) {
          if (k >= p) continue;
          load_vec<D, VW>(st + (size_t)k * ch, (long long)v * VW, u[k]);
        }
        fold<OP, MP, VW, TREE>(u, p, m, excess);
        if (average) {
#pragma unroll
          for (int w = 0; w < VW; ++w) u[0][w] = div_p<A>(u[0][w], p);
        }
        const long long i = e0 + (long long)v * VW;
        store_vec<D, VW>(out, i - out_shift, u[0]);
        if (red) store_vec<D, VW>(red, i - red_shift, u[0]);
      }
      __syncwarp();
      if ((tid & 31) == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&B.empty[s])) : "memory");
      if (prog && ((c + 1) % prog->every == 0 || c + 1 == C)) {   // chunks stored by every consumer: report
        asm volatile("bar.sync 1, %0;" ::"r"(T.ncons) : "memory");
        if (tid == 0) {
          // the scalar tail [body_hi, hi) was reduced before the first chunk
          const long long done = c + 1 == C ? hi - lo : body_lo - lo + (long long)(c + 1) * (ch / SZ);
          prog_publish(prog, prog->base + done);
        }
      }
      if (++s == B.stages) { s = 0; ph ^= 1u; }
    }
  }
  team_sync(T);
  if (tid == 0) *B.seqno = base + (unsigned)C;
  team_sync(T);
}
__device__ __forceinline__ bool al16s(const char* base, long long shift_elems, int sz) {
  return (((uintptr_t)base - (uintptr_t)(shift_elems * sz)) & 15u) == 0;
}

}  // namespace dev
}  // namespace cm
