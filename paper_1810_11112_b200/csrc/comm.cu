// Communicator: CUDA-IPC symmetric heap over NVLink/NVSwitch, algorithm
// selection, pointer-cache classification on every call, and kernel launches.
//
// Host flow of one cm_allreduce (collectives.py:250-260):
//   resolve_algorithm (size threshold) -> classify send/recv through the
//   pointer cache (no driver query on a cache hit, PAPER §V-B) -> pick the
//   source mode (zero-copy from the symmetric pool, copy-in, or host staging)
//   -> ONE kernel launch (one-shot or two-shot) -> logical CollectiveStats.
//
// Sections:
//   struct cm_comm                      per-rank state (heap, staging, knobs, counters)
//   launch_collective / plan_algo       grid sizing, kernel choice, parameters
//   place / do_allreduce / do_rs / do_ag  buffer placement and the single collectives
//   launch_batched_copy / coalesce / HostPipe   packs and the host-gradient pipeline
//   cm_comm_* (extern "C")              lifecycle, IPC bootstrap, registration, knobs
//   agreement helpers, cm_agree         ready-set agreement (LL kernel / inline)
//   cm_allreduce..cm_allgather_v        the C ABI of the collectives
//   cm_fused_allreduce_agreed           aggregate(): plan, agreement, launches, pipeline
//   cm_ps_step(_v)                      parameter-server step
//   cm_local_reduce, cm_batched_copy, cm_bench_p2p, cm_time_allreduce
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"
#include "ptrcache.hpp"

using namespace cm;
using namespace cm::dev;

struct cm_comm {
  int rank = 0, size = 1, device = 0;
  bool virt = false;
  size_t staging_bytes = 0, pool_bytes = 0, heap_bytes = 0;
  size_t staging_off = 0;           // runtime heap layout (after the LL region)
  int64_t ll_units = 0;             // LL units per (parity, phase, source)
  char* local = nullptr;            // own heap (virtual: all vranks' heaps)
  char* heap[MAXP] = {};
  bool connected = false;
  unsigned* herr_host = nullptr;
  unsigned* herr_dev = nullptr;
  unsigned long long timeout_cycles = 20000000000ull;  // ~10 s at 2 GHz
  Registry reg;
  std::map<size_t, size_t> pool_free;  // offset -> bytes
  std::map<size_t, size_t> pool_used;
  char* scratch = nullptr;             // device bounce buffer for host-memory buffers
  // host-memory aggregate pipeline: inputs land in `indev` on the h2d stream,
  // results leave `outdev` on the d2h stream, overlapping both PCIe directions
  char* indev = nullptr;
  char* outdev = nullptr;
  int64_t indev_bytes = 0, outdev_bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> sync_events;
  int64_t* agree_host = nullptr;       // mapped pinned agreement words (AGH_* layout below)
  int64_t* agree_dev = nullptr;        // device alias of agree_host
  int64_t* agree_in = nullptr;         // device copy of the virtual ranks' agreement inputs
  unsigned long long agree_ticket = 0;
  // registered buffers (cm_comm_register): local start -> {bytes, id}; opened
  // peer allocations cached by (peer, handle bytes) -> mapped base
  struct Reg {
    int64_t bytes;
    int64_t id;
  };
  std::map<uintptr_t, Reg> regs;
  std::map<std::string, char*> opened;
  std::map<std::string, long long*> gtabs;   // member tables of registered fused batches
  int64_t next_reg = 0;
  // automatic registration of user allocations (dev_common.cuh MAILBOX/AUTOTAB/ACK):
  // allocation base -> {bytes, mailbox slot (-1: not IPC-exportable), buffer id}
  struct AutoReg {
    size_t size;
    int64_t slot;
    unsigned long long buffer_id;
  };
  int auto_reg = 1;
  std::map<uintptr_t, AutoReg> autoregs;
  int64_t reg_seq = 0;                      // slots published in my mailbox
  int64_t mapped_seq[MAXP] = {};            // peers' slots mapped into AUTOTAB
  unsigned long long* areg_host = nullptr;  // mapped pinned: notice[MAXP], acked
  unsigned long long* areg_dev = nullptr;
  unsigned char* areg_pin = nullptr;        // pinned scratch for mailbox reads / table writes
  cudaStream_t reg_stream = nullptr;
  int64_t auto_published = 0, auto_mapped = 0, auto_zc_calls = 0, auto_checks = 0;
  int sms = 148;
  // tuning knobs (cm_comm_set_param)
  int64_t oneshot_max_bytes = 32 * 1024;
  int64_t ll_max_bytes = 32 * 1024;           // one-shot via LL slots up to here
  int64_t ll_units_per_cta = 512;
  int64_t ll2_max_bytes = -1;                 // two-shot via LL slots up to here (-1: p x 512 KiB)
  int64_t ll2_units_per_cta = 512;
  int64_t stream_chunk = 0;                   // elements; 0 disables the pipelined two-shot
  int multi_buffer = 1;                       // batch fused buffers into one launch
  int rhd_logp = 0;                           // 1: rhd_rsa runs the log2(p)-step halving/doubling kernel
  int bulk_copy = 0;                          // fusion pack through the TMA bulk-copy engine (opt-in)
  int bulk_rs = 6;                            // reduce phase: bulk-engine stages in smem (0: SM loads)
  int dyn_ag = 0;                             // allgather as a shared (slice, peer) task queue (opt-in)
  int inline_agree = 1;                       // aggregate's agreement inside the collective's records
  int overlap = 0;                            // multi-buffer two-shot: RS and AG CTAs run concurrently
                                              // (opt-in: measured slower, the RS needs every SM)
  int ovl_chunks = 4;                         // reduce chunks per progress report (overlap, ws)
  int ws = 0;                                 // multi-buffer two-shot: RS and AG warps in every CTA
  int pack_waves = 2;                         // batched copy: CTA waves (4 per SM per wave)
  int pack_max_ctas = 0;                      // batched copy: CTA cap (0: none; overlapped aggregation)
  int pack_unroll = 4;                        // batched copy: 16-byte loads in flight per thread (4 or 8)
  bool host_split = true;                     // host pipeline (p > 1): fused groups move in pieces
  int64_t host_piece = 4 << 20;               // ... of about this many bytes
  bool pdl = true;                            // programmatic dependent launch of the collective kernels
  bool cluster2 = false;                      // capped collective grids in 2-CTA clusters (whole TPCs)
  int bulk_stage = 2 * RS_STAGE_BYTES;        // bytes per bulk-reduce stage (64 KiB: 3 stages fit)
  int64_t host_chunk = 8 << 20;               // host-gradient pipeline: bytes per H2D/D2H piece
  int64_t oneshot_bytes_per_cta = 8 * 1024;
  int64_t twoshot_bytes_per_cta = 4 * 1024;
  int max_ctas = 148;
  // counters
  int64_t messages = 0, bytes = 0, nvlink_in = 0, calls = 0, launches = 0;
  // optional per-launch CUDA-event profiling (bench roofline)
  struct Prof {
    int kind;
    cudaEvent_t e0, e1;
    int64_t alg_bytes;
  };
  unsigned long long* trace = nullptr;  // cm_comm_set_trace
  int trace_ctas = 0;
  bool profiling = false;
  std::vector<Prof> prof;
  std::vector<cudaEvent_t> event_pool;
};

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();
  return fail(CM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                              \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// The communicator's device for the duration of one entry point (restored
// after), so callers need not switch devices around every collective.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Launch with programmatic stream serialization (the kernel starts with
// pdl_begin(): it waits for the preceding grid itself), or plainly.
// cluster2: CTAs in clusters of two (both SMs of a TPC), so a capped grid
// running next to 2-CTA-cluster GEMMs takes whole TPCs instead of breaking
// one pair per CTA.
cudaError_t launch_k(bool pdl, const void* k, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s,
                     bool cluster2 = false) {
  if (!pdl && !cluster2) return cudaLaunchKernel(k, grid, block, args, smem, s);
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster2) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelExC(&cfg, k, args);
}

// LL payload capacity per source: 2 MiB on real communicators (two-shot LL up
// to p x 2 MiB), 256 KiB per virtual rank (single-GPU emulation)
constexpr int64_t CM_LL_UNITS_REAL = 256 * 1024;
constexpr int64_t CM_LL_UNITS_VIRTUAL = 32 * 1024;

cudaEvent_t take_event(cm_comm* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// bracket one launch with events when profiling (kind 0 collective, 1 pack)
struct ProfScope {
  cm_comm* c;
  cudaStream_t s;
  int kind;
  int64_t bytes;
  cudaEvent_t e0 = nullptr;
  ProfScope(cm_comm* c_, cudaStream_t s_, int k, int64_t b) : c(c_), s(s_), kind(k), bytes(b) {
    if (c && c->profiling) {
      e0 = take_event(c);
      cudaEventRecord(e0, s);
    }
  }
  ~ProfScope() {
    if (e0) {
      cudaEvent_t e1 = take_event(c);
      cudaEventRecord(e1, s);
      c->prof.push_back({kind, e0, e1, bytes});
    }
  }
};

using KFn = void (*)(CollParams);

// cudaFuncAttributeMaxDynamicSharedMemorySize is set per (device, kernel):
// `want` < 0 opts in to everything next to the static shared memory and
// returns that amount in *avail
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_attr;

int dyn_smem_optin(int device, const void* k, int* avail, int want = -1) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  auto key = std::make_pair(device, k);
  auto it = g_attr.find(key);
  if (it != g_attr.end()) { *avail = it->second; return CM_OK; }
  int optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  cudaFuncAttributes fa;
  CUDA_TRY(cudaFuncGetAttributes(&fa, k));
  const int a = want >= 0 ? want : optin - (int)fa.sharedSizeBytes;
  CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a));
  g_attr[key] = a;
  *avail = a;
  return CM_OK;
}

// kernel tables live in one translation unit per element type (csrc/inst_*.cu)
// so the instantiations compile in parallel
enum KernelKind { K_COLL = 0, K_STREAM = 1, K_LL = 2, K_LL2 = 3, K_RHD = 4, K_MULTI = 5 };

KFn pick(int kind, int dtype, int op, int p, bool tree) {
  const bool sum = op == CM_SUM;
  switch (dtype) {
    case CM_FLOAT32: return sum ? cm_kernels_f32_sum(kind, p, tree) : cm_kernels_f32_max(kind, p, tree);
    case CM_FLOAT64: return sum ? cm_kernels_f64_sum(kind, p, tree) : cm_kernels_f64_max(kind, p, tree);
    case CM_BFLOAT16: return sum ? cm_kernels_bf16_sum(kind, p, tree) : cm_kernels_bf16_max(kind, p, tree);
    case CM_INT32: return sum ? cm_kernels_i32_sum(kind, p, tree) : cm_kernels_i32_max(kind, p, tree);
    case CM_INT64: return sum ? cm_kernels_i64_sum(kind, p, tree) : cm_kernels_i64_max(kind, p, tree);
  }
  return nullptr;
}

int check_dtype_op(int dtype, int op) {
  if (!dtype_size(dtype)) return fail(CM_ERR_SHAPE, "unsupported dtype " + std::to_string(dtype));
  if (op != CM_SUM && op != CM_MAX) return fail(CM_ERR_VALUE, "unknown reduce op " + std::to_string(op));
  return CM_OK;
}

int check_async_error(cm_comm* c) {
  volatile unsigned* h = c->herr_host;
  const unsigned code = *h;
  if (!code) return CM_OK;
  *h = 0;
  if (code == ERR_SHAPE)
    return fail(CM_ERR_SHAPE,
                "collective shape error: peers disagree on element count, dtype, op or algorithm");
  if (code == ERR_CHECK)
    return fail(CM_ERR_CUDA, "device-side bounds check failed (checked build; see the kernel's printf)");
  return fail(CM_ERR_TRANSPORT, "peer did not arrive within the timeout (rank failed or "
                                "called a different collective)");
}

// Where the data of `ptr` lives, through the pointer cache (PAPER §V-B).
int classify(cm_comm* c, const void* ptr, int* kind) {
  const uint64_t a = reinterpret_cast<uint64_t>(ptr);
  // our own symmetric heap is always known (it is an intercepted allocation)
  if (!c->virt && a >= (uint64_t)c->local && a < (uint64_t)c->local + c->heap_bytes) {
    *kind = CM_KIND_DEVICE;
    return CM_OK;
  }
  return c->reg.classify(a, kind);
}

bool in_pool(cm_comm* c, const void* ptr, int64_t bytes) {
  if (c->virt || !c->local) return false;
  const char* p = static_cast<const char*>(ptr);
  const char* lo = c->local + c->staging_off + 2 * c->staging_bytes;
  return p >= lo && p + bytes <= c->local + c->heap_bytes;
}

unsigned long long make_hdr(int64_t n, int dtype, int op, int order, int phases, int oneshot,
                            int average, int layout) {
  unsigned long long h = (unsigned long long)n & ((1ull << 40) - 1);
  h |= (unsigned long long)(dtype & 7) << 40;
  h |= (unsigned long long)(op & 1) << 43;
  h |= (unsigned long long)(order & 3) << 44;
  h |= (unsigned long long)(phases & 3) << 46;
  h |= (unsigned long long)(oneshot & 1) << 48;
  h |= (unsigned long long)(average & 1) << 49;
  h |= (unsigned long long)(layout & 1) << 50;
  return h;
}

static_assert(SLICE_ALIGN == 64, "segments_of (hostlogic.cpp) cuts pieces on 64-element slice boundaries");

struct Launch {
  int64_t n = 0;
  int dtype = 0, op = 0, order = ORD_SEQ, phases = PH_RS | PH_AG, oneshot = 0;
  int out_rel = 0, ag_in_rel = 0, average = 0, layout = CM_LAYOUT_RING;
  int srcmode = SRC_COPYIN;
  const long long* inl = nullptr;   // SRC_INLINE payload (<= 8 words)
  const long long* gtab = nullptr;  // SRC_GATHER member table (device)
  int gmem = 0;
  unsigned long long gsig = 0;      // member-table signature (checked across ranks)
  int nbuf = 1;                     // multi-buffer launch (prestaged, two-shot pull)
  int64_t bn[MAXBUF] = {};
  int64_t bboff[MAXBUF] = {};
  int64_t bout_off[MAXBUF] = {};    // element offset of buffer k's output in out[lr]
  unsigned long long* done_flag = nullptr;
  unsigned long long done_value = 0;
  unsigned long long agree_gate = 0;  // run only if agreement check `agree_gate` succeeded
  int agree_inline = 0;               // agreement values travel in the start-barrier records
  long long akey[MAXP] = {}, acnt[MAXP] = {};
  unsigned long long* agree_out = nullptr;
  unsigned long long agree_ticket = 0;
  int force_pull = 0;               // pull collective kernel on the full grid (inline agreement:
                                    // the launch must have the same shape on every rank)
  int ll = 0;                       // one-shot through the LL slots
  int piece = 0, npieces = 1;       // host pipeline: the piece-th 1/npieces of every segment
  const void* in[MAXP] = {};
  void* out[MAXP] = {};
  int64_t zc_srcoff[MAXP] = {};
};

int launch_collective(cm_comm* c, const Launch& L, cudaStream_t stream) {
  const int p = c->size;
  const size_t sz = dtype_size(L.dtype);
  CollParams P;
  memset(&P, 0, sizeof P);
  for (int q = 0; q < p; ++q) P.heap[q] = c->heap[q];
  const int nloc = c->virt ? p : 1;
  for (int q = 0; q < nloc; ++q) {
    P.in[q] = static_cast<const char*>(L.in[q]);
    P.out[q] = static_cast<char*>(L.out[q]);
    P.zc_srcoff[q] = L.zc_srcoff[q];
  }
  int64_t off[MAXP], len[MAXP];
  if (L.oneshot) {
    for (int q = 0; q < p; ++q) { off[q] = 0; len[q] = L.n; }
  } else {
    segments_of(L.n, p, L.layout, L.piece, L.npieces, off, len);
  }
  int64_t maxseg = 0;
  for (int q = 0; q < p; ++q) {
    P.seg_off[q] = off[q];
    P.seg_len[q] = len[q];
    maxseg = std::max(maxseg, len[q]);
  }
  P.n = L.n;
  unsigned long long multi_hash = 0;
  P.gtab = L.gtab;
  P.gmem = L.gmem;
  if (L.nbuf > 1 || L.srcmode == SRC_GATHER) {
    P.nbuf = L.nbuf;
    maxseg = 0;
    multi_hash = 1469598103934665603ull;
    for (int k = 0; k < L.nbuf; ++k) {
      int64_t bo[MAXP], bl[MAXP];
      if (L.layout == CM_LAYOUT_RHD) rhd_layout(L.bn[k], p, bo, bl);
      else chunk_partition(L.bn[k], p, bo, bl);
      int64_t mk = 0;
      for (int q = 0; q < p; ++q) {
        P.bseg_off[k][q] = bo[q];
        P.bseg_len[k][q] = bl[q];
        mk = std::max(mk, bl[q]);
      }
      maxseg += mk;                    // per-CTA work spans every buffer
      P.bn[k] = L.bn[k];
      P.bboff[k] = L.bboff[k];
      P.bout_off[k] = L.bout_off[k];
      multi_hash = (multi_hash ^ (unsigned long long)L.bn[k]) * 1099511628211ull;
    }
    multi_hash = (multi_hash ^ L.gsig) * 1099511628211ull;
  }
  P.hdr = make_hdr(P.nbuf >= 1 && (L.nbuf > 1 || L.srcmode == SRC_GATHER) ? (int64_t)(multi_hash >> 24) : L.n, L.dtype, L.op, L.order, L.phases,
                   L.oneshot, L.average, L.layout) ^ ((unsigned long long)(L.nbuf - 1) << 51);
  P.timeout_cycles = c->timeout_cycles;
  P.staging_bytes = (long long)c->staging_bytes;
  P.herr = c->herr_dev;
  P.heap_bytes = (long long)c->heap_bytes;
  P.p = p;
  P.rank = c->rank;
  P.virt = c->virt ? 1 : 0;
  P.srcmode = L.srcmode;
  P.order = L.order;
  P.phases = L.phases;
  P.oneshot = L.oneshot;
  P.out_rel = L.out_rel;
  P.ag_in_rel = L.ag_in_rel;
  P.average = L.average;
  P.staging_off = (long long)c->staging_off;
  P.ll_units = c->ll_units;
  if (L.inl) for (int i = 0; i < 8; ++i) P.inl[i] = L.inl[i];
  P.done_flag = L.done_flag;
  P.done_value = L.done_value;
  P.agree_gate = L.agree_gate;
  P.agree_inline = L.agree_inline;
  for (int q = 0; q < MAXP; ++q) { P.akey[q] = L.akey[q]; P.acnt[q] = L.acnt[q]; }
  P.agree_out = L.agree_out;
  P.agree_ticket = L.agree_ticket;
  P.dyn_ag = c->dyn_ag;
  if (!c->virt && c->areg_dev) {
    P.reg_seq = c->reg_seq;
    for (int q = 0; q < p; ++q) P.mapped_seq[q] = c->mapped_seq[q];
    P.notice = c->areg_dev;
    P.acked = c->areg_dev + MAXP;
  }
  P.trace = c->trace;
  P.trace_ctas = c->trace_ctas;

  // grid: CTAs per rank; identical on every rank (depends on n, p, dtype only)
  const int64_t work = L.oneshot ? L.n * (int64_t)sz : maxseg * (int64_t)sz;
  const int64_t per = L.oneshot ? c->oneshot_bytes_per_cta : c->twoshot_bytes_per_cta;
  int64_t nb = (work + per - 1) / per;
  int ll = L.ll;
  // literal recursive halving/doubling (log2 p pairwise steps) for rhd_rsa allreduce
  const bool logp = !L.force_pull && L.npieces == 1 && c->rhd_logp && L.order == ORD_TREE && L.nbuf == 1 && L.dtype != CM_BFLOAT16 &&
                    !L.out_rel && (L.oneshot || L.phases == (PH_RS | PH_AG)) &&
                    (L.srcmode == SRC_COPYIN || L.srcmode == SRC_ZEROCOPY || L.srcmode == SRC_REGISTERED);
  if (logp || L.force_pull) ll = 0;
  if (ll == 1 && (L.n * (int64_t)sz + 7) / 8 > c->ll_units) ll = 0;
  if (ll == 2 && (maxseg * (int64_t)sz + 7) / 8 > c->ll_units) ll = 0;  // rhd segments > n/p
  // staging capacity (LL kernels read the input directly unless it is prestaged)
  {
    int64_t need = (L.srcmode == SRC_ZEROCOPY) ? (maxseg + SLICE_ALIGN) * (int64_t)sz
                                              : L.n * (int64_t)sz;
    if (L.nbuf > 1 || L.srcmode == SRC_GATHER) need = (L.bboff[L.nbuf - 1] + L.bn[L.nbuf - 1]) * (int64_t)sz;
    if (logp) need = L.n * (int64_t)sz;
    const bool uses_staging = ll == 0 || L.srcmode == SRC_PRESTAGED;
    if (uses_staging && need > (int64_t)c->staging_bytes)
      return fail(CM_ERR_CONFIG, "message of " + std::to_string(L.n * sz) + " B needs " +
                                     std::to_string(need) + " B of staging; the communicator has " +
                                     std::to_string(c->staging_bytes) +
                                     " (raise staging_bytes or allocate the buffers with comm.alloc)");
  }
  if (ll == 1) nb = ((L.n * (int64_t)sz + 7) / 8 + c->ll_units_per_cta - 1) / c->ll_units_per_cta;
  if (ll == 2) nb = ((maxseg * (int64_t)sz + 7) / 8 + c->ll2_units_per_cta - 1) / c->ll2_units_per_cta;
  if (logp) nb = (L.n * (int64_t)sz + c->twoshot_bytes_per_cta - 1) / c->twoshot_bytes_per_cta;
  const int full = std::max(2, std::min(c->max_ctas, MAXBLK) & ~1);
  if (L.force_pull) nb = full;        // the full grid (even): independent of the (rank-local) plan
  nb = std::max<int64_t>(1, std::min<int64_t>(nb, full));
  const bool tree = L.order == ORD_TREE;
  // pipelined two-shot when every CTA's slice spans >= 2 chunks
  const bool pipelined = ll == 0 && L.nbuf == 1 && L.srcmode != SRC_GATHER && !L.oneshot &&
                         L.phases == (PH_RS | PH_AG) &&
                         c->stream_chunk > 0 && maxseg / std::max<int64_t>(nb, 1) >= 2 * c->stream_chunk;
  P.stream_chunk = c->stream_chunk;
  if (L.agree_inline && (logp || ll != 0))
    return fail(CM_ERR_CONFIG, "internal: inline agreement needs the pull collective kernel");
  const bool multi = L.nbuf > 1 || L.srcmode == SRC_GATHER;
  KFn k = pick(logp ? K_RHD : ll == 1 ? K_LL : ll == 2 ? K_LL2 : pipelined ? K_STREAM : multi ? K_MULTI : K_COLL,
               L.dtype, L.op, p, tree);
  if (!k) return fail(CM_ERR_SHAPE, "unsupported dtype");
  // reduce phase through the bulk-copy engine (shared-memory stage ring)
  const bool bulk = c->bulk_rs > 0 && !logp && ll == 0 && !pipelined && (L.phases & PH_RS);
  // dynamic shared memory available next to the kernel's static arrays (the
  // opt-in is a per-device function attribute)
  int avail = 0;
  if (bulk) {
    int st = dyn_smem_optin(c->device, (const void*)k, &avail);
    if (st) return st;
  }
  int stages = c->bulk_rs;
  if (bulk)
    while (stages > 1 && rs_smem_bytes(stages, c->bulk_stage) > (size_t)avail) --stages;
  P.bulk_rs = bulk ? stages : 0;
  P.bulk_stage = c->bulk_stage;
  // overlapped two-shot: half the grid reduce-scatters, half allgathers
  const bool ovl = multi && c->overlap && bulk && !c->dyn_ag;
  if (ovl) {
    int64_t nrs = std::max<int64_t>(1, std::min<int64_t>(nb, full / 2));
    if (L.force_pull) nrs = full / 2;
    nb = 2 * nrs;
  }
  const size_t dsm = bulk ? rs_smem_bytes(stages, c->bulk_stage) : 0;
  void* args[] = {&P};
  int64_t alg = 0;   // busBW bytes of this launch (nccl-tests convention)
  int64_t ntot = L.n;
  if (L.nbuf > 1 || L.srcmode == SRC_GATHER) { ntot = 0; for (int k = 0; k < L.nbuf; ++k) ntot += L.bn[k]; }
  if (L.phases == (PH_RS | PH_AG) || L.oneshot) alg = 2 * (int64_t)(p - 1) * ntot * (int64_t)sz / p;
  else alg = (int64_t)(p - 1) * L.n * (int64_t)sz / p;
  ProfScope prof_scope(c, stream, (ll != 0 || logp) ? 2 : 0, alg);   // 0 pull collective, 2 LL / log-p
  if (c->virt) {
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k, THREADS, dsm));
    const int64_t cap = (int64_t)per_sm * c->sms / p;
    if (cap < (ovl ? 2 : 1)) return fail(CM_ERR_CONFIG, "virtual group too large for one GPU");
    nb = std::min<int64_t>(nb, ovl ? (cap & ~(int64_t)1) : cap);
    P.overlap = ovl ? 1 : 0;
    P.nrs = (int)(nb / 2);
    P.ovl_chunks = c->ovl_chunks;
    P.ws = (multi && c->ws && bulk && !ovl && !c->dyn_ag) ? 1 : 0;
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)nb, (unsigned)p),
                                         dim3(THREADS), args, dsm, stream));
  } else {
    P.overlap = ovl ? 1 : 0;
    P.nrs = (int)(nb / 2);
    P.ovl_chunks = c->ovl_chunks;
    P.ws = (multi && c->ws && bulk && !ovl && !c->dyn_ag) ? 1 : 0;
    // pairs only for small (capped) grids: every cluster must be co-resident
    // (CTA b of every rank waits for the others), which 2-SM clusters on
    // partially floor-swept GPCs do not guarantee for a full-GPU grid
    const bool pairs = c->cluster2 && nb % 2 == 0 && nb <= 64;
    CUDA_TRY(launch_k(c->pdl, (const void*)k, dim3((unsigned)nb), dim3(THREADS), args, dsm, stream, pairs));
  }
  c->launches += 1;
  // real bytes pulled over NVLink by this rank
  if (!c->virt) {
    const int r = c->rank;
    int64_t in_bytes = 0;
    if (logp) {
      // halving moves n/2 + n/4 + ..., doubling the same again; +n for a fold partner
      int m = 1;
      while ((m << 1) <= p) m <<= 1;
      const int excess = p - m;
      const bool odd = r < 2 * excess && (r & 1), even = r < 2 * excess && !(r & 1);
      if (odd) in_bytes = L.n * (int64_t)sz;
      else in_bytes = 2 * (L.n - L.n / m) * (int64_t)sz + (even ? L.n * (int64_t)sz : 0);
    } else if (ll == 1) in_bytes = (int64_t)(p - 1) * ((L.n * (int64_t)sz + 7) / 8) * 16;
    else if (ll == 2) in_bytes = 2 * (int64_t)(p - 1) * ((maxseg * (int64_t)sz + 7) / 8) * 16;
    else if (L.oneshot) in_bytes = (int64_t)(p - 1) * L.n * sz;
    else {
      if (L.nbuf > 1 || L.srcmode == SRC_GATHER) {
        for (int k = 0; k < L.nbuf; ++k)
          for (int q = 0; q < p; ++q)
            in_bytes += (q == r ? (int64_t)(p - 1) : 1) * P.bseg_len[k][q] * (int64_t)sz;
      } else {
        if (L.phases & PH_RS) in_bytes += (int64_t)(p - 1) * len[r] * sz;
        if (L.phases & PH_AG)
          for (int q = 0; q < p; ++q)
            if (q != r) in_bytes += len[q] * sz;
      }
    }
    c->nvlink_in += in_bytes;
  }
  return CM_OK;
}

// Resolve send/recv placement for one call. Host buffers are bounced through
// the device scratch buffer with cudaMemcpyAsync (CUDA-aware MPI semantics).
struct Placement {
  int srcmode = SRC_COPYIN;
  const void* in = nullptr;
  void* out = nullptr;
  int64_t zc = 0;
  bool recv_host = false;
  bool send_host = false;   // send staged into `scratch` (H2D deferred when defer_host_copy)
};

// ---- automatic registration (the pointer cache's IPC side) ----------------
typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
typedef CUresult (*GetAttrFn)(void*, CUpointer_attribute, CUdeviceptr);

template <class F>
F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<F>(fn);
}

unsigned long long buffer_id_of(cm_comm* c, const void* ptr) {
  static GetAttrFn get_attr = driver_fn<GetAttrFn>("cuPointerGetAttribute");
  unsigned long long id = 0;
  c->auto_checks += 1;
  if (!get_attr || get_attr(&id, CU_POINTER_ATTRIBUTE_BUFFER_ID, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return 0;
  return id;
}

// Map the allocation slots peers have published since the last call (their
// kernels report the counts in c->areg_host[q]): read the mailbox entries over
// NVLink, open the IPC handles (cached), write AUTOTAB[slot][q] in my heap and
// acknowledge in the peer's heap. Synchronous on a private stream; runs only
// when a peer published something new.
int service_autoreg(cm_comm* c, cudaStream_t stream) {
  if (!c->areg_host) return CM_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return CM_OK;                    // mapped at the next eager call
  }
  for (int q = 0; q < c->size; ++q) {
    if (q == c->rank) continue;
    const int64_t n = (int64_t) reinterpret_cast<volatile unsigned long long*>(c->areg_host)[q];
    if (n <= c->mapped_seq[q]) continue;
    const int64_t lo = c->mapped_seq[q], cnt = std::min<int64_t>(n, MAXAUTO) - lo;
    if (cnt <= 0) continue;
    unsigned char* mb = c->areg_pin;
    unsigned long long* vals = reinterpret_cast<unsigned long long*>(c->areg_pin + MAXAUTO * MAILBOX_BYTES);
    CUDA_TRY(cudaMemcpyAsync(mb, c->heap[q] + MAILBOX_OFF + lo * MAILBOX_BYTES, cnt * MAILBOX_BYTES,
                             cudaMemcpyDeviceToHost, c->reg_stream));
    CUDA_TRY(cudaStreamSynchronize(c->reg_stream));
    for (int64_t i = 0; i < cnt; ++i) {
      const std::string key = std::to_string(q) + ":" +
                              std::string(reinterpret_cast<const char*>(mb + i * MAILBOX_BYTES), CM_IPC_HANDLE_BYTES);
      auto it = c->opened.find(key);
      char* base;
      if (it != c->opened.end()) {
        base = it->second;
      } else {
        cudaIpcMemHandle_t h;
        memcpy(&h, mb + i * MAILBOX_BYTES, sizeof h);
        void* mapped = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&mapped, h, cudaIpcMemLazyEnablePeerAccess));
        base = static_cast<char*>(mapped);
        c->opened[key] = base;
      }
      vals[i] = reinterpret_cast<unsigned long long>(base);
      CUDA_TRY(cudaMemcpyAsync(c->local + AUTOTAB_OFF + ((size_t)(lo + i) * MAXP + q) * 8, &vals[i], 8,
                               cudaMemcpyHostToDevice, c->reg_stream));
    }
    vals[MAXAUTO] = (unsigned long long)(lo + cnt);
    CUDA_TRY(cudaMemcpyAsync(c->heap[q] + ACK_OFF + (size_t)c->rank * 8, &vals[MAXAUTO], 8,
                             cudaMemcpyHostToDevice, c->reg_stream));
    CUDA_TRY(cudaStreamSynchronize(c->reg_stream));
    c->mapped_seq[q] = lo + cnt;
    c->auto_mapped += cnt;
  }
  return CM_OK;
}

// Mailbox slot of the allocation holding [ptr, ptr+bytes) (publishing it on
// first sight), or -1 if it cannot be shared (not cudaMalloc memory, or the
// mailbox is full). The allocation's buffer id is re-checked on every use so
// a freed and re-allocated range at the same address gets a new slot.
int64_t auto_slot(cm_comm* c, const void* ptr, int64_t bytes, bool may_publish) {
  static GetRangeFn get_range = driver_fn<GetRangeFn>("cuMemGetAddressRange");
  const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  const unsigned long long bid = buffer_id_of(c, ptr);
  auto it = c->autoregs.upper_bound(a);
  if (it != c->autoregs.begin()) {
    --it;
    if (a + (uintptr_t)bytes <= it->first + it->second.size && it->second.buffer_id == bid && bid)
      return it->second.slot;
    if (a < it->first + it->second.size) c->autoregs.erase(it);     // stale: the range was re-allocated
  }
  if (!may_publish) return -1;       // e.g. inside a CUDA-graph capture: no synchronous copies
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!get_range || !bid || get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return -1;
  if (a + (uintptr_t)bytes > (uintptr_t)base + size) return -1;
  cm_comm::AutoReg r{size, -1, bid};
  cudaIpcMemHandle_t h;
  if (c->reg_seq < MAXAUTO && cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) == cudaSuccess) {
    unsigned char* e = c->areg_pin;
    memset(e, 0, MAILBOX_BYTES);
    memcpy(e, &h, sizeof h);
    memcpy(e + 64, &size, 8);
    memcpy(e + 72, &bid, 8);
    memcpy(e + 80, &base, 8);     // own entry of the slot table: the kernels resolve every rank's record
    if (cudaMemcpyAsync(c->local + MAILBOX_OFF + (size_t)c->reg_seq * MAILBOX_BYTES, e, MAILBOX_BYTES,
                        cudaMemcpyHostToDevice, c->reg_stream) == cudaSuccess &&
        cudaMemcpyAsync(c->local + AUTOTAB_OFF + ((size_t)c->reg_seq * MAXP + c->rank) * 8, e + 80, 8,
                        cudaMemcpyHostToDevice, c->reg_stream) == cudaSuccess &&
        cudaStreamSynchronize(c->reg_stream) == cudaSuccess) {
      r.slot = c->reg_seq++;
      c->auto_published += 1;
    }
  }
  cudaGetLastError();
  c->autoregs[(uintptr_t)base] = r;
  return r.slot;
}

int place(cm_comm* c, const void* send, int64_t send_bytes, void* recv, int64_t recv_bytes,
          cudaStream_t stream, Placement* pl, bool peers_read_send = false, bool defer_host_copy = false) {
  int ks = CM_KIND_DEVICE, kr = CM_KIND_DEVICE;
  int st;
  if (send_bytes > 0 && (st = classify(c, send, &ks))) return st;
  if (recv_bytes > 0 && (st = classify(c, recv, &kr))) return st;
  pl->in = send;
  pl->out = recv;
  const int64_t need = std::max(send_bytes, recv_bytes);
  if ((ks == CM_KIND_HOST || kr == CM_KIND_HOST) && need > (int64_t)c->staging_bytes)
    return fail(CM_ERR_CONFIG, "host buffer larger than the device bounce buffer");
  if (ks == CM_KIND_HOST) {
    if (!defer_host_copy) CUDA_TRY(cudaMemcpyAsync(c->scratch, send, send_bytes, cudaMemcpyHostToDevice, stream));
    pl->in = c->scratch;
    pl->send_host = true;
  } else if (in_pool(c, send, send_bytes)) {
    pl->srcmode = SRC_ZEROCOPY;
    pl->zc = static_cast<const char*>(send) - c->local;
  } else if (!c->regs.empty() && send_bytes > 0) {
    // pointer cache: is the send buffer inside a collectively registered range?
    const uintptr_t a = reinterpret_cast<uintptr_t>(send);
    auto it = c->regs.upper_bound(a);
    if (it != c->regs.begin()) {
      --it;
      if (a + (uintptr_t)send_bytes <= it->first + (uintptr_t)it->second.bytes) {
        pl->srcmode = SRC_REGISTERED;
        pl->zc = (int64_t)(REG_FLAG | ((unsigned long long)it->second.id << 40) |
                           (unsigned long long)(a - it->first));
      }
    }
  }
  if (pl->srcmode == SRC_COPYIN && ks == CM_KIND_DEVICE && peers_read_send && c->auto_reg && c->areg_host &&
      send_bytes > 0) {
    // automatic registration: peers read this allocation in place once every
    // peer has mapped its mailbox slot; until then it is copied in
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cap);
    const int64_t slot = auto_slot(c, send, send_bytes, cap == cudaStreamCaptureStatusNone);
    const int64_t acked = (int64_t) reinterpret_cast<volatile unsigned long long*>(c->areg_host)[MAXP];
    if (slot >= 0 && slot < acked) {
      auto it = c->autoregs.upper_bound(reinterpret_cast<uintptr_t>(send));
      --it;
      pl->srcmode = SRC_REGISTERED;
      pl->zc = (int64_t)(REG_FLAG | AUTO_FLAG | ((unsigned long long)slot << 40) |
                         (unsigned long long)(reinterpret_cast<uintptr_t>(send) - it->first));
      c->auto_zc_calls += 1;
    }
  }
  if (kr == CM_KIND_HOST) {
    pl->out = c->scratch;
    pl->recv_host = true;
  }
  return CM_OK;
}

void count_stats(cm_comm* c, const cm_stats_t& s) {
  c->messages += s.messages_per_rank;
  c->bytes += s.bytes_sent_per_rank;
  c->calls += 1;
}

int identity_copy(cm_comm* c, const void* send, void* recv, int64_t bytes, cudaStream_t stream) {
  (void)c;
  if (bytes > 0 && send != recv) CUDA_TRY(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDefault, stream));
  return CM_OK;
}

// one-shot or two-shot for a concrete algorithm
void plan_algo(cm_comm* c, int concrete, int64_t nbytes, Launch* L) {
  const bool small = nbytes <= c->oneshot_max_bytes;
  if (concrete == CM_ALGO_RING) {
    L->order = ORD_RING;
    L->oneshot = 0;
    L->layout = CM_LAYOUT_RING;
  } else if (concrete == CM_ALGO_RHD) {
    L->order = ORD_TREE;
    L->oneshot = small ? 1 : 0;
    L->layout = CM_LAYOUT_RHD;
  } else {
    L->order = ORD_SEQ;
    L->oneshot = small ? 1 : 0;
    L->layout = CM_LAYOUT_RING;
  }
  L->phases = L->oneshot ? PH_RS : (PH_RS | PH_AG);
  const int64_t cap = c->ll_units * 8;      // LL payload bytes per source
  const int64_t ll2_max = c->ll2_max_bytes >= 0 ? c->ll2_max_bytes : (int64_t)c->size * cap;
  if (L->oneshot) {
    L->ll = nbytes <= std::min<int64_t>(c->ll_max_bytes, cap) ? 1 : 0;
  } else {
    // a segment of ceil(n/p) elements must fit one source's LL slot range
    const int64_t seg_bytes = (nbytes + c->size - 1) / c->size + 8;
    L->ll = (nbytes <= ll2_max && seg_bytes <= cap) ? 2 : 0;
  }
}

int host_allreduce_pieces(cm_comm* c, const Launch& L, const void* send, void* recv, bool recv_host, int K,
                          cudaStream_t stream);

int do_allreduce(cm_comm* c, const void* const* sends, void* const* recvs, int64_t count,
                 int dtype, int op, int algo, int64_t switch_bytes, int average, void* stream_,
                 cm_stats_t* stats) {
  int st = check_dtype_op(dtype, op);
  if (st) return st;
  if (count < 0) return fail(CM_ERR_SHAPE, "negative element count");
  if (average && (dtype == CM_INT32 || dtype == CM_INT64))
    return fail(CM_ERR_SHAPE, "averaging needs a floating-point dtype");
  if ((st = check_async_error(c))) return st;
  const int64_t sz = (int64_t)dtype_size(dtype), nbytes = count * sz;
  int concrete;
  if ((st = cm_resolve_algorithm(algo, nbytes, switch_bytes, &concrete))) return st;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int p = c->size;
  const int nloc = c->virt ? p : 1;
  for (int q = 0; q < nloc; ++q) {
    const int r = c->virt ? q : c->rank;
    cm_algo_stats(concrete, p, r, count, dtype, switch_bytes, &stats[q]);
    count_stats(c, stats[q]);
  }
  if (p == 1) {  // collectives.py:86-87,119-120,169-170: input returned as is
    return identity_copy(c, sends[0], recvs[0], nbytes, stream);
  }
  Launch L;
  L.n = count;
  L.dtype = dtype;
  L.op = op;
  L.average = average;
  plan_algo(c, concrete, nbytes, &L);
  Placement pl;
  if (!c->virt) {
    if ((st = service_autoreg(c, stream))) return st;
    const bool peers_read = !L.ll && !L.oneshot;    // the two-shot pull reads inputs in place
    const bool pieceable = c->host_split && peers_read && L.phases == (PH_RS | PH_AG);
    if ((st = place(c, sends[0], nbytes, recvs[0], nbytes, stream, &pl, peers_read, pieceable))) return st;
    if (pl.send_host && pieceable) {
      // host send buffer: H2D / collective / D2H in pieces (host_allreduce_pieces)
      const int K = (int)std::max<int64_t>(1, std::min<int64_t>(128, (nbytes + c->host_piece / 2) / c->host_piece));
      if (K > 1) {
        L.srcmode = SRC_COPYIN;
        L.in[0] = pl.in;
        L.out[0] = pl.out;
        return host_allreduce_pieces(c, L, sends[0], recvs[0], pl.recv_host, K, stream);
      }
      CUDA_TRY(cudaMemcpyAsync(c->scratch, sends[0], nbytes, cudaMemcpyHostToDevice, stream));
    }
    L.srcmode = pl.srcmode;
    L.in[0] = pl.in;
    L.out[0] = pl.out;
    L.zc_srcoff[0] = pl.zc;
  } else {
    for (int q = 0; q < p; ++q) { L.in[q] = sends[q]; L.out[q] = recvs[q]; }
  }
  // a one-shot pull kernel has no barrier after peers read my input, so user
  // buffers must not be read in place there: stage them
  if (L.oneshot && !L.ll && (L.srcmode == SRC_ZEROCOPY || L.srcmode == SRC_REGISTERED)) {
    L.srcmode = SRC_COPYIN;
  }
  if ((st = launch_collective(c, L, stream))) return st;
  if (pl.recv_host) CUDA_TRY(cudaMemcpyAsync(recvs[0], pl.out, nbytes, cudaMemcpyDeviceToHost, stream));
  return CM_OK;
}

int do_rs(cm_comm* c, const void* const* sends, void* const* recvs, int64_t count, int dtype,
          int op, int layout, void* stream_, cm_stats_t* stats) {
  int st = check_dtype_op(dtype, op);
  if (st) return st;
  if (count < 0) return fail(CM_ERR_SHAPE, "negative element count");
  if (layout != CM_LAYOUT_RING && layout != CM_LAYOUT_RHD) return fail(CM_ERR_CONFIG, "unknown layout");
  if ((st = check_async_error(c))) return st;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int p = c->size;
  const int64_t sz = (int64_t)dtype_size(dtype);
  int64_t off[MAXP], len[MAXP];
  cm_layout(layout, count, p, off, len);
  const int nloc = c->virt ? p : 1;
  for (int q = 0; q < nloc; ++q) {
    const int r = c->virt ? q : c->rank;
    cm_rs_stats(layout, p, r, count, dtype, &stats[q]);
    count_stats(c, stats[q]);
  }
  if (p == 1) return identity_copy(c, sends[0], recvs[0], count * sz, stream);
  Launch L;
  L.n = count;
  L.dtype = dtype;
  L.op = op;
  L.layout = layout;
  L.order = layout == CM_LAYOUT_RING ? ORD_RING : ORD_TREE;
  L.phases = PH_RS;
  L.out_rel = 1;
  Placement pl;
  if (!c->virt) {
    if ((st = service_autoreg(c, stream))) return st;
    if ((st = place(c, sends[0], count * sz, recvs[0], len[c->rank] * sz, stream, &pl, true))) return st;
    L.srcmode = pl.srcmode;
    L.in[0] = pl.in;
    L.out[0] = pl.out;
    L.zc_srcoff[0] = pl.zc;
  } else {
    for (int q = 0; q < p; ++q) { L.in[q] = sends[q]; L.out[q] = recvs[q]; }
  }
  if ((st = launch_collective(c, L, stream))) return st;
  if (pl.recv_host)
    CUDA_TRY(cudaMemcpyAsync(recvs[0], pl.out, len[c->rank] * sz, cudaMemcpyDeviceToHost, stream));
  return CM_OK;
}

int do_ag(cm_comm* c, const void* const* sends, void* const* recvs, int64_t count, int dtype,
          int layout, void* stream_, cm_stats_t* stats) {
  int st = check_dtype_op(dtype, CM_SUM);
  if (st) return st;
  if (count < 0) return fail(CM_ERR_SHAPE, "negative element count");
  if (layout != CM_LAYOUT_RING && layout != CM_LAYOUT_RHD) return fail(CM_ERR_CONFIG, "unknown layout");
  if ((st = check_async_error(c))) return st;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int p = c->size;
  const int64_t sz = (int64_t)dtype_size(dtype);
  int64_t off[MAXP], len[MAXP];
  cm_layout(layout, count, p, off, len);
  const int nloc = c->virt ? p : 1;
  for (int q = 0; q < nloc; ++q) {
    const int r = c->virt ? q : c->rank;
    cm_ag_stats(layout, p, r, count, dtype, &stats[q]);
    count_stats(c, stats[q]);
  }
  if (p == 1) return identity_copy(c, sends[0], recvs[0], count * sz, stream);
  Launch L;
  L.n = count;
  L.dtype = dtype;
  L.op = CM_SUM;
  L.layout = layout;
  L.order = ORD_SEQ;
  L.phases = PH_AG;
  L.ag_in_rel = 1;
  Placement pl;
  if (!c->virt) {
    if ((st = service_autoreg(c, stream))) return st;
    if ((st = place(c, sends[0], len[c->rank] * sz, recvs[0], count * sz, stream, &pl, true))) return st;
    L.srcmode = pl.srcmode;
    L.in[0] = pl.in;
    L.out[0] = pl.out;
    L.zc_srcoff[0] = pl.zc;
  } else {
    for (int q = 0; q < p; ++q) { L.in[q] = sends[q]; L.out[q] = recvs[q]; }
  }
  if ((st = launch_collective(c, L, stream))) return st;
  if (pl.recv_host)
    CUDA_TRY(cudaMemcpyAsync(recvs[0], pl.out, count * sz, cudaMemcpyDeviceToHost, stream));
  return CM_OK;
}

bool g_bulk_copy_default = true;   // cm_batched_copy without a communicator (fuse/unfuse)

int launch_batched_copy(cm_comm* c, int n, const void* const* srcs, void* const* dsts,
                        const int64_t* nbytes, bool staged, cudaStream_t stream, char* heap = nullptr) {
  for (int base = 0; base < n; base += MAXCOPY) {
    const int m = std::min(MAXCOPY, n - base);
    CopyParams P;
    memset(&P, 0, sizeof P);
    P.n = m;
    P.start[0] = 0;
    for (int i = 0; i < m; ++i) {
      P.src[i] = static_cast<const char*>(srcs[base + i]);
      P.dst[i] = static_cast<char*>(dsts[base + i]);
      P.start[i + 1] = P.start[i] + nbytes[base + i];
    }
    if (P.start[m] == 0) continue;
    P.staged = staged ? 1 : 0;
    if (c) {
      P.heap = heap ? heap : c->local;      // staged: whose staging (virtual ranks share one process)
      P.staging_bytes = (long long)c->staging_bytes;
      P.staging_off = (long long)c->staging_off;
    }
    // TMA bulk-copy engine when every piece is 16-byte aligned (addresses and sizes)
    bool aligned = P.start[m] >= (256 << 10) && (c ? c->bulk_copy : g_bulk_copy_default);
    for (int i = 0; i < m && aligned; ++i)
      aligned = ((((uintptr_t)P.src[i]) | ((uintptr_t)P.dst[i]) | (uintptr_t)nbytes[base + i]) & 15u) == 0;
    if (aligned) {
      int dev = 0, avail = 0;
      CUDA_TRY(cudaGetDevice(&dev));
      int st = dyn_smem_optin(dev, (const void*)bulk_copy_kernel, &avail, (int)BULK_SMEM);
      if (st) return st;
      const int sms = c ? c->sms : 148;
      int64_t nb = (P.start[m] + 4 * BULK_CHUNK - 1) / (4 * BULK_CHUNK);
      nb = std::max<int64_t>(1, std::min<int64_t>(nb, 2 * (int64_t)sms));
      void* args[] = {&P};
      ProfScope prof_scope(c, stream, 1, 2 * P.start[m]);
      CUDA_TRY(launch_k(c ? c->pdl : true, (const void*)bulk_copy_kernel, dim3((unsigned)nb), dim3(BULK_THREADS),
                        args, BULK_SMEM, stream));
      if (c) c->launches += 1;
      continue;
    }
    // `pack_waves` waves of 512-thread CTAs (4 resident per SM) for large packs
    const int sms = c ? c->sms : 148;
    const int waves = c ? c->pack_waves : 2;
    int64_t nb = (P.start[m] + (64 << 10) - 1) / (64 << 10);
    nb = std::max<int64_t>(1, std::min<int64_t>(nb, (int64_t)sms * 4 * waves));
    if (c && c->pack_max_ctas > 0) nb = std::min<int64_t>(nb, c->pack_max_ctas);
    void* args[] = {&P};
    ProfScope prof_scope(c, stream, 1, 2 * P.start[m]);
    const void* kfn = (c && c->pack_unroll == 8) ? (const void*)batched_copy_kernel<8> : (const void*)batched_copy_kernel<4>;
    CUDA_TRY(launch_k(c ? c->pdl : true, kfn, dim3((unsigned)nb), dim3(THREADS), args, 0, stream));
    if (c) c->launches += 1;
  }
  return CM_OK;
}

// Consecutive members whose sources are adjacent in memory (a flat gradient
// buffer viewed as tensors) become one copy: {source, offset in the fused
// layout, bytes}, cut into pieces of at most `piece` bytes.
struct Run {
  const char* src;
  int64_t off, bytes;
};

std::vector<Run> coalesce(const void* const* srcs, const int64_t* bytes, int n, int64_t piece) {
  std::vector<Run> runs;
  int64_t off = 0;
  for (int k = 0; k < n; ++k) {
    const char* s = static_cast<const char*>(srcs[k]);
    if (bytes[k] > 0) {
      if (!runs.empty() && runs.back().src + runs.back().bytes == s && runs.back().off + runs.back().bytes == off)
        runs.back().bytes += bytes[k];
      else
        runs.push_back(Run{s, off, bytes[k]});
    }
    off += bytes[k];
  }
  std::vector<Run> out;
  for (const Run& r : runs)
    for (int64_t a = 0; a < r.bytes; a += piece) out.push_back(Run{r.src + a, r.off + a, std::min(piece, r.bytes - a)});
  return out;
}

// Piece boundaries over [0, total) for the single-rank host pipeline: pieces
// of `piece` bytes, ramped piece/8, /4, /2 at both ends so the first D2H starts
// after a small H2D and the last D2H after a small one (pipeline fill and
// drain ~1/8 of a uniform piece); short totals get eight even pieces.
std::vector<int64_t> graded_cuts(int64_t total, int64_t piece) {
  std::vector<int64_t> cuts;
  const int64_t ramp[3] = {piece / 8, piece / 4, piece / 2};
  const int64_t head = ramp[0] + ramp[1] + ramp[2];
  if (total <= 2 * head + piece) {
    const int64_t q = std::max<int64_t>(64 << 10, (total + 7) / 8);
    for (int64_t a = q; a < total; a += q) cuts.push_back(a);
    cuts.push_back(total);
    return cuts;
  }
  int64_t a = 0;
  for (int64_t r : ramp) cuts.push_back(a += r);
  const int64_t mid_end = total - head;
  while (a + 2 * piece <= mid_end) cuts.push_back(a += piece);
  if (a < mid_end) cuts.push_back(a = mid_end);
  for (int i = 2; i >= 0; --i) cuts.push_back(a += ramp[i]);
  return cuts;
}

// runs (sorted by offset, disjoint) split at the given offsets
std::vector<Run> split_runs(const std::vector<Run>& runs, const std::vector<int64_t>& cuts) {
  std::vector<Run> out;
  for (const Run& r : runs) {
    int64_t a = r.off;
    const int64_t end = r.off + r.bytes;
    auto it = std::upper_bound(cuts.begin(), cuts.end(), a);
    while (a < end) {
      const int64_t b = (it == cuts.end()) ? end : std::min(end, *it);
      out.push_back(Run{r.src + (a - r.off), a, b - a});
      a = b;
      if (it != cuts.end() && *it <= a) ++it;
    }
  }
  return out;
}

// Host-memory aggregate pipeline (CUDA-aware semantics for host gradients).
// Stream roles: h2d copies inputs into `indev`, the caller's stream runs the
// collectives, d2h copies results out of `outdev`. Every hand-off is an
// event, so H2D of group g+1 and D2H of group g run concurrently (PCIe is
// full duplex) and overlap the NVLink collectives; the caller's stream joins
// both copy streams before the call returns (stream-ordered semantics kept).
struct HostPipe {
  cm_comm* c;
  cudaStream_t main;
  bool active = false;
  size_t next_ev = 0;
  explicit HostPipe(cm_comm* c_, cudaStream_t s) : c(c_), main(s) {}
  int ev(cudaEvent_t* out) {
    if (next_ev == c->sync_events.size()) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->sync_events.push_back(e);
    }
    *out = c->sync_events[next_ev++];
    return CM_OK;
  }
  // order `to` after everything queued so far on `from`
  int link(cudaStream_t from, cudaStream_t to) {
    cudaEvent_t e;
    int st = ev(&e);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(e, from));
    CUDA_TRY(cudaStreamWaitEvent(to, e, 0));
    return CM_OK;
  }
  static int grow(char** buf, int64_t* have, int64_t need) {
    if (*have >= need) return CM_OK;
    if (*buf) {
      CUDA_TRY(cudaDeviceSynchronize());
      CUDA_TRY(cudaFree(*buf));
      *buf = nullptr;
      *have = 0;
    }
    CUDA_TRY(cudaMalloc(buf, need));
    *have = need;
    return CM_OK;
  }
  int start(int64_t in_bytes, int64_t out_bytes) {
    if (!c->h2d) CUDA_TRY(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    if (!c->d2h) CUDA_TRY(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    int st;
    if ((st = grow(&c->indev, &c->indev_bytes, std::max<int64_t>(in_bytes, 1)))) return st;
    if ((st = grow(&c->outdev, &c->outdev_bytes, std::max<int64_t>(out_bytes, 1)))) return st;
    // copy streams start after all earlier work of the caller's stream (which
    // produced device inputs and last read indev/outdev)
    if ((st = link(main, c->h2d))) return st;
    if ((st = link(main, c->d2h))) return st;
    active = true;
    return CM_OK;
  }
  int join() {
    if (!active) return CM_OK;
    active = false;
    int st;
    if ((st = link(c->h2d, main))) return st;
    return link(c->d2h, main);
  }
  ~HostPipe() { join(); }
};

// allreduce() of a host send buffer at p > 1: the K pieces of segments_of move
// H2D (h2d stream, queued up front) -> collective (caller's stream, after
// the piece's event) -> D2H (d2h stream) so the two PCIe directions and the
// collective overlap; every element keeps the owner and fold order of the
// one-launch allreduce. L is the planned launch with `scratch` as in/out.
int host_allreduce_pieces(cm_comm* c, const Launch& L, const void* send, void* recv, bool recv_host, int K,
                          cudaStream_t stream) {
  const int p = c->size;
  const int64_t sz = (int64_t)dtype_size(L.dtype);
  HostPipe hp(c, stream);
  int st;
  if ((st = hp.start(0, 0))) return st;
  std::vector<cudaEvent_t> ready(K);
  int64_t off[MAXP], len[MAXP];
  for (int k = 0; k < K; ++k) {
    segments_of(L.n, p, L.layout, k, K, off, len);
    for (int q = 0; q < p; ++q)
      if (len[q] > 0)
        CUDA_TRY(cudaMemcpyAsync(c->scratch + off[q] * sz, static_cast<const char*>(send) + off[q] * sz,
                                 len[q] * sz, cudaMemcpyHostToDevice, c->h2d));
    if ((st = hp.ev(&ready[k]))) return st;
    CUDA_TRY(cudaEventRecord(ready[k], c->h2d));
  }
  for (int k = 0; k < K; ++k) {
    CUDA_TRY(cudaStreamWaitEvent(stream, ready[k], 0));
    Launch Lk = L;
    Lk.piece = k;
    Lk.npieces = K;
    if ((st = launch_collective(c, Lk, stream))) return st;
    if (recv_host) {
      if ((st = hp.link(stream, c->d2h))) return st;
      segments_of(L.n, p, L.layout, k, K, off, len);
      for (int q = 0; q < p; ++q)
        if (len[q] > 0)
          CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + off[q] * sz, static_cast<char*>(L.out[0]) + off[q] * sz,
                                   len[q] * sz, cudaMemcpyDeviceToHost, c->d2h));
    }
  }
  return hp.join();
}

}  // namespace

extern "C" {

int cm_comm_create(int rank, int size, int device, int64_t staging_bytes, int64_t pool_bytes,
                   cm_comm_t** out) {
  if (size < 1 || size > MAXP) return fail(CM_ERR_INVALID_GROUP, "group size must be in 1.." + std::to_string(MAXP));
  if (rank < 0 || rank >= size) return fail(CM_ERR_INVALID_GROUP, "rank outside group");
  if (staging_bytes < 0 || pool_bytes < 0) return fail(CM_ERR_VALUE, "negative size");
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new cm_comm();
  c->rank = rank;
  c->size = size;
  c->device = device;
  c->staging_bytes = round_up(std::max<int64_t>(staging_bytes, 1), HEAP_ALIGN);
  c->pool_bytes = round_up((size_t)pool_bytes, HEAP_ALIGN);
  c->ll_units = CM_LL_UNITS_REAL;
  c->staging_off = round_up(LL_OFF + 4 * (size_t)size * (size_t)c->ll_units * 16, HEAP_ALIGN);
  c->heap_bytes = c->staging_off + 2 * c->staging_bytes + c->pool_bytes;
  c->reg.policy = CM_LAZY_CACHE;
  c->reg.simulated = false;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMalloc(&c->local, c->heap_bytes);
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "cudaMalloc(heap)"); }
  e = cudaMemset(c->local, 0, CTRL_REGION);
  if (e == cudaSuccess) e = cudaMalloc(&c->scratch, c->staging_bytes);
  if (e == cudaSuccess) e = cudaHostAlloc(&c->herr_host, sizeof(unsigned), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&c->herr_dev, c->herr_host, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { cm_comm_destroy(c); return cuda_fail(e, "cm_comm_create"); }
  *c->herr_host = 0;
  c->heap[rank] = c->local;
  if (c->pool_bytes) c->pool_free[c->staging_off + 2 * c->staging_bytes] = c->pool_bytes;
  if (size == 1) c->connected = true;
  *out = c;
  return CM_OK;
}

int cm_comm_ipc_handle(cm_comm_t* c, void* handle_out) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "virtual groups have no IPC handle");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->local));
  static_assert(sizeof(h) == CM_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof h);
  return CM_OK;
}

int cm_comm_connect(cm_comm_t* c, const void* all_handles) {
  if (c->virt) return CM_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const char* hs = static_cast<const char*>(all_handles);
  for (int q = 0; q < c->size; ++q) {
    if (q == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, hs + (size_t)q * CM_IPC_HANDLE_BYTES, sizeof h);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, ("cudaIpcOpenMemHandle(peer " + std::to_string(q) + ")").c_str());
    c->heap[q] = static_cast<char*>(ptr);
  }
  if (c->size > 1) {
    CUDA_TRY(cudaHostAlloc(&c->areg_host, (MAXP + 1) * sizeof(unsigned long long), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer((void**)&c->areg_dev, c->areg_host, 0));
    memset(c->areg_host, 0, (MAXP + 1) * sizeof(unsigned long long));
    CUDA_TRY(cudaHostAlloc(&c->areg_pin, MAXAUTO * MAILBOX_BYTES + (MAXAUTO + 1) * 8, cudaHostAllocDefault));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->reg_stream, cudaStreamNonBlocking));
  }
  c->connected = true;
  return CM_OK;
}

int cm_comm_create_virtual(int size, int device, int64_t staging_bytes, cm_comm_t** out) {
  if (size < 1 || size > MAXP) return fail(CM_ERR_INVALID_GROUP, "group size must be in 1.." + std::to_string(MAXP));
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new cm_comm();
  c->virt = true;
  c->size = size;
  c->device = device;
  c->staging_bytes = round_up(std::max<int64_t>(staging_bytes, 1), HEAP_ALIGN);
  c->ll_units = CM_LL_UNITS_VIRTUAL;
  c->staging_off = round_up(LL_OFF + 4 * (size_t)size * (size_t)c->ll_units * 16, HEAP_ALIGN);
  c->heap_bytes = c->staging_off + 2 * c->staging_bytes;
  c->reg.policy = CM_LAZY_CACHE;
  c->reg.simulated = false;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMalloc(&c->local, c->heap_bytes * size);
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "cudaMalloc(virtual heaps)"); }
  for (int q = 0; q < size && e == cudaSuccess; ++q) {
    c->heap[q] = c->local + c->heap_bytes * q;
    e = cudaMemset(c->heap[q], 0, CTRL_REGION);
  }
  if (e == cudaSuccess) e = cudaHostAlloc(&c->herr_host, sizeof(unsigned), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&c->herr_dev, c->herr_host, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { cm_comm_destroy(c); return cuda_fail(e, "cm_comm_create_virtual"); }
  *c->herr_host = 0;
  c->connected = true;
  *out = c;
  return CM_OK;
}

int cm_comm_destroy(cm_comm_t* c) {
  if (!c) return CM_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (!c->virt)
    for (int q = 0; q < c->size; ++q)
      if (q != c->rank && c->heap[q]) cudaIpcCloseMemHandle(c->heap[q]);
  for (auto& kv : c->opened) cudaIpcCloseMemHandle(kv.second);
  for (auto& kv : c->gtabs) cudaFree(kv.second);
  if (c->local) cudaFree(c->local);
  if (c->scratch) cudaFree(c->scratch);
  if (c->agree_in) cudaFree(c->agree_in);
  if (c->areg_host) cudaFreeHost(c->areg_host);
  if (c->areg_pin) cudaFreeHost(c->areg_pin);
  if (c->reg_stream) cudaStreamDestroy(c->reg_stream);
  if (c->indev) cudaFree(c->indev);
  if (c->outdev) cudaFree(c->outdev);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  for (auto e : c->sync_events) cudaEventDestroy(e);
  if (c->herr_host) cudaFreeHost(c->herr_host);
  if (c->agree_host) cudaFreeHost(c->agree_host);
  for (auto& pr : c->prof) { cudaEventDestroy(pr.e0); cudaEventDestroy(pr.e1); }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  cudaGetLastError();
  delete c;
  return CM_OK;
}

int cm_comm_rank(cm_comm_t* c, int* rank) { *rank = c->rank; return CM_OK; }
int cm_comm_size(cm_comm_t* c, int* size) { *size = c->size; return CM_OK; }

int cm_comm_set_timeout(cm_comm_t* c, double seconds) {
  if (!(seconds > 0)) return fail(CM_ERR_VALUE, "timeout must be positive");
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, c->device);
  if (khz <= 0) khz = 2000000;
  c->timeout_cycles = (unsigned long long)(seconds * khz * 1e3);
  return CM_OK;
}

int cm_comm_set_policy(cm_comm_t* c, int policy) {
  if (policy < CM_NO_CACHE || policy > CM_INTERCEPT_CACHE) return fail(CM_ERR_VALUE, "unknown policy");
  std::lock_guard<std::mutex> g(c->reg.mu);
  c->reg.policy = policy;
  c->reg.cache.clear();
  return CM_OK;
}

int cm_comm_registry(cm_comm_t* c, cm_registry_t** reg) {
  *reg = reinterpret_cast<cm_registry_t*>(&c->reg);
  return CM_OK;
}

int cm_comm_set_param(cm_comm_t* c, const char* key, int64_t value) {
  const std::string k(key);
  if (value <= 0) return fail(CM_ERR_VALUE, "parameter must be positive");
  if (k == "oneshot_max_bytes") c->oneshot_max_bytes = value;
  else if (k == "ll_max_bytes") c->ll_max_bytes = value;
  else if (k == "ll_units_per_cta") c->ll_units_per_cta = value;
  else if (k == "ll2_max_bytes") c->ll2_max_bytes = value;
  else if (k == "ll2_units_per_cta") c->ll2_units_per_cta = value;
  else if (k == "stream_chunk") c->stream_chunk = value == 1 ? 0 : ((value + 63) / 64) * 64;
  else if (k == "multi_buffer") c->multi_buffer = value > 1 ? 1 : 0;
  else if (k == "rhd_logp") c->rhd_logp = value > 1 ? 1 : 0;
  else if (k == "bulk_copy") c->bulk_copy = value > 1 ? 1 : 0;
  else if (k == "bulk_rs") c->bulk_rs = value == 1 ? 0 : (int)std::min<int64_t>(value, RS_MAX_STAGES);
  else if (k == "dyn_ag") c->dyn_ag = value > 1 ? 1 : 0;
  else if (k == "inline_agree") c->inline_agree = value > 1 ? 1 : 0;
  else if (k == "auto_register") c->auto_reg = value > 1 ? 1 : 0;
  else if (k == "overlap") c->overlap = value > 1 ? 1 : 0;
  else if (k == "overlap_chunks") c->ovl_chunks = (int)std::min<int64_t>(value, 1 << 20);
  else if (k == "ws") c->ws = value > 1 ? 1 : 0;
  else if (k == "pack_waves") c->pack_waves = (int)std::min<int64_t>(value, 64);
  else if (k == "pack_max_ctas") c->pack_max_ctas = value <= 1 ? 0 : (int)std::min<int64_t>(value, 4096);
  else if (k == "pack_unroll") c->pack_unroll = value >= 8 ? 8 : 4;
  else if (k == "host_split") c->host_split = value > 1;
  else if (k == "host_piece_kb") c->host_piece = std::max<int64_t>(64, std::min<int64_t>(value, 1 << 20)) * 1024;
  else if (k == "pdl") c->pdl = value > 1;
  else if (k == "cluster_pairs") c->cluster2 = value > 1;
  else if (k == "host_chunk_kb") c->host_chunk = std::max<int64_t>(64, value) * 1024;
  else if (k == "bulk_stage_kb") c->bulk_stage = (int)std::max<int64_t>(4, std::min<int64_t>(value, 112)) * 1024;
  else if (k == "oneshot_bytes_per_cta") c->oneshot_bytes_per_cta = value;
  else if (k == "twoshot_bytes_per_cta") c->twoshot_bytes_per_cta = value;
  else if (k == "max_ctas") c->max_ctas = (int)std::min<int64_t>(value, MAXBLK);
  else return fail(CM_ERR_CONFIG, "unknown parameter " + k);
  return CM_OK;
}

int cm_comm_get_param(cm_comm_t* c, const char* key, int64_t* value) {
  const std::string k(key);
  if (k == "oneshot_max_bytes") *value = c->oneshot_max_bytes;
  else if (k == "ll_max_bytes") *value = c->ll_max_bytes;
  else if (k == "ll_units_per_cta") *value = c->ll_units_per_cta;
  else if (k == "ll2_max_bytes") *value = c->ll2_max_bytes;
  else if (k == "ll2_units_per_cta") *value = c->ll2_units_per_cta;
  else if (k == "stream_chunk") *value = c->stream_chunk;
  else if (k == "multi_buffer") *value = c->multi_buffer ? 2 : 1;
  else if (k == "rhd_logp") *value = c->rhd_logp ? 2 : 1;
  else if (k == "bulk_copy") *value = c->bulk_copy ? 2 : 1;
  else if (k == "bulk_rs") *value = c->bulk_rs ? c->bulk_rs : 1;
  else if (k == "dyn_ag") *value = c->dyn_ag ? 2 : 1;
  else if (k == "inline_agree") *value = c->inline_agree ? 2 : 1;
  else if (k == "auto_register") *value = c->auto_reg ? 2 : 1;
  else if (k == "overlap") *value = c->overlap ? 2 : 1;
  else if (k == "overlap_chunks") *value = c->ovl_chunks;
  else if (k == "ws") *value = c->ws ? 2 : 1;
  else if (k == "pack_waves") *value = c->pack_waves;
  else if (k == "pack_max_ctas") *value = c->pack_max_ctas ? c->pack_max_ctas : 1;
  else if (k == "pack_unroll") *value = c->pack_unroll;
  else if (k == "host_split") *value = c->host_split ? 2 : 1;
  else if (k == "host_piece_kb") *value = c->host_piece / 1024;
  else if (k == "pdl") *value = c->pdl ? 2 : 1;
  else if (k == "cluster_pairs") *value = c->cluster2 ? 2 : 1;
  else if (k == "auto_published") *value = c->auto_published;
  else if (k == "auto_mapped") *value = c->auto_mapped;
  else if (k == "auto_zero_copy_calls") *value = c->auto_zc_calls;
  else if (k == "auto_buffer_checks") *value = c->auto_checks;
  else if (k == "bulk_stage_kb") *value = c->bulk_stage / 1024;
  else if (k == "host_chunk_kb") *value = c->host_chunk / 1024;
  else if (k == "oneshot_bytes_per_cta") *value = c->oneshot_bytes_per_cta;
  else if (k == "twoshot_bytes_per_cta") *value = c->twoshot_bytes_per_cta;
  else if (k == "max_ctas") *value = c->max_ctas;
  else if (k == "staging_bytes") *value = (int64_t)c->staging_bytes;
  else if (k == "ll_payload_per_source") *value = c->ll_units * 8;
  else if (k == "pool_bytes") *value = (int64_t)c->pool_bytes;
  else return fail(CM_ERR_CONFIG, "unknown parameter " + k);
  return CM_OK;
}

int cm_comm_alloc(cm_comm_t* c, int64_t bytes, void** ptr) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "virtual groups have no symmetric pool");
  if (bytes <= 0) return fail(CM_ERR_VALUE, "allocation size must be positive");
  const size_t need = round_up((size_t)bytes, 512);
  for (auto it = c->pool_free.begin(); it != c->pool_free.end(); ++it) {
    if (it->second >= need) {
      const size_t off = it->first, rest = it->second - need;
      c->pool_free.erase(it);
      if (rest) c->pool_free[off + need] = rest;
      c->pool_used[off] = need;
      *ptr = c->local + off;
      return CM_OK;
    }
  }
  return fail(CM_ERR_CONFIG, "symmetric pool exhausted (" + std::to_string(bytes) + " B requested)");
}

int cm_comm_free(cm_comm_t* c, void* ptr) {
  const size_t off = static_cast<char*>(ptr) - c->local;
  auto it = c->pool_used.find(off);
  if (it == c->pool_used.end()) return fail(CM_ERR_INVALID_HANDLE, "free of unknown symmetric buffer");
  size_t o = off, len = it->second;
  c->pool_used.erase(it);
  auto nx = c->pool_free.lower_bound(o);
  if (nx != c->pool_free.end() && nx->first == o + len) { len += nx->second; c->pool_free.erase(nx); }
  auto pv = c->pool_free.lower_bound(o);
  if (pv != c->pool_free.begin()) {
    --pv;
    if (pv->first + pv->second == o) { o = pv->first; len += pv->second; c->pool_free.erase(pv); }
  }
  c->pool_free[o] = len;
  return CM_OK;
}

int cm_comm_export(cm_comm_t* c, const void* ptr, int64_t bytes, void* handle_out, int64_t* offset) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "virtual groups do not register buffers");
  static CUresult (*get_range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      cudaGetLastError();
      return fail(CM_ERR_UNSUPPORTED, "cuMemGetAddressRange unavailable");
    }
    get_range = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(CM_ERR_UNKNOWN_BUFFER, "not device memory of this process (cuMemGetAddressRange)");
  if (reinterpret_cast<uintptr_t>(ptr) + (uintptr_t)bytes > (uintptr_t)base + size)
    return fail(CM_ERR_SHAPE, "buffer crosses the end of its allocation");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle_out, &h, sizeof h);
  *offset = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - (uintptr_t)base);
  return CM_OK;
}

int cm_comm_register(cm_comm_t* c, const void* ptr, int64_t bytes, const void* all_handles,
                     const int64_t* all_offsets, int64_t* reg_id) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "virtual groups do not register buffers");
  if (c->next_reg >= MAXREG) return fail(CM_ERR_CONFIG, "registered-buffer table is full");
  const int p = c->size;
  char* table[MAXP] = {};
  const char* hs = static_cast<const char*>(all_handles);
  for (int q = 0; q < p; ++q) {
    if (q == c->rank) { table[q] = static_cast<char*>(const_cast<void*>(ptr)); continue; }
    const std::string key = std::to_string(q) + ":" + std::string(hs + (size_t)q * CM_IPC_HANDLE_BYTES, CM_IPC_HANDLE_BYTES);
    auto it = c->opened.find(key);
    char* base;
    if (it != c->opened.end()) {
      base = it->second;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, hs + (size_t)q * CM_IPC_HANDLE_BYTES, sizeof h);
      void* mapped = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&mapped, h, cudaIpcMemLazyEnablePeerAccess));
      base = static_cast<char*>(mapped);
      c->opened[key] = base;
    }
    table[q] = base + all_offsets[q];
  }
  const int64_t id = c->next_reg++;
  CUDA_TRY(cudaMemcpy(c->local + REG_OFF + (size_t)id * MAXP * 8, table, sizeof(char*) * MAXP,
                      cudaMemcpyHostToDevice));
  c->regs[reinterpret_cast<uintptr_t>(ptr)] = cm_comm::Reg{bytes, id};
  // the pointer cache now knows this range (intercept-style insert)
  c->reg.register_range(reinterpret_cast<uint64_t>(ptr), bytes, CM_KIND_DEVICE);
  *reg_id = id;
  return CM_OK;
}

// virtual group: every local rank's buffer under one id (the registered-buffer
// table of every virtual rank's heap holds all of them; no IPC involved)
int cm_comm_register_v(cm_comm_t* c, const void* const* ptrs, int64_t bytes, int64_t* reg_id) {
  if (!c->virt) return fail(CM_ERR_UNSUPPORTED, "cm_comm_register_v needs a virtual group");
  if (c->next_reg >= MAXREG) return fail(CM_ERR_CONFIG, "registered-buffer table is full");
  if (bytes < 0) return fail(CM_ERR_VALUE, "negative size");
  const char* table[MAXP] = {};
  for (int q = 0; q < c->size; ++q) table[q] = static_cast<const char*>(ptrs[q]);
  const int64_t id = c->next_reg++;
  for (int q = 0; q < c->size; ++q)
    CUDA_TRY(cudaMemcpy(c->heap[q] + REG_OFF + (size_t)id * MAXP * 8, table, sizeof(char*) * MAXP,
                        cudaMemcpyHostToDevice));
  *reg_id = id;
  return CM_OK;
}

int cm_comm_deregister(cm_comm_t* c, const void* ptr) {
  auto it = c->regs.find(reinterpret_cast<uintptr_t>(ptr));
  if (it == c->regs.end()) return fail(CM_ERR_INVALID_HANDLE, "buffer is not registered");
  c->regs.erase(it);
  c->reg.unregister_range(reinterpret_cast<uint64_t>(ptr));
  return CM_OK;
}

int cm_buffer_ids(cm_comm_t* c, int n, const void* const* ptrs, uint64_t* ids) {
  if (n < 0 || (n > 0 && (!ptrs || !ids))) return fail(CM_ERR_VALUE, "bad arguments");
  for (int i = 0; i < n; ++i) ids[i] = buffer_id_of(c, ptrs[i]);
  return CM_OK;
}

int cm_comm_sync(cm_comm_t* c, void* stream) {
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return check_async_error(c);
}

int cm_comm_poll(cm_comm_t* c) { return check_async_error(c); }

}  // extern "C"

// Element-wise MAX over ranks of n int64 host values, synchronously: the
// control-plane primitive behind negotiate_ready's fast path (one one-shot
// kernel over NVLink instead of a host gather/broadcast).
namespace {
// Agreement words in mapped pinned memory (int64 indices):
//   AGH_RES + 8*lr   cm_agree maxima of local rank lr
//   AGH_DONE + lr    completion ticket of the LL agreement kernel (per local rank)
//   AGH_INL + 2*lr   inline agreement {ticket, ok} written by CTA 0 of the first collective
//   AGH_IN + 8*lr    staging of the virtual ranks' agreement inputs
constexpr int AGH_RES = 0, AGH_DONE = 8 * MAXP, AGH_INL = 9 * MAXP, AGH_IN = 11 * MAXP, AGH_WORDS = 19 * MAXP;

int ensure_agree_buf(cm_comm* c) {
  if (!c->agree_host) {
    CUDA_TRY(cudaHostAlloc(&c->agree_host, AGH_WORDS * sizeof(int64_t), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer((void**)&c->agree_dev, c->agree_host, 0));
    memset(c->agree_host, 0, AGH_WORDS * sizeof(int64_t));
  }
  if (c->virt && !c->agree_in) CUDA_TRY(cudaMalloc(&c->agree_in, 8 * MAXP * sizeof(int64_t)));
  return CM_OK;
}

// host spin on a mapped completion word (bounded; device errors end it early)
int spin_ticket(cm_comm* c, int64_t idx, unsigned long long ticket, cudaStream_t stream, const char* what) {
  volatile unsigned long long* flag = reinterpret_cast<volatile unsigned long long*>(c->agree_host + idx);
  const auto t0 = std::chrono::steady_clock::now();
  while (*flag != ticket) {
    if (*reinterpret_cast<volatile unsigned*>(c->herr_host)) break;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) {
      cudaError_t e = cudaStreamQuery(stream);
      if (e != cudaErrorNotReady && e != cudaSuccess) return cuda_fail(e, what);
      return fail(CM_ERR_TRANSPORT, std::string(what) + ": peers did not answer within 60 s");
    }
  }
  return check_async_error(c);
}

// inline agreement: CTA 0 of the first collective of every local rank writes
// {ticket, ok} right after its start barrier
int inline_agree_wait(cm_comm* c, unsigned long long ticket, cudaStream_t stream, int* agreed) {
  const int nloc = c->virt ? c->size : 1;
  for (int lr = 0; lr < nloc; ++lr) {
    int st = spin_ticket(c, AGH_INL + 2 * lr, ticket, stream, "aggregate agreement");
    if (st) return st;
    agreed[lr] = reinterpret_cast<volatile int64_t*>(c->agree_host)[AGH_INL + 2 * lr + 1] ? 1 : 0;
  }
  return CM_OK;
}

// launch half of cm_agree: an LL one-shot MAX over the ranks' n values (same
// shape on every rank); the result lands in mapped host memory with a
// completion ticket, and the last CTA leaves {agree_tag, agree_ok} in Ctrl for
// gated collectives queued behind it. values: nloc * n (local-rank major).
int agree_launch(cm_comm* c, const int64_t* values, int n, cudaStream_t stream,
                 unsigned long long* ticket_out) {
  int st0 = ensure_agree_buf(c);
  if (st0) return st0;
  const int nloc = c->virt ? c->size : 1;
  long long inl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const unsigned long long ticket = ++c->agree_ticket;
  Launch L;
  L.n = n;
  L.dtype = CM_INT64;
  L.op = CM_MAX;
  plan_algo(c, CM_ALGO_RHD, n * 8, &L);
  L.ll = 1;
  L.oneshot = 1;
  if (!c->virt) {
    for (int i = 0; i < n; ++i) inl[i] = values[i];
    L.srcmode = SRC_INLINE;
    L.inl = inl;
  } else {
    // every local rank's values: pinned staging -> device (the host does not
    // touch the staging again before this call's completion word is seen)
    for (int lr = 0; lr < nloc; ++lr)
      for (int i = 0; i < 8; ++i) c->agree_host[AGH_IN + 8 * lr + i] = i < n ? values[lr * n + i] : 0;
    CUDA_TRY(cudaMemcpyAsync(c->agree_in, c->agree_host + AGH_IN, 8 * nloc * sizeof(int64_t),
                             cudaMemcpyHostToDevice, stream));
    L.srcmode = SRC_COPYIN;
    for (int lr = 0; lr < nloc; ++lr) L.in[lr] = c->agree_in + 8 * lr;
  }
  for (int lr = 0; lr < nloc; ++lr) L.out[lr] = c->agree_dev + AGH_RES + 8 * lr;
  L.done_flag = reinterpret_cast<unsigned long long*>(c->agree_dev + AGH_DONE);
  L.done_value = ticket;
  int st = launch_collective(c, L, stream);
  if (st) return st;
  *ticket_out = ticket;
  return CM_OK;
}

// wait half: host spin on every local rank's completion word; maxes: nloc * n
int agree_wait(cm_comm* c, unsigned long long ticket, int n, int64_t* maxes, cudaStream_t stream) {
  const int nloc = c->virt ? c->size : 1;
  for (int lr = 0; lr < nloc; ++lr) {
    int st = spin_ticket(c, AGH_DONE + lr, ticket, stream, "cm_agree");
    if (st) return st;
    for (int i = 0; i < n; ++i)
      maxes[lr * n + i] = reinterpret_cast<volatile int64_t*>(c->agree_host)[AGH_RES + 8 * lr + i];
  }
  return CM_OK;
}

int agree_impl(cm_comm* c, const int64_t* values, int n, int64_t* maxes, cudaStream_t stream) {
  if (n < 1 || n > 8) return fail(CM_ERR_VALUE, "cm_agree takes 1..8 values");
  int st = check_async_error(c);
  if (st) return st;
  if (c->size == 1) {
    memcpy(maxes, values, n * sizeof(int64_t));
    return CM_OK;
  }
  unsigned long long ticket;
  if ((st = agree_launch(c, values, n, stream, &ticket))) return st;
  return agree_wait(c, ticket, n, maxes, stream);
}
}  // namespace

extern "C" {

int cm_agree(cm_comm_t* c, const int64_t* values, int n, int64_t* maxes, void* stream) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "use cm_agree_v on a virtual group");
  return agree_impl(c, values, n, maxes, static_cast<cudaStream_t>(stream));
}

int cm_agree_v(cm_comm_t* c, const int64_t* values, int n, int64_t* maxes, void* stream) {
  if (!c->virt) return fail(CM_ERR_UNSUPPORTED, "cm_agree_v needs a virtual group");
  return agree_impl(c, values, n, maxes, static_cast<cudaStream_t>(stream));
}

int cm_comm_counters(cm_comm_t* c, int64_t* messages_sent, int64_t* bytes_sent,
                     int64_t* nvlink_bytes_in, int64_t* calls) {
  *messages_sent = c->messages;
  *bytes_sent = c->bytes;
  *nvlink_bytes_in = c->nvlink_in;
  *calls = c->calls;
  return CM_OK;
}

int cm_comm_launches(cm_comm_t* c, int64_t* launches) {
  *launches = c->launches;
  return CM_OK;
}

int cm_comm_set_trace(cm_comm_t* c, void* device_buffer, int ctas) {
  c->trace = static_cast<unsigned long long*>(device_buffer);
  c->trace_ctas = device_buffer ? ctas : 0;
  return CM_OK;
}

int cm_comm_profile(cm_comm_t* c, int enable) {
  c->profiling = enable != 0;
  return CM_OK;
}

int cm_comm_profile_read(cm_comm_t* c, int kind, int64_t* launches, double* total_ms,
                         int64_t* alg_bytes) {
  int64_t n = 0, b = 0;
  double ms = 0;
  std::vector<cm_comm::Prof> keep;
  for (auto& pr : c->prof) {
    if (pr.kind != kind) { keep.push_back(pr); continue; }
    CUDA_TRY(cudaEventSynchronize(pr.e1));
    float t = 0;
    cudaEventElapsedTime(&t, pr.e0, pr.e1);
    ms += t;
    b += pr.alg_bytes;
    ++n;
    c->event_pool.push_back(pr.e0);
    c->event_pool.push_back(pr.e1);
  }
  c->prof.swap(keep);
  *launches = n;
  *total_ms = ms;
  *alg_bytes = b;
  return CM_OK;
}

int cm_allreduce(cm_comm_t* c, const void* send, void* recv, int64_t count, int dtype, int op,
                 int algo, int64_t switch_bytes, int average, void* stream, cm_stats_t* stats) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "use cm_allreduce_v on a virtual group");
  DeviceScope ds(c->device);
  return do_allreduce(c, &send, &recv, count, dtype, op, algo, switch_bytes, average, stream, stats);
}

int cm_allreduce_v(cm_comm_t* c, const void* const* sends, void* const* recvs, int64_t count,
                   int dtype, int op, int algo, int64_t switch_bytes, int average, void* stream,
                   cm_stats_t* stats) {
  if (!c->virt) return fail(CM_ERR_UNSUPPORTED, "cm_allreduce_v needs a virtual group");
  DeviceScope ds(c->device);
  return do_allreduce(c, sends, recvs, count, dtype, op, algo, switch_bytes, average, stream, stats);
}

int cm_reduce_scatter(cm_comm_t* c, const void* send, void* recv, int64_t count, int dtype, int op,
                      int layout, void* stream, cm_stats_t* stats) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "use cm_reduce_scatter_v on a virtual group");
  DeviceScope ds(c->device);
  return do_rs(c, &send, &recv, count, dtype, op, layout, stream, stats);
}

int cm_reduce_scatter_v(cm_comm_t* c, const void* const* sends, void* const* recvs, int64_t count,
                        int dtype, int op, int layout, void* stream, cm_stats_t* stats) {
  if (!c->virt) return fail(CM_ERR_UNSUPPORTED, "needs a virtual group");
  DeviceScope ds(c->device);
  return do_rs(c, sends, recvs, count, dtype, op, layout, stream, stats);
}

int cm_allgather(cm_comm_t* c, const void* send, void* recv, int64_t count, int dtype, int layout,
                 void* stream, cm_stats_t* stats) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "use cm_allgather_v on a virtual group");
  DeviceScope ds(c->device);
  return do_ag(c, &send, &recv, count, dtype, layout, stream, stats);
}

int cm_allgather_v(cm_comm_t* c, const void* const* sends, void* const* recvs, int64_t count,
                   int dtype, int layout, void* stream, cm_stats_t* stats) {
  if (!c->virt) return fail(CM_ERR_UNSUPPORTED, "needs a virtual group");
  DeviceScope ds(c->device);
  return do_ag(c, sends, recvs, count, dtype, layout, stream, stats);
}

}  // extern "C"

namespace {

// aggregate() hot loop (aggregation.py:138-176) for every local rank of the
// communicator (nloc = size on a virtual group, else 1):
//   sends[lr * n + k]   member k of local rank lr (device, pinned or pageable host)
//   recvs[lr]           its concatenated means (device or host)
//   agree_values[lr * n_agree + i], agreed[lr], stats[lr * n + g]
// Call structure under a pending agreement is the same on every rank whatever
// its plan: the first launch either is the LL agreement kernel or carries the
// agreement inline on the full grid (force_pull); every later collective is
// gated and, on a mismatch, returns without a barrier or an epoch advance.
int fused_impl(cm_comm* c, int n, const void* const* sends, const int64_t* counts, int dtype,
               void* const* recvs, int algo, int64_t threshold, int64_t switch_bytes, int average,
               const int64_t* agree_values, int n_agree, int* agreed, const int64_t* reg_ids,
               cudaStream_t stream, cm_stats_t* stats, int* n_calls) {
  int st = check_dtype_op(dtype, CM_SUM);
  if (st) return st;
  if (average && (dtype == CM_INT32 || dtype == CM_INT64))
    return fail(CM_ERR_SHAPE, "averaging needs a floating-point dtype");
  if ((st = check_async_error(c))) return st;
  if (threshold <= 0) return fail(CM_ERR_VALUE, "fusion threshold must be positive");
  if (n < 0) return fail(CM_ERR_VALUE, "negative member count");
  if (n_agree < 0 || n_agree > 4) return fail(CM_ERR_VALUE, "at most 4 agreement values");
  for (int k = 0; k < n; ++k)
    if (counts[k] < 0) return fail(CM_ERR_SHAPE, "negative element count");
  const int p = c->size;
  const int nloc = c->virt ? p : 1;
  *n_calls = 0;
  if (n_agree > 0)
    for (int lr = 0; lr < nloc; ++lr) agreed[lr] = 1;
  const int64_t sz = (int64_t)dtype_size(dtype);
  std::vector<int64_t> nbytes(n);
  std::vector<int> dts(n, dtype), group(n);
  int64_t total_bytes = 0;
  for (int i = 0; i < n; ++i) {
    nbytes[i] = counts[i] * sz;
    total_bytes += nbytes[i];
  }
  int ngroups = 0;
  if (n > 0) cm_fuse_plan(n, nbytes.data(), dts.data(), threshold, group.data(), &ngroups);
  auto rank_of = [&](int lr) { return c->virt ? lr : c->rank; };
  // every member of every local rank is classified once per call through the
  // pointer cache (aggregation.py:159-161), and so is every output
  std::vector<int> kinds((size_t)nloc * n, CM_KIND_DEVICE);
  bool any_host_in = false, out_host = false, out_dev = false;
  for (int lr = 0; lr < nloc; ++lr) {
    for (int k = 0; k < n; ++k)
      if (counts[k] > 0 && (st = classify(c, sends[(size_t)lr * n + k], &kinds[(size_t)lr * n + k]))) return st;
    int rk = CM_KIND_DEVICE;
    if (total_bytes > 0 && (st = classify(c, recvs[lr], &rk))) return st;
    (rk == CM_KIND_HOST ? out_host : out_dev) = true;
  }
  for (int v : kinds) any_host_in = any_host_in || v == CM_KIND_HOST;
  if (out_host && out_dev) return fail(CM_ERR_UNSUPPORTED, "local ranks mix host and device outputs");
  HostPipe hp(c, stream);
  if (p == 1) {
    // single rank: every allreduce is the identity and the mean divides by 1
    // (collectives.py:119-120), so all fused groups collapse into ONE batched
    // copy of the members into the concatenated output
    std::vector<const void*> srcs(n);
    std::vector<void*> dsts(n);
    int64_t off = 0;
    for (int k = 0; k < n; ++k) {
      srcs[k] = sends[k];
      dsts[k] = static_cast<char*>(recvs[0]) + off;
      off += nbytes[k];
    }
    for (int g = 0; g < ngroups; ++g) {
      stats[g] = cm_stats_t{0, 0, 0};
      count_stats(c, stats[g]);
    }
    if (any_host_in || out_host) {
      // H2D into the device (h2d stream) and, for host outputs, D2H back out
      // (d2h stream) in host_chunk pieces so both PCIe directions stream at
      // once; members adjacent in memory are copied as one run (one DMA)
      if ((st = hp.start(out_host ? off : 0, 0))) return st;
      const std::vector<int64_t> cuts = graded_cuts(off, c->host_chunk);
      const std::vector<Run> runs = split_runs(coalesce(srcs.data(), nbytes.data(), n, INT64_MAX), cuts);
      int64_t chunk_lo = 0;
      size_t ci = 0;
      for (size_t k = 0; k < runs.size(); ++k) {
        const Run& r = runs[k];
        CUDA_TRY(cudaMemcpyAsync((out_host ? c->indev : static_cast<char*>(recvs[0])) + r.off, r.src, r.bytes,
                                 cudaMemcpyDefault, c->h2d));
        const int64_t end = r.off + r.bytes;
        while (ci < cuts.size() && cuts[ci] < end) ++ci;
        const bool at_cut = ci < cuts.size() && cuts[ci] == end;
        if (out_host && (at_cut || k + 1 == runs.size())) {
          if ((st = hp.link(c->h2d, c->d2h))) return st;
          CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recvs[0]) + chunk_lo, c->indev + chunk_lo, end - chunk_lo,
                                   cudaMemcpyDeviceToHost, c->d2h));
          chunk_lo = end;
        }
      }
      if ((st = hp.join())) return st;
    } else if ((st = launch_batched_copy(c, n, srcs.data(), dsts.data(), nbytes.data(), false, stream))) {
      return st;
    }
    *n_calls = ngroups;
    return CM_OK;
  }
  // host inputs or outputs: the copy-stream pipeline (device buffers sized for
  // every local rank's whole call) starts before the plan takes their addresses
  if (!c->virt && (st = service_autoreg(c, stream))) return st;   // peers' new allocations, if any
  if ((any_host_in || out_host) &&
      (st = hp.start(any_host_in ? nloc * total_bytes : 0, out_host ? nloc * total_bytes : 0)))
    return st;
  auto outbase = [&](int lr) -> char* {
    return out_host ? c->outdev + (int64_t)lr * total_bytes : static_cast<char*>(recvs[lr]);
  };
  // Pass 1: per fused group, members, size, algorithm and launch plan
  struct Grp {
    int i, j;
    int64_t ng, off;   // elements, offset in the fused output
    bool any_host;
    Launch L;
    bool batchable;
  };
  std::vector<Grp> gr;
  {
    int i = 0;
    int64_t fused_off = 0;
    for (int g = 0; g < ngroups; ++g) {
      Grp G;
      G.i = i;
      G.ng = 0;
      G.any_host = false;
      int j = i;
      while (j < n && group[j] == g) {
        for (int lr = 0; lr < nloc; ++lr) G.any_host = G.any_host || kinds[(size_t)lr * n + j] == CM_KIND_HOST;
        G.ng += counts[j];
        ++j;
      }
      G.j = j;
      G.off = fused_off;
      int concrete;
      if ((st = cm_resolve_algorithm(algo, G.ng * sz, switch_bytes, &concrete))) return st;
      for (int lr = 0; lr < nloc; ++lr)
        cm_algo_stats(concrete, p, rank_of(lr), G.ng, dtype, switch_bytes, &stats[(size_t)lr * n + g]);
      if (G.ng * sz > (int64_t)c->staging_bytes)
        return fail(CM_ERR_CONFIG, "fused buffer of " + std::to_string(G.ng * sz) +
                                       " B exceeds the staging area; lower the fusion threshold");
      G.L.n = G.ng;
      G.L.dtype = dtype;
      G.L.op = CM_SUM;
      G.L.average = average;
      plan_algo(c, concrete, G.ng * sz, &G.L);
      for (int lr = 0; lr < nloc; ++lr) G.L.out[lr] = outbase(lr) + fused_off * sz;
      G.batchable = c->multi_buffer && !G.any_host && G.L.ll == 0 && !G.L.oneshot &&
                    G.L.phases == (PH_RS | PH_AG);
      gr.push_back(G);
      fused_off += G.ng;
      i = j;
    }
  }
  // agreement (negotiate_ready fast path, aggregation.py:72-92)
  const bool want_agree = n_agree > 0;
  const bool inline_mode = want_agree && n_agree == 2 && c->inline_agree && !gr.empty();
  unsigned long long ticket = 0;
  if (want_agree) {
    if ((st = ensure_agree_buf(c))) return st;
    if (inline_mode) {
      ticket = ++c->agree_ticket;
    } else {
      std::vector<int64_t> vals((size_t)nloc * 2 * n_agree);
      for (int lr = 0; lr < nloc; ++lr)
        for (int i = 0; i < n_agree; ++i) {
          vals[(size_t)lr * 2 * n_agree + i] = agree_values[lr * n_agree + i];
          vals[(size_t)lr * 2 * n_agree + n_agree + i] = -agree_values[lr * n_agree + i];
        }
      if ((st = agree_launch(c, vals.data(), 2 * n_agree, stream, &ticket))) return st;
    }
  }
  bool first_launch = true;
  auto tag_launch = [&](Launch& L) {
    if (!want_agree) return;
    if (inline_mode && first_launch) {
      L.agree_inline = 1;
      L.force_pull = 1;
      for (int lr = 0; lr < nloc; ++lr) {
        L.akey[lr] = agree_values[lr * n_agree];
        L.acnt[lr] = agree_values[lr * n_agree + 1];
      }
      L.agree_out = reinterpret_cast<unsigned long long*>(c->agree_dev + AGH_INL);
      L.agree_ticket = ticket;
    } else {
      L.agree_gate = ticket;
    }
    first_launch = false;
  };
  // host-input groups: every group's H2D is queued up front on the h2d stream
  // (into indev at the local rank's and the group's offset); each collective
  // waits only for its own input's event. A two-shot group moves in pieces of
  // ~host_piece bytes (the piece-th 1/K of every rank's segment, segments_of):
  // H2D of piece k+1 overlaps the collective of piece k and the D2H of piece
  // k-1, so only one piece, not the whole group, fills and drains the pipeline
  std::vector<std::vector<cudaEvent_t>> in_ready(gr.size());
  auto indev_at = [&](int lr, const Grp& G) { return c->indev + (int64_t)lr * total_bytes + G.off * sz; };
  auto npieces = [&](const Grp& G) -> int {
    if (!c->host_split || !G.any_host || G.L.ll != 0 || G.L.oneshot || G.L.phases != (PH_RS | PH_AG)) return 1;
    return (int)std::max<int64_t>(1, std::min<int64_t>(128, (G.ng * sz + c->host_piece / 2) / c->host_piece));
  };
  // element ranges [a, z) of piece k of group G (one per rank segment)
  auto piece_ranges = [&](const Grp& G, int k, int K, int64_t* a, int64_t* z) {
    int64_t off[MAXP], len[MAXP];
    segments_of(G.ng, p, G.L.layout, k, K, off, len);
    for (int q = 0; q < p; ++q) { a[q] = off[q]; z[q] = off[q] + len[q]; }
  };
  for (size_t t = 0; t < gr.size(); ++t) {
    if (!gr[t].any_host) continue;
    std::vector<int64_t> gb(nbytes.begin() + gr[t].i, nbytes.begin() + gr[t].j);
    const int K = npieces(gr[t]);
    in_ready[t].assign(K, nullptr);
    std::vector<std::vector<Run>> runs(nloc);
    for (int lr = 0; lr < nloc; ++lr)
      runs[lr] = coalesce(sends + (size_t)lr * n + gr[t].i, gb.data(), gr[t].j - gr[t].i, INT64_MAX);
    for (int k = 0; k < K; ++k) {
      int64_t a[MAXP], z[MAXP];
      if (K > 1) piece_ranges(gr[t], k, K, a, z);
      const int nr = K > 1 ? p : 1;
      for (int lr = 0; lr < nloc; ++lr)
        for (int q = 0; q < nr; ++q) {
          const int64_t lo = K > 1 ? a[q] * sz : 0, hi = K > 1 ? z[q] * sz : gr[t].ng * sz;
          for (const Run& r : runs[lr]) {           // the runs' parts inside [lo, hi)
            const int64_t x = std::max(lo, r.off), y = std::min(hi, r.off + r.bytes);
            if (y > x)
              CUDA_TRY(cudaMemcpyAsync(indev_at(lr, gr[t]) + x, r.src + (x - r.off), y - x, cudaMemcpyDefault,
                                       c->h2d));
          }
        }
      if ((st = hp.ev(&in_ready[t][k]))) return st;
      CUDA_TRY(cudaEventRecord(in_ready[t][k], c->h2d));
    }
  }
  // host outputs: after the launch of groups [a, b), copy their results out
  auto drain = [&](size_t a, size_t b) -> int {
    if (!out_host) return CM_OK;
    int s2 = hp.link(stream, c->d2h);
    if (s2) return s2;
    for (size_t t = a; t < b; ++t)
      if (gr[t].ng)
        for (int lr = 0; lr < nloc; ++lr)
          CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recvs[lr]) + gr[t].off * sz, outbase(lr) + gr[t].off * sz,
                                   gr[t].ng * sz, cudaMemcpyDeviceToHost, c->d2h));
    return CM_OK;
  };
  // pack members [i, j) of every local rank into its staging (byte offsets from `base`)
  auto pack = [&](int i, int j) -> int {
    std::vector<void*> dsts;
    int64_t o = 0;
    for (int k = i; k < j; ++k) {
      dsts.push_back(reinterpret_cast<void*>((uintptr_t)o));
      o += nbytes[k];
    }
    for (int lr = 0; lr < nloc; ++lr) {
      int s2 = launch_batched_copy(c, j - i, sends + (size_t)lr * n + i, dsts.data(), nbytes.data() + i, true, stream,
                                   c->virt ? c->heap[lr] : nullptr);
      if (s2) return s2;
    }
    return CM_OK;
  };
  // Pass 2: launches. Consecutive two-shot groups with the same layout share
  // one pack + one multi-buffer launch (up to MAXBUF); others go one by one.
  size_t g = 0;
  while (g < gr.size()) {
    size_t h = g + 1;
    if (gr[g].batchable) {
      int64_t tot = gr[g].ng;
      while (h < gr.size() && h - g < (size_t)MAXBUF && gr[h].batchable &&
             gr[h].L.order == gr[g].L.order && gr[h].L.layout == gr[g].L.layout &&
             (tot + gr[h].ng) * sz <= (int64_t)c->staging_bytes) {
        tot += gr[h].ng;
        ++h;
      }
    }
    bool gather_ok = reg_ids != nullptr && gr[g].batchable;
    if (gather_ok)
      for (size_t t = g; t < h && gather_ok; ++t)
        for (int k = gr[t].i; k < gr[t].j; ++k) gather_ok = gather_ok && reg_ids[k] >= 0;
    if (gather_ok || h - g > 1) {
      Launch L = gr[g].L;
      L.nbuf = (int)(h - g);
      for (int lr = 0; lr < nloc; ++lr) L.out[lr] = outbase(lr);
      int64_t boff = 0;
      for (size_t t = g; t < h; ++t) {
        L.bn[t - g] = gr[t].ng;
        L.bboff[t - g] = boff;
        L.bout_off[t - g] = gr[t].off;
        boff += gr[t].ng;
      }
      L.n = L.bn[0];
      if (gather_ok) {
        // registered gradients: peers' members are read in place, no pack
        std::vector<long long> tab(1, 0), ids;
        int64_t e = 0;
        for (size_t t = g; t < h; ++t)
          for (int k = gr[t].i; k < gr[t].j; ++k) {
            e += counts[k];
            tab.push_back(e);
            ids.push_back(reg_ids[k]);
          }
        const int gm = (int)ids.size();
        tab.insert(tab.end(), ids.begin(), ids.end());
        std::string key(reinterpret_cast<const char*>(tab.data()), tab.size() * sizeof(long long));
        auto it = c->gtabs.find(key);
        long long* dtab;
        if (it != c->gtabs.end()) {
          dtab = it->second;
        } else {
          CUDA_TRY(cudaMalloc(&dtab, tab.size() * sizeof(long long)));
          CUDA_TRY(cudaMemcpy(dtab, tab.data(), tab.size() * sizeof(long long), cudaMemcpyHostToDevice));
          c->gtabs[key] = dtab;
        }
        unsigned long long sig = 1469598103934665603ull;
        for (long long v : tab) sig = (sig ^ (unsigned long long)v) * 1099511628211ull;
        L.gtab = dtab;
        L.gmem = gm;
        L.gsig = sig;
        L.srcmode = SRC_GATHER;
      } else {
        // members of all groups are consecutive in the staged layout
        if ((st = pack(gr[g].i, gr[h - 1].j))) return st;
        L.srcmode = SRC_PRESTAGED;
      }
      tag_launch(L);
      if ((st = launch_collective(c, L, stream))) return st;
      if ((st = drain(g, h))) return st;
      g = h;
      continue;
    }
    Grp& G = gr[g];
    Launch L = G.L;
    if (G.any_host && in_ready[g].size() > 1) {   // piece by piece (see the H2D loop above)
      const int K = (int)in_ready[g].size();
      for (int k = 0; k < K; ++k) {
        Launch Lk = G.L;
        CUDA_TRY(cudaStreamWaitEvent(stream, in_ready[g][k], 0));
        Lk.srcmode = SRC_COPYIN;
        Lk.piece = k;
        Lk.npieces = K;
        for (int lr = 0; lr < nloc; ++lr) Lk.in[lr] = indev_at(lr, G);
        tag_launch(Lk);
        if ((st = launch_collective(c, Lk, stream))) return st;
        if (out_host) {
          if ((st = hp.link(stream, c->d2h))) return st;
          int64_t a[MAXP], z[MAXP];
          piece_ranges(G, k, K, a, z);
          for (int lr = 0; lr < nloc; ++lr)
            for (int q = 0; q < p; ++q)
              if (z[q] > a[q])
                CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recvs[lr]) + (G.off + a[q]) * sz,
                                         outbase(lr) + (G.off + a[q]) * sz, (z[q] - a[q]) * sz,
                                         cudaMemcpyDeviceToHost, c->d2h));
        }
      }
      ++g;
      continue;
    }
    if (G.any_host) {  // inputs arrive in indev on the h2d stream, then copy-in
      CUDA_TRY(cudaStreamWaitEvent(stream, in_ready[g][0], 0));
      L.srcmode = SRC_COPYIN;
      for (int lr = 0; lr < nloc; ++lr) L.in[lr] = indev_at(lr, G);
    } else {         // pack straight into the IPC staging area (no extra copy)
      if ((st = pack(G.i, G.j))) return st;
      L.srcmode = SRC_PRESTAGED;
    }
    tag_launch(L);
    if ((st = launch_collective(c, L, stream))) return st;
    if ((st = drain(g, g + 1))) return st;
    ++g;
  }
  if ((st = hp.join())) return st;
  // the agreement result arrives while the gated collectives run; on a
  // mismatch they were no-ops on every rank and the caller negotiates
  if (want_agree) {
    if (inline_mode) {
      if ((st = inline_agree_wait(c, ticket, stream, agreed))) return st;
    } else {
      std::vector<int64_t> mx((size_t)nloc * 2 * n_agree);
      if ((st = agree_wait(c, ticket, 2 * n_agree, mx.data(), stream))) return st;
      for (int lr = 0; lr < nloc; ++lr) {
        bool same = true;
        for (int i = 0; i < n_agree; ++i)
          same = same && mx[(size_t)lr * 2 * n_agree + i] == agree_values[lr * n_agree + i] &&
                 mx[(size_t)lr * 2 * n_agree + n_agree + i] == -agree_values[lr * n_agree + i];
        agreed[lr] = same ? 1 : 0;
      }
    }
    for (int lr = 0; lr < nloc; ++lr)
      if (!agreed[lr]) return CM_OK;
  }
  for (int lr = 0; lr < nloc; ++lr)
    for (int q = 0; q < ngroups; ++q) count_stats(c, stats[(size_t)lr * n + q]);
  *n_calls = ngroups;
  return CM_OK;
}

}  // namespace

extern "C" {

int cm_fused_allreduce(cm_comm_t* c, int n, const void* const* sends, const int64_t* counts,
                       int dtype, void* recv_fused, int algo, int64_t threshold,
                       int64_t switch_bytes, int average, void* stream_, cm_stats_t* stats,
                       int* n_calls) {
  return cm_fused_allreduce_agreed(c, n, sends, counts, dtype, recv_fused, algo, threshold,
                                   switch_bytes, average, nullptr, 0, nullptr, nullptr, stream_,
                                   stats, n_calls);
}

int cm_fused_allreduce_agreed(cm_comm_t* c, int n, const void* const* sends,
                              const int64_t* counts, int dtype, void* recv_fused, int algo,
                              int64_t threshold, int64_t switch_bytes, int average,
                              const int64_t* agree_values, int n_agree, int* agreed,
                              const int64_t* reg_ids, void* stream, cm_stats_t* stats,
                              int* n_calls) {
  if (c->virt) return fail(CM_ERR_UNSUPPORTED, "use cm_fused_allreduce_agreed_v on a virtual group");
  DeviceScope ds(c->device);
  void* rv[1] = {recv_fused};
  return fused_impl(c, n, sends, counts, dtype, rv, algo, threshold, switch_bytes, average, agree_values,
                    n_agree, agreed, reg_ids, static_cast<cudaStream_t>(stream), stats, n_calls);
}

int cm_fused_allreduce_agreed_v(cm_comm_t* c, int n, const void* const* sends, const int64_t* counts,
                                int dtype, void* const* recvs_fused, int algo, int64_t threshold,
                                int64_t switch_bytes, int average, const int64_t* agree_values, int n_agree,
                                int* agreed, const int64_t* reg_ids, void* stream, cm_stats_t* stats,
                                int* n_calls) {
  if (!c->virt) return fail(CM_ERR_UNSUPPORTED, "cm_fused_allreduce_agreed_v needs a virtual group");
  DeviceScope ds(c->device);
  return fused_impl(c, n, sends, counts, dtype, recvs_fused, algo, threshold, switch_bytes, average,
                    agree_values, n_agree, agreed, reg_ids, static_cast<cudaStream_t>(stream), stats, n_calls);
}

// Parameter-server step (paramserver.py:171-271) on the NVLink heap: workers
// stage their gradients, owners update their shards in float64, workers pull
// the others'. `grads`: nloc * n pointers (rank-major; ignored for non-workers),
// `params`: nloc fused parameter buffers (in/out, sorted-name layout).
int cm_ps_step_v(cm_comm_t* c, int n, const void* const* grads, void* const* params, const int64_t* counts,
                 int dtype, const int* owners, uint32_t worker_mask, double lr, void* stream_) {
  if (dtype != CM_FLOAT32 && dtype != CM_FLOAT64)
    return fail(CM_ERR_SHAPE, "the parameter server handles float32 / float64 (core.py:18-21)");
  const int p = c->size;
  if (n < 1) return fail(CM_ERR_VALUE, "no tensors");
  if (worker_mask == 0 || (p < 32 && (worker_mask >> p) != 0)) return fail(CM_ERR_VALUE, "bad worker mask");
  int st;
  if ((st = check_async_error(c))) return st;
  const int64_t sz = (int64_t)dtype_size(dtype);
  int64_t gtot = 0;
  std::vector<int64_t> goff(n);
  for (int t = 0; t < n; ++t) {
    if (counts[t] < 0) return fail(CM_ERR_SHAPE, "negative element count");
    if (owners[t] < 0 || owners[t] >= p) return fail(CM_ERR_VALUE, "shard owner outside the group");
    goff[t] = gtot;
    gtot += counts[t];
  }
  if (served_off(gtot, sz) + gtot * sz > (int64_t)c->staging_bytes)
    return fail(CM_ERR_CONFIG, "parameter-server step needs " + std::to_string(served_off(gtot, sz) + gtot * sz) +
                                   " B of staging; the communicator has " + std::to_string(c->staging_bytes));
  // owner table: own_first[0..p], then {prefix, goff, len} per owned tensor
  std::vector<long long> tab(p + 1, 0);
  std::vector<long long> ent;
  int64_t maxown = 0;
  for (int q = 0; q < p; ++q) {
    tab[q] = (long long)(ent.size() / 3);
    int64_t pre = 0;
    for (int t = 0; t < n; ++t)
      if (owners[t] == q && counts[t] > 0) {
        ent.push_back(pre);
        ent.push_back(goff[t]);
        ent.push_back(counts[t]);
        pre += counts[t];
      }
    maxown = std::max(maxown, pre);
  }
  tab[p] = (long long)(ent.size() / 3);
  tab.insert(tab.end(), ent.begin(), ent.end());
  std::string key = "ps:" + std::string(reinterpret_cast<const char*>(tab.data()), tab.size() * sizeof(long long));
  long long* dtab;
  auto it = c->gtabs.find(key);
  if (it != c->gtabs.end()) {
    dtab = it->second;
  } else {
    CUDA_TRY(cudaMalloc(&dtab, tab.size() * sizeof(long long)));
    CUDA_TRY(cudaMemcpy(dtab, tab.data(), tab.size() * sizeof(long long), cudaMemcpyHostToDevice));
    c->gtabs[key] = dtab;
  }
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int nloc = c->virt ? p : 1;
  // 1. workers stage their gradients (sorted-name layout) into staging[next parity]
  for (int l = 0; l < nloc; ++l) {
    const int r = c->virt ? l : c->rank;
    if (!((worker_mask >> r) & 1u)) continue;
    std::vector<const void*> srcs(n);
    std::vector<void*> dsts(n);
    std::vector<int64_t> bytes(n);
    for (int t = 0; t < n; ++t) {
      srcs[t] = grads[(size_t)l * n + t];
      dsts[t] = reinterpret_cast<void*>((uintptr_t)(goff[t] * sz));
      bytes[t] = counts[t] * sz;
    }
    if ((st = launch_batched_copy(c, n, srcs.data(), dsts.data(), bytes.data(), true, stream, c->heap[r])))
      return st;
  }
  // 2. the step kernel
  PsParams P;
  memset(&P, 0, sizeof P);
  for (int q = 0; q < p; ++q) P.heap[q] = c->heap[q];
  for (int l = 0; l < nloc; ++l) P.params[l] = static_cast<char*>(params[l]);
  P.table = dtab;
  P.p = p;
  P.rank = c->rank;
  P.virt = c->virt ? 1 : 0;
  for (int q = 0; q < p; ++q)
    if ((worker_mask >> q) & 1u) P.workers[P.nworkers++] = q;
  P.worker_mask = worker_mask;
  P.gtot = gtot;
  P.lr = lr;
  unsigned long long h = make_hdr(gtot, dtype, 0, 0, 3, 0, 0, 0) ^ ((unsigned long long)worker_mask << 52);
  for (long long v : tab) h = (h ^ (unsigned long long)v) * 1099511628211ull;
  P.hdr = h;
  P.timeout_cycles = c->timeout_cycles;
  P.staging_off = (long long)c->staging_off;
  P.staging_bytes = (long long)c->staging_bytes;
  P.herr = c->herr_dev;
  int64_t nb = (maxown * sz + c->twoshot_bytes_per_cta - 1) / c->twoshot_bytes_per_cta;
  nb = std::max<int64_t>(1, std::min<int64_t>(nb, std::min(c->max_ctas, MAXBLK)));
  const void* k = dtype == CM_FLOAT32 ? (const void*)ps_kernel<F32> : (const void*)ps_kernel<F64>;
  void* args[] = {&P};
  if (c->virt) {
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, 0));
    nb = std::min<int64_t>(nb, std::max<int64_t>(1, (int64_t)per_sm * c->sms / p));
    CUDA_TRY(cudaLaunchCooperativeKernel(k, dim3((unsigned)nb, (unsigned)p), dim3(THREADS), args, 0, stream));
  } else {
    CUDA_TRY(cudaLaunchKernel(k, dim3((unsigned)nb), dim3(THREADS), args, 0, stream));
  }
  c->launches += 1;
  c->calls += 1;
  return CM_OK;
}

int cm_ps_step(cm_comm_t* c, int n, const void* const* grads, void* params, const int64_t* counts, int dtype,
               const int* owners, uint32_t worker_mask, double lr, void* stream) {
  void* pv[1] = {params};
  return cm_ps_step_v(c, n, grads, pv, counts, dtype, owners, worker_mask, lr, stream);
}

int cm_local_reduce(const void* a, const void* b, void* out, int64_t count, int dtype, int op,
                    void* stream) {
  int st = check_dtype_op(dtype, op);
  if (st) return st;
  if (count <= 0) return CM_OK;
  const bool vec = ((((uintptr_t)a) | ((uintptr_t)b) | ((uintptr_t)out)) & 15u) == 0;
  const int64_t nb = std::max<int64_t>(1, std::min<int64_t>((count + THREADS * 8 - 1) / (THREADS * 8), 148 * 8));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  char* po = static_cast<char*>(out);
  const int v = vec ? 1 : 0;
#define LR(D)                                                                                   \
  if (op == CM_SUM) local_reduce_kernel<D, CM_SUM><<<(unsigned)nb, THREADS, 0, s>>>(pa, pb, po, count, v); \
  else local_reduce_kernel<D, CM_MAX><<<(unsigned)nb, THREADS, 0, s>>>(pa, pb, po, count, v);
  switch (dtype) {
    case CM_FLOAT32: LR(F32); break;
    case CM_FLOAT64: LR(F64); break;
    case CM_BFLOAT16: LR(BF16); break;
    case CM_INT32: LR(I32); break;
    case CM_INT64: LR(I64); break;
  }
#undef LR
  CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

int cm_batched_copy(int n, const void* const* srcs, void* const* dsts, const int64_t* nbytes,
                    void* stream) {
  if (n < 0) return fail(CM_ERR_VALUE, "negative count");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // members the kernel cannot dereference (pageable host memory) go through
  // the copy engines; the rest are one batched-copy launch
  std::vector<const void*> ks;
  std::vector<void*> kd;
  std::vector<int64_t> kb;
  for (int i = 0; i < n; ++i) {
    bool direct = true;
    for (const void* ptr : {srcs[i], static_cast<const void*>(dsts[i])}) {
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        direct = false;
      } else if (a.type == cudaMemoryTypeUnregistered) {
        direct = false;
      }
    }
    if (direct) {
      ks.push_back(srcs[i]);
      kd.push_back(dsts[i]);
      kb.push_back(nbytes[i]);
    } else if (nbytes[i] > 0) {
      CUDA_TRY(cudaMemcpyAsync(dsts[i], srcs[i], nbytes[i], cudaMemcpyDefault, s));
    }
  }
  return launch_batched_copy(nullptr, (int)ks.size(), ks.data(), kd.data(), kb.data(), false, s);
}

int cm_bench_p2p(cm_comm_t* c, int mode, int64_t bytes, int ctas, int iters, void* stream_,
                 double* ms_per_iter) {
  if (c->virt || c->size < 2) return fail(CM_ERR_UNSUPPORTED, "needs a real group of >= 2 ranks");
  // modes 10/11 (flag latency): `bytes` is the number of iterations per launch
  const int64_t need = (mode >= 10) ? 0 : (int64_t)bytes * ((mode >= 6 && mode <= 9) ? 6 : c->size);
  if (need > (int64_t)c->staging_bytes) return fail(CM_ERR_CONFIG, "bytes too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  CollParams P;
  memset(&P, 0, sizeof P);
  for (int q = 0; q < c->size; ++q) P.heap[q] = c->heap[q];
  P.p = c->size;
  P.rank = c->rank;
  P.staging_off = (long long)c->staging_off;
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CopyParams B;
  memset(&B, 0, sizeof B);
  if (mode == 4) {
    CUDA_TRY(cudaFuncSetAttribute((const void*)bulk_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)BULK_SMEM));
    int m = 0;
    B.start[0] = 0;
    for (int i = 1; i < c->size; ++i) {
      const int q = (c->rank + i) % c->size;
      B.src[m] = c->heap[q] + c->staging_off + (int64_t)c->rank * bytes;
      B.dst[m] = c->local + c->staging_off + (int64_t)q * bytes;
      B.start[m + 1] = B.start[m] + bytes;
      ++m;
    }
    B.n = m;
  }
  // modes 14/15: copy engines (cudaMemcpyAsync over the IPC mappings), one
  // stream per peer so the p-1 transfers run concurrently; 14 pulls, 15 pushes
  std::vector<cudaStream_t> ce_s;
  std::vector<cudaEvent_t> ce_e;
  cudaEvent_t fork = nullptr;
  if (mode == 14 || mode == 15) {
    CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (int i = 1; i < c->size; ++i) {
      cudaStream_t t;
      cudaEvent_t e;
      CUDA_TRY(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ce_s.push_back(t);
      ce_e.push_back(e);
    }
  }
  if (mode == 17)
    CUDA_TRY(cudaFuncSetAttribute((const void*)empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bytes));
  if (mode == 20 && bytes > 0)
    CUDA_TRY(cudaFuncSetAttribute((const void*)spin_kernel_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bytes));
  int spin_i = 0;   // modes 18/19: launch index (stamps at staging[2 i], [2 i + 1])
  if (mode >= 18 && mode <= 24 && (int64_t)(iters + 1) * 16 + 65536 > (int64_t)c->staging_bytes)
    return fail(CM_ERR_CONFIG, "too many iterations");
  static unsigned long long flag_base = 1ull << 40;   // slot values only grow (same sequence on every rank)
  auto launch = [&]() {
    if (mode == 14 || mode == 15) {
      cudaEventRecord(fork, s);
      for (int i = 1; i < c->size; ++i) {
        const int q = (c->rank + i) % c->size;
        cudaStream_t t = ce_s[i - 1];
        cudaStreamWaitEvent(t, fork, 0);
        if (mode == 14)
          cudaMemcpyAsync(c->local + c->staging_off + (int64_t)q * bytes,
                          c->heap[q] + c->staging_off + (int64_t)c->rank * bytes, bytes, cudaMemcpyDeviceToDevice, t);
        else
          cudaMemcpyAsync(c->heap[q] + c->staging_off + (int64_t)c->rank * bytes,
                          c->local + c->staging_off + (int64_t)q * bytes, bytes, cudaMemcpyDeviceToDevice, t);
        cudaEventRecord(ce_e[i - 1], t);
        cudaStreamWaitEvent(s, ce_e[i - 1], 0);
      }
    } else if (mode == 18 || mode == 19) {
      auto* out = reinterpret_cast<unsigned long long*>(c->local + c->staging_off);
      if (mode == 18) spin_kernel_big<<<ctas, THREADS, 0, s>>>(P, out, spin_i, 20000);
      else spin_kernel_small<<<ctas, THREADS, 0, s>>>(out, spin_i, 20000);
      ++spin_i;
    } else if (mode == 20) {
      auto* out = reinterpret_cast<unsigned long long*>(c->local + c->staging_off);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)ctas);
      cfg.blockDim = dim3(THREADS);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.dynamicSmemBytes = (size_t)bytes;   // > 114 KiB: one CTA per SM, the next grid cannot co-reside
      cudaLaunchKernelEx(&cfg, spin_kernel_pdl, P, out, spin_i, (long long)20000);
      ++spin_i;
    } else if (mode >= 21 && mode <= 24) {
      auto* out = reinterpret_cast<unsigned long long*>(c->local + c->staging_off);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)ctas);
      cfg.blockDim = dim3(THREADS);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, spin_kernel_remote, P, out, spin_i, (long long)20000, mode - 21);
      ++spin_i;
    } else if (mode == 16) {
      empty_kernel<<<ctas, THREADS, 0, s>>>(0);
    } else if (mode == 17) {
      empty_kernel<<<ctas, THREADS, (size_t)bytes, s>>>(0);
    } else if (mode == 4) bulk_copy_kernel<<<ctas, BULK_THREADS, BULK_SMEM, s>>>(B);
    else if (mode >= 10 && mode <= 13) {
      flag_latency_kernel<<<mode == 10 ? 1 : ctas, THREADS, 0, s>>>(P, mode, bytes, flag_base);
      flag_base += (unsigned long long)bytes + 1;
    } else p2p_bw_kernel<<<ctas, THREADS, 0, s>>>(P, mode, bytes);
  };
  launch();
  CUDA_TRY(cudaEventRecord(e0, s));
  for (int i = 0; i < iters; ++i) launch();
  CUDA_TRY(cudaEventRecord(e1, s));
  CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (mode >= 18 && mode <= 24) {   // median device gap between consecutive launches
    std::vector<unsigned long long> st((size_t)2 * spin_i);
    CUDA_TRY(cudaMemcpy(st.data(), c->local + c->staging_off, st.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<double> gaps;
    for (int i = 1; i < spin_i; ++i) gaps.push_back((double)(st[2 * i] - st[2 * i - 1]) * 1e-6);
    std::sort(gaps.begin(), gaps.end());
    ms = gaps.empty() ? 0.f : (float)(gaps[gaps.size() / 2] * iters);
  }
  for (auto t : ce_s) cudaStreamDestroy(t);
  for (auto e : ce_e) cudaEventDestroy(e);
  if (fork) cudaEventDestroy(fork);
  *ms_per_iter = ms / iters;
  return CM_OK;
}

int cm_time_allreduce(cm_comm_t* c, const void* send, void* recv, int64_t count, int dtype, int op,
                      int algo, int64_t switch_bytes, int iters, int warmup, void* stream,
                      double* ms_per_call) {
  if (iters < 1) return fail(CM_ERR_VALUE, "iters must be >= 1");
  cm_stats_t stv[MAXP];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < warmup; ++i) {
    int st = c->virt ? CM_ERR_UNSUPPORTED : cm_allreduce(c, send, recv, count, dtype, op, algo, switch_bytes, 0, stream, stv);
    if (st) return st;
  }
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaEventRecord(e0, s));
  for (int i = 0; i < iters; ++i) {
    int st = cm_allreduce(c, send, recv, count, dtype, op, algo, switch_bytes, 0, stream, stv);
    if (st) return st;
  }
  CUDA_TRY(cudaEventRecord(e1, s));
  CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_per_call = ms / iters;
  return check_async_error(c);
}

}  // extern "C"
