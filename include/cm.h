/*
 * cm.h — C ABI of the B200-native CUDA-aware allreduce ("collective memory").
 *
 * Drop-in boundary for the reference's allreduce hot path
 * (/root/reference/pkg/src/collectium/, paths below relative to it). The
 * reference is pure Python, so there is no reference FFI to bind; each entry
 * point below names the reference interface it replaces. The Python façade
 * (paper_1810_11112_b200/_lib.py) binds these with ctypes and keeps the
 * reference's signatures, argument meanings and exception classes.
 *
 * Conventions
 *  - Every function returns an int status (CM_OK = 0). On failure
 *    cm_last_error() returns a thread-local message. Status codes map 1:1 onto
 *    the reference exception classes of errors.py:4-56.
 *  - Plain pointers and sizes only; `stream` is a cudaStream_t passed as void*.
 *  - Collectives are out-of-place (const send, recv) like the reference, which
 *    copies its input and returns a new Tensor (collectives.py:123,176); send ==
 *    recv (in place) is also accepted. They are stream-ordered: they return
 *    after enqueueing; device-side errors (peer shape mismatch, timeouts) are
 *    reported by cm_comm_sync()/cm_comm_poll().
 */
#ifndef CM_H_
#define CM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CM_MAX_RANKS 16

/* status codes <-> errors.py exception classes */
enum cm_status {
  CM_OK = 0,
  CM_ERR_SHAPE = 1,           /* ShapeError            errors.py:8   */
  CM_ERR_INVALID_GROUP = 2,   /* InvalidGroupError     errors.py:12  */
  CM_ERR_ROUTING = 3,         /* RoutingError          errors.py:16  */
  CM_ERR_TRANSPORT = 4,       /* TransportError        errors.py:20  (peer timeout) */
  CM_ERR_DEADLOCK = 5,        /* DeadlockError         errors.py:24  */
  CM_ERR_CONFIG = 6,          /* ConfigError           errors.py:55  */
  CM_ERR_INVALID_HANDLE = 7,  /* InvalidHandleError    errors.py:47  */
  CM_ERR_UNKNOWN_BUFFER = 8,  /* UnknownBufferError    errors.py:51  */
  CM_ERR_UNSUPPORTED = 9,     /* UnsupportedOperationError errors.py:36 */
  CM_ERR_CUDA = 10,           /* CUDA runtime failure (TransportError in Python) */
  CM_ERR_VALUE = 11           /* ValueError (bad argument)           */
};

/* element types: core.py:18-21 has float32/float64; bf16 and ints are extensions */
enum cm_dtype { CM_FLOAT32 = 0, CM_FLOAT64 = 1, CM_BFLOAT16 = 2, CM_INT32 = 3, CM_INT64 = 4 };
/* ReduceOp core.py:24-26 */
enum cm_op { CM_SUM = 0, CM_MAX = 1 };
/* ALGORITHMS collectives.py:20 */
enum cm_algo { CM_ALGO_AUTO = 0, CM_ALGO_FLAT = 1, CM_ALGO_RING = 2, CM_ALGO_RHD = 3 };
/* reduce-scatter / allgather ownership layouts (collectives.py:128-150 ring, :198-229 rhd) */
enum cm_layout { CM_LAYOUT_RING = 0, CM_LAYOUT_RHD = 1 };
/* Policy registry.py:32-35 */
enum cm_policy { CM_NO_CACHE = 0, CM_LAZY_CACHE = 1, CM_INTERCEPT_CACHE = 2 };
/* BufferKind registry.py:27-29 */
enum cm_kind { CM_KIND_HOST = 0, CM_KIND_DEVICE = 1 };

/* CollectiveStats collectives.py:28-32 (the reference's logical schedule) */
typedef struct {
  int64_t rounds;
  int64_t messages_per_rank;
  int64_t bytes_sent_per_rank;
} cm_stats_t;

/* RegistryStats registry.py:44-49 */
typedef struct {
  int64_t driver_queries;
  int64_t cache_hits;
  int64_t inserts;
  int64_t invalidations;
} cm_registry_stats_t;

/* what the pointer cache records about an address (real backend: memory type,
 * device ordinal, allocation range and buffer id from one
 * cuPointerGetAttributes; intercept cache: the registered range) */
typedef struct {
  int32_t kind;          /* cm_kind */
  int32_t device;        /* device ordinal, -1 for host memory / unknown */
  uint64_t range_start;  /* allocation holding the address (0 if unknown) */
  int64_t range_size;
  uint64_t buffer_id;    /* unique per allocation (0 if unknown) */
} cm_buffer_info_t;

typedef struct cm_comm cm_comm_t;
typedef struct cm_registry cm_registry_t;

const char* cm_version(void);
const char* cm_last_error(void);

/* ---------------------------------------------------------------------------
 * Host-side logic (no GPU required)
 * ------------------------------------------------------------------------- */

/* chunk_partition core.py:113-130 -> offsets[p], lengths[p] */
int cm_chunk_partition(int64_t n, int p, int64_t* offsets, int64_t* lengths);
/* ownership after reduce-scatter: ring = chunk_partition, rhd = halving segments
 * (collectives.py:198-216; folded odd ranks own (0,0)) */
int cm_layout(int layout, int64_t n, int p, int64_t* offsets, int64_t* lengths);
/* piece `piece` of `npieces` of every rank's segment (the host-gradient
 * pipeline's unit, cm.h "host_split"): the piece-th 1/npieces of each segment,
 * cut on 64-element boundaries; pieces of a segment are disjoint and cover it */
int cm_layout_piece(int layout, int64_t n, int p, int piece, int npieces, int64_t* offsets, int64_t* lengths);
/* resolve_algorithm collectives.py:239-247 (CM_ERR_CONFIG on bad algo/switch) */
int cm_resolve_algorithm(int algo, int64_t nbytes, int64_t switch_bytes, int* concrete);
/* CollectiveStats the reference reports for (algo, p, rank, n) — collectives.py:75-236 */
int cm_algo_stats(int algo, int p, int rank, int64_t n, int dtype, int64_t switch_bytes,
                  cm_stats_t* out);
int cm_rs_stats(int layout, int p, int rank, int64_t n, int dtype, cm_stats_t* out);
int cm_ag_stats(int layout, int p, int rank, int64_t n, int dtype, cm_stats_t* out);
/* fuse() greedy first-fit aggregation.py:95-130: group_of[i] = group index of member i */
int cm_fuse_plan(int n, const int64_t* nbytes, const int* dtypes, int64_t threshold,
                 int* group_of, int* n_groups);
size_t cm_dtype_size(int dtype);

/* ---------------------------------------------------------------------------
 * Pointer cache (registry.py:52-151, PAPER §V-B)
 *   simulated=1: the reference's model — fake addresses from 0x1000, lowest
 *     freed address reused, "driver query" = ground-truth lookup + counter.
 *   simulated=0: real memory — alloc = cudaMalloc / cudaHostAlloc (the
 *     intercepted allocation API), the driver query = cudaPointerGetAttributes,
 *     range lookups resolve interior pointers of registered allocations.
 * ------------------------------------------------------------------------- */
int cm_registry_create(int policy, int64_t query_delay_ns, int simulated, cm_registry_t** out);
int cm_registry_destroy(cm_registry_t* reg);
int cm_registry_alloc(cm_registry_t* reg, int kind, int64_t size, uint64_t* address);
int cm_registry_free(cm_registry_t* reg, uint64_t address);
/* tell an intercept cache about memory allocated elsewhere (e.g. torch) */
int cm_registry_register(cm_registry_t* reg, uint64_t address, int64_t size, int kind);
int cm_registry_unregister(cm_registry_t* reg, uint64_t address);
int cm_registry_classify(cm_registry_t* reg, uint64_t address, int* kind);
/* classify through the policy and return the cache entry's details */
int cm_registry_info(cm_registry_t* reg, uint64_t address, cm_buffer_info_t* out);
int cm_registry_ground_truth(cm_registry_t* reg, uint64_t address, int* kind);
int cm_registry_stats(cm_registry_t* reg, cm_registry_stats_t* out);
int cm_registry_policy(cm_registry_t* reg, int* policy);
/* total wall time spent in real driver queries (ns); simulated: queries*delay */
int cm_registry_query_time_ns(cm_registry_t* reg, int64_t* ns);
/* {"policy": ..., "driver_queries": ..., "cache_hits": ..., "inserts": ..., "invalidations": ...} */
int cm_registry_stats_json(cm_registry_t* reg, char* buf, size_t len);

/* ---------------------------------------------------------------------------
 * Communicator: one per rank (one process per GPU). Replaces the Transport
 * plugin (transport/base.py:8-57) — rank, size and the logical counters stay,
 * byte send/recv is replaced by a CUDA-IPC peer-mapped symmetric heap over
 * NVLink/NVSwitch.
 * Bootstrap: create -> exchange cm_comm_ipc_handle() bytes over any host
 * channel -> connect(all handles in rank order).
 * ------------------------------------------------------------------------- */
#define CM_IPC_HANDLE_BYTES 64
int cm_comm_create(int rank, int size, int device, int64_t staging_bytes, int64_t pool_bytes,
                   cm_comm_t** out);
int cm_comm_ipc_handle(cm_comm_t* comm, void* handle_out);
int cm_comm_connect(cm_comm_t* comm, const void* all_handles);
/* one process drives `size` virtual ranks on ONE GPU (single-GPU emulation
 * of the group, the GPU analogue of the reference's SimNetwork): every
 * collective launches one cooperative kernel holding all ranks' CTAs. */
int cm_comm_create_virtual(int size, int device, int64_t staging_bytes, cm_comm_t** out);
int cm_comm_destroy(cm_comm_t* comm);
int cm_comm_rank(cm_comm_t* comm, int* rank);
int cm_comm_size(cm_comm_t* comm, int* size);
/* device-side wait budget before a peer is declared dead (TransportError) */
int cm_comm_set_timeout(cm_comm_t* comm, double seconds);
/* pointer-cache policy used to classify send/recv on every call */
int cm_comm_set_policy(cm_comm_t* comm, int policy);
int cm_comm_registry(cm_comm_t* comm, cm_registry_t** reg);
/* tuning knobs (values must be > 0):
 *   "oneshot_max_bytes"   largest message reduced one-shot
 *   "ll_max_bytes"        one-shot through the low-latency slots up to here
 *   "ll2_max_bytes"       two-shot through the low-latency slots up to here
 *   "ll_units_per_cta", "ll2_units_per_cta", "oneshot_bytes_per_cta",
 *   "twoshot_bytes_per_cta", "max_ctas"   grid sizing
 *   "stream_chunk"        elements per chunk of the pipelined two-shot (1 = off)
 *   "multi_buffer"        2 = batch fused buffers into one launch, 1 = off
 *   "rhd_logp"            2 = rhd_rsa runs the literal log2(p)-step recursive
 *                         halving/doubling kernel (pairwise flags), 1 = off
 *                         (default: one-/two-shot kernels with the same tree)
 *   "bulk_copy"           2 = fusion pack through the TMA bulk-copy engine when
 *                         every member is 16-byte aligned, 1 = SM copy (default:
 *                         same kernel time, but its 96 KiB shared-memory carve-out
 *                         costs ~5 us of reconfiguration per step in the bench)
 *   "bulk_rs"             2..6 = the reduce phase streams its sources into this
 *                         many 32 KiB shared-memory stages with the bulk-copy
 *                         engine (default 6), 1 = SM loads
 *   "dyn_ag"              2 = the allgather is a (slice, peer) task queue shared
 *                         by the CTAs, 1 = each CTA pulls its own slice index
 *                         after a per-index barrier (default; measured equal)
 *   "host_chunk_kb"       KiB per H2D/D2H piece of the host-gradient pipeline
 *                         (default 8192; at p = 1 2048/4096/16384 measured slower)
 *   "host_split"          2 = with host gradients at p > 1 (aggregate's fused groups
 *                         and allreduce() of a host send buffer), a two-shot
 *                         collective moves H2D -> collective -> D2H in
 *                         ~host_piece_kb pieces
 *                         (the k-th 1/K of every rank's segment: same owners and
 *                         fold order as one launch, bit-identical); 1 = one
 *                         launch per group
 *   "host_piece_kb"       KiB per piece of host_split (default 4096)
 *   "bulk_stage_kb"       KiB per bulk-reduce stage (default 64; the stage count
 *                         is clamped to the shared memory available)
 *   "inline_agree"        2 = aggregate's ready-set agreement travels in the fused
 *                         collective's start-barrier records (default), 1 = a
 *                         separate LL agreement kernel gates the collective
 *   "overlap"             2 = the multi-buffer two-shot splits its grid: half the
 *                         CTAs reduce-scatter and push per-chunk progress, half
 *                         allgather each peer's chunks as soon as they are
 *                         reduced (no RS->AG barrier); 1 = off (default: the
 *                         reduce-scatter needs every SM to reach the NVLink
 *                         ceiling, measured 206 vs 191 us on the N=2 headline)
 *   "overlap_chunks"      reduce chunks per progress report (default 4)
 *   "auto_register"       2 = (default) the pointer cache registers the allocation
 *                         behind a plain device send buffer on first sight: its
 *                         CUDA-IPC handle goes into this rank's heap mailbox,
 *                         peers map it when their kernels report the new slot
 *                         and acknowledge in this heap; from then on peers read
 *                         the buffer in place (no copy into staging). 1 = off.
 *   "pdl"                 2 = (default) collective, low-latency, RHD and pack
 *                         kernels are launched with programmatic stream
 *                         serialization: the next launch is scheduled while the
 *                         previous kernel drains and waits in griddepcontrol.wait
 *                         (device gap between launches 2.5 -> 0.6 us); 1 = off.
 *   "pack_max_ctas"       CTA cap of the fusion pack (batched copy); 1 = none
 *                         (default). OverlappedAggregator(pack_ctas=...) sets it
 *                         so a pack next to the backward pass keeps SMs free
 *   "cluster_pairs"       2 = collective grids of <= 64 CTAs launch in 2-CTA
 *                         clusters (whole TPCs), so a capped collective next to
 *                         2-CTA-cluster GEMMs does not break their SM pairs;
 *                         1 = off (default; OverlappedAggregator(cluster_pairs=True) sets it)
 * get also reads the counters "auto_published", "auto_mapped",
 * "auto_zero_copy_calls" and "auto_buffer_checks" (allocation-id re-checks)
 * get also reads "staging_bytes", "pool_bytes" and "ll_payload_per_source" */
int cm_comm_set_param(cm_comm_t* comm, const char* key, int64_t value);
int cm_comm_get_param(cm_comm_t* comm, const char* key, int64_t* value);
/* symmetric allocation from the IPC heap (collective: same sizes, same order
 * on every rank). Buffers from here are read by peers in place (zero copy). */
int cm_comm_alloc(cm_comm_t* comm, int64_t bytes, void** ptr);
int cm_comm_free(cm_comm_t* comm, void* ptr);
/* Registered buffers — the pointer cache's IPC side (PAPER §V-B; NCCL-style
 * user-buffer registration). Collective: every rank exports the buffer it
 * passes at this registration (allocation handle + offset, cm_comm_export),
 * the 64-byte handles and offsets are all-gathered over any host channel, and
 * cm_comm_register opens every peer allocation once (cached) and records the
 * peer pointers under one id. Later collectives whose send buffer lies inside
 * a registered range are read by peers in place (no staging copy). Buffers
 * must stay allocated until cm_comm_deregister. */
int cm_comm_export(cm_comm_t* comm, const void* ptr, int64_t bytes, void* handle_out,
                   int64_t* offset);
int cm_comm_register(cm_comm_t* comm, const void* ptr, int64_t bytes, const void* all_handles,
                     const int64_t* all_offsets, int64_t* reg_id);
int cm_comm_deregister(cm_comm_t* comm, const void* ptr);
/* allocation ids (CU_POINTER_ATTRIBUTE_BUFFER_ID, 0 if unknown) of n device
 * pointers: a re-allocated range gets a new id even at the same address
 * (aggregate's automatic member registration checks its members with it) */
int cm_buffer_ids(cm_comm_t* comm, int n, const void* const* ptrs, uint64_t* ids);
/* virtual group (single-GPU emulation): register every virtual rank's buffer
 * (ptrs[size]) under one id; fused aggregates whose members all carry ids read
 * the members in place (the SRC_GATHER path of real communicators) */
int cm_comm_register_v(cm_comm_t* comm, const void* const* ptrs, int64_t bytes, int64_t* reg_id);
/* wait for `stream`, then report any device-side error of earlier calls */
int cm_comm_sync(cm_comm_t* comm, void* stream);
/* non-blocking error check of completed calls */
int cm_comm_poll(cm_comm_t* comm);
/* synchronous element-wise MAX over ranks of n <= 8 host int64 values (one
 * one-shot NVLink kernel); control-plane primitive of negotiate_ready
 * (aggregation.py:72-92) — equal (key, -key) maxima prove equal ready sets */
int cm_agree(cm_comm_t* comm, const int64_t* values, int n, int64_t* maxes, void* stream);
/* virtual group: values[size * n] (rank-major) -> maxes[size * n] */
int cm_agree_v(cm_comm_t* comm, const int64_t* values, int n, int64_t* maxes, void* stream);
/* logical counters (Transport.messages_sent / bytes_sent, base.py:43-57) and
 * the real NVLink bytes this rank pulled from peers */
int cm_comm_counters(cm_comm_t* comm, int64_t* messages_sent, int64_t* bytes_sent,
                     int64_t* nvlink_bytes_in, int64_t* calls);
/* number of kernels this comm has launched (bench "gpu_launches") */
int cm_comm_launches(cm_comm_t* comm, int64_t* launches);
/* diagnostics: every collective kernel writes globaltimer stamps of its
 * phases (start, copied-in, start barrier, reduced, mid barrier, end) into
 * device_buffer[(local_rank * ctas + cta) * 8 + phase] for ctas < `ctas`;
 * NULL disables */
int cm_comm_set_trace(cm_comm_t* comm, void* device_buffer, int ctas);
/* bracket every kernel this comm launches with CUDA events on its stream */
int cm_comm_profile(cm_comm_t* comm, int enable);
/* drain recorded launches of one kind (0 = pull collective kernel, 1 =
 * pack/copy kernel, 2 = LL / log-p collective kernels, e.g. the agreement
 * check): count, summed device ms, summed algorithmic bytes (collectives:
 * busBW bytes 2(p-1)/p*S; pack: bytes read + written) */
int cm_comm_profile_read(cm_comm_t* comm, int kind, int64_t* launches, double* total_ms,
                         int64_t* alg_bytes);

/* allreduce collectives.py:250-260 (+ allreduce_ring :107, allreduce_rhd :155,
 * allreduce_flat :75 via `algo`). Results are bit-identical to the reference
 * fold order of the resolved algorithm. average=1 divides by p inside the
 * reduction (the fused mean of aggregation.py:167-172). */
int cm_allreduce(cm_comm_t* comm, const void* send, void* recv, int64_t count, int dtype, int op,
                 int algo, int64_t switch_bytes, int average, void* stream, cm_stats_t* stats);
/* reduce-scatter / allgather phases of collectives.py:128-150 (ring) and
 * :178-229 (rhd) as public operations. recv of reduce_scatter holds this rank's
 * layout segment; send of allgather holds it. */
int cm_reduce_scatter(cm_comm_t* comm, const void* send, void* recv, int64_t count, int dtype,
                      int op, int layout, void* stream, cm_stats_t* stats);
int cm_allgather(cm_comm_t* comm, const void* send, void* recv, int64_t count, int dtype,
                 int layout, void* stream, cm_stats_t* stats);
/* aggregate() hot loop aggregation.py:158-174: members (already in negotiated
 * order, one dtype) are fused greedily under `threshold`, packed into the
 * IPC staging heap by one kernel per group, allreduced with the mean fused
 * in, and written to recv_fused (the members' concatenation; member i's mean
 * is recv_fused[sum(counts[:i]) : ...]). stats[] gets one entry per issued
 * allreduce; *n_calls their number. */
int cm_fused_allreduce(cm_comm_t* comm, int n, const void* const* sends, const int64_t* counts,
                       int dtype, void* recv_fused, int algo, int64_t threshold,
                       int64_t switch_bytes, int average, void* stream, cm_stats_t* stats,
                       int* n_calls);

/* cm_fused_allreduce preceded by the negotiation check: every rank passes the
 * same n_agree (<= 4) values (e.g. a hash of its ready names) when its ready
 * set is identical; *agreed = 1 and the fused launches follow in the same call,
 * or *agreed = 0 and no data moves on any rank (the caller negotiates the
 * intersection, aggregation.py:72-92, and calls again). The call's structure
 * does not depend on the rank's plan while the agreement is pending: with
 * n_agree == 2 the first collective carries the values in its start-barrier
 * records on the full grid, otherwise an LL agreement kernel goes first; all
 * later collectives are gated and skip (no barrier, no epoch advance) on a
 * mismatch, so ranks whose ready sets — and launch counts — differ stay in
 * step. reg_ids (nullable): per member, its cm_comm_register id (same on every
 * rank) or -1; fused groups whose members are all registered skip the pack —
 * peers read the member tensors in place. */
int cm_fused_allreduce_agreed(cm_comm_t* comm, int n, const void* const* sends,
                              const int64_t* counts, int dtype, void* recv_fused, int algo,
                              int64_t threshold, int64_t switch_bytes, int average,
                              const int64_t* agree_values, int n_agree, int* agreed,
                              const int64_t* reg_ids, void* stream, cm_stats_t* stats,
                              int* n_calls);

/* virtual-group variants: arrays of `size` per-rank pointers */
/* sends[size * n] (rank-major), recvs_fused[size], agree_values[size * n_agree],
 * agreed[size], stats[size * n] (rank r's group g at r * n + g) */
int cm_fused_allreduce_agreed_v(cm_comm_t* comm, int n, const void* const* sends,
                                const int64_t* counts, int dtype, void* const* recvs_fused, int algo,
                                int64_t threshold, int64_t switch_bytes, int average,
                                const int64_t* agree_values, int n_agree, int* agreed,
                                const int64_t* reg_ids, void* stream, cm_stats_t* stats,
                                int* n_calls);
int cm_allreduce_v(cm_comm_t* comm, const void* const* sends, void* const* recvs, int64_t count,
                   int dtype, int op, int algo, int64_t switch_bytes, int average, void* stream,
                   cm_stats_t* stats);
int cm_reduce_scatter_v(cm_comm_t* comm, const void* const* sends, void* const* recvs,
                        int64_t count, int dtype, int op, int layout, void* stream,
                        cm_stats_t* stats);
int cm_allgather_v(cm_comm_t* comm, const void* const* sends, void* const* recvs, int64_t count,
                   int dtype, int layout, void* stream, cm_stats_t* stats);

/* ---------------------------------------------------------------------------
 * Local kernels
 * ------------------------------------------------------------------------- */
/* local_reduce core.py:94-110: out = a op b (a is the accumulator) */
/* parameter-server pull step paramserver.py:171-271 (round-robin shard map
 * :159-165 given as owners[], tensors in sorted-name order): worker ranks
 * (worker_mask bit q) stage their gradients; each owner sums the workers'
 * shards in worker-rank order in float64, divides by the worker count and
 * applies params -= lr * mean (float64, then rounded to the dtype); workers
 * then pull every other owner's updated shards into `params` (a fused
 * device buffer, in/out). float32 / float64. Stream-ordered. */
int cm_ps_step(cm_comm_t* comm, int n, const void* const* grads, void* params, const int64_t* counts,
               int dtype, const int* owners, uint32_t worker_mask, double lr, void* stream);
int cm_ps_step_v(cm_comm_t* comm, int n, const void* const* grads, void* const* params,
                 const int64_t* counts, int dtype, const int* owners, uint32_t worker_mask, double lr,
                 void* stream);

int cm_local_reduce(const void* a, const void* b, void* out, int64_t count, int dtype, int op,
                    void* stream);
/* fuse/unfuse payload moves aggregation.py:110-111,133-135: one launch copies
 * n (src, dst, bytes) triples; members in pageable host memory (which the
 * kernel cannot dereference) are moved by the copy engines instead */
int cm_batched_copy(int n, const void* const* srcs, void* const* dsts, const int64_t* nbytes,
                    void* stream);
/* diagnostics: all-to-all NVLink bandwidth, every rank moving `bytes` to or
 * from each peer per round (ms per round): 2 = SM pull (all peers
 * concurrently), 3 = SM push, 4 = TMA bulk pull, 5 = pull + local add,
 * 6..9 = two-rank store anatomy, 14 = copy-engine pull, 15 = copy-engine push
 * (cudaMemcpyAsync over the IPC mappings, one stream per peer).
 * Flag latency: mode 10 = ping-pong between ranks 0 and 1 (one thread),
 * 11..13 = the start-barrier pattern on `ctas` CTAs; `bytes` = iterations
 * per launch, ms_per_iter = time per launch (divide by the iterations) */
int cm_bench_p2p(cm_comm_t* comm, int mode, int64_t bytes, int ctas, int iters, void* stream,
                 double* ms_per_iter);
/* device-timed loop of cm_allreduce (CUDA events on `stream`), ms per call */
int cm_time_allreduce(cm_comm_t* comm, const void* send, void* recv, int64_t count, int dtype,
                      int op, int algo, int64_t switch_bytes, int iters, int warmup,
                      void* stream, double* ms_per_call);

#ifdef __cplusplus
}
#endif
#endif /* CM_H_ */
