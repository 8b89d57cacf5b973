// Host-side reference-schedule logic: chunking, ownership layouts, algorithm
// resolution, the reference's per-rank CollectiveStats, and greedy fusion.
// Pure C++ (no CUDA calls) so it runs in the CPU test tier.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"

namespace cm {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

// core.py:113-130 — the first n mod p chunks get one extra element.
void chunk_partition(int64_t n, int p, int64_t* off, int64_t* len) {
  const int64_t base = n / p, rem = n % p;
  int64_t o = 0;
  for (int i = 0; i < p; ++i) {
    const int64_t l = base + (i < rem ? 1 : 0);
    off[i] = o;
    len[i] = l;
    o += l;
  }
}

struct RhdParams {
  int m, excess, steps;
};

static RhdParams rhd_params(int p) {
  int m = 1;
  while ((m << 1) <= p) m <<= 1;                       // collectives.py:172
  int steps = 0;
  while ((1 << steps) < m) ++steps;                   // :174
  return {m, p - m, steps};                           // :173
}

int rhd_vrank(int rank, int p) {                      // collectives.py:180-192
  const RhdParams rp = rhd_params(p);
  if (rank < 2 * rp.excess) return (rank % 2 == 1) ? -1 : rank / 2;
  return rank - rp.excess;
}

// Segment each vrank owns after recursive halving (collectives.py:198-216):
// bit k of vrank selects the upper half at step k; mid = lo + (hi-lo)//2.
void rhd_layout(int64_t n, int p, int64_t* off, int64_t* len) {
  const RhdParams rp = rhd_params(p);
  for (int r = 0; r < p; ++r) {
    const int v = rhd_vrank(r, p);
    if (v < 0) {
      off[r] = 0;
      len[r] = 0;
      continue;
    }
    int64_t lo = 0, hi = n;
    for (int k = 0; k < rp.steps; ++k) {
      const int64_t mid = lo + (hi - lo) / 2;
      if ((v >> k) & 1) lo = mid; else hi = mid;
    }
    off[r] = lo;
    len[r] = hi - lo;
  }
}

// Per-vrank element counts sent in halving then doubling (collectives.py:198-229).
static void rhd_sent(int64_t n, int p, std::vector<std::vector<int64_t>>& sent) {
  const RhdParams rp = rhd_params(p);
  std::vector<int64_t> lo(rp.m, 0), hi(rp.m, n);
  sent.assign(rp.m, {});
  for (int k = 0; k < rp.steps; ++k) {
    std::vector<int64_t> nlo(lo), nhi(hi);
    for (int v = 0; v < rp.m; ++v) {
      const int64_t mid = lo[v] + (hi[v] - lo[v]) / 2;
      const int pv = v ^ (1 << k);
      if (v < pv) { sent[v].push_back(hi[v] - mid); nhi[v] = mid; }
      else        { sent[v].push_back(mid - lo[v]); nlo[v] = mid; }
    }
    lo.swap(nlo);
    hi.swap(nhi);
  }
  for (int k = rp.steps - 1; k >= 0; --k) {
    std::vector<int64_t> nlo(lo), nhi(hi);
    for (int v = 0; v < rp.m; ++v) {
      const int pv = v ^ (1 << k);
      sent[v].push_back(hi[v] - lo[v]);
      const int64_t incoming = hi[pv] - lo[pv];
      if (v < pv) nhi[v] = hi[v] + incoming; else nlo[v] = lo[v] - incoming;
    }
    lo.swap(nlo);
    hi.swap(nhi);
  }
}

static cm_stats_t mk(int64_t r, int64_t m, int64_t b) { return cm_stats_t{r, m, b}; }

static cm_stats_t ring_stats(int p, int rank, int64_t n, int64_t isz) {   // :107-152
  if (p == 1) return mk(0, 0, 0);
  std::vector<int64_t> off(p), len(p);
  chunk_partition(n, p, off.data(), len.data());
  int64_t b = 0;
  for (int s = 0; s < p - 1; ++s) b += len[(rank + s + 1) % p] + len[(rank + s) % p];
  return mk(2 * (p - 1), 2 * (p - 1), b * isz);
}

static cm_stats_t rhd_stats(int p, int rank, int64_t n, int64_t isz) {    // :155-236
  if (p == 1) return mk(0, 0, 0);
  const RhdParams rp = rhd_params(p);
  const int64_t rounds = 2 * rp.steps + (rp.excess ? 2 : 0);
  const int v = rhd_vrank(rank, p);
  if (v < 0) return mk(rounds, 1, n * isz);
  std::vector<std::vector<int64_t>> sent;
  rhd_sent(n, p, sent);
  int64_t msgs = (int64_t)sent[v].size(), b = 0;
  for (int64_t x : sent[v]) b += x;
  if (rank < 2 * rp.excess) { msgs += 1; b += n; }
  return mk(rounds, msgs, b * isz);
}

static cm_stats_t flat_stats(int p, int rank, int64_t n, int64_t isz) {   // :82-104
  if (p == 1) return mk(0, 0, 0);
  if (rank == 0) return mk(2, p - 1, (int64_t)(p - 1) * n * isz);
  return mk(2, 1, n * isz);
}

}  // namespace cm

namespace cm {
constexpr int64_t kSliceAlign = 64;   // = dev::SLICE_ALIGN (kernel slice boundaries)
// Segment of every rank (ring chunk_partition or rhd layout of n elements),
// optionally only the piece-th 1/npieces of each, cut on kSliceAlign element
// boundaries: the host pipeline moves a fused buffer through H2D -> collective
// -> D2H in such pieces, and every element keeps the owner (and so the fold
// order) it has in the whole-buffer allreduce, so pieces are bit-identical to
// one launch over the buffer.
void segments_of(int64_t n, int p, int layout, int piece, int npieces, int64_t* off, int64_t* len) {
  if (layout == CM_LAYOUT_RHD) rhd_layout(n, p, off, len);
  else chunk_partition(n, p, off, len);
  if (npieces <= 1) return;
  for (int q = 0; q < p; ++q) {
    auto cut = [&](int i) -> int64_t {
      if (i <= 0) return off[q];
      if (i >= npieces) return off[q] + len[q];
      const int64_t x = (off[q] + len[q] * i / npieces) / kSliceAlign * kSliceAlign;
      return std::min(std::max(x, off[q]), off[q] + len[q]);
    };
    const int64_t a = cut(piece), z = cut(piece + 1);
    off[q] = a;
    len[q] = z - a;
  }
}

}  // namespace cm

using namespace cm;

extern "C" {

const char* cm_version(void) { return "cm 0.1.0 (sm_100a)"; }
const char* cm_last_error(void) { return g_last_error.c_str(); }
size_t cm_dtype_size(int dtype) { return dtype_size(dtype); }

int cm_chunk_partition(int64_t n, int p, int64_t* offsets, int64_t* lengths) {
  if (p < 1) return fail(CM_ERR_INVALID_GROUP, "cannot partition over p=" + std::to_string(p) + " processes");
  if (n < 0) return fail(CM_ERR_SHAPE, "negative element count " + std::to_string(n));
  chunk_partition(n, p, offsets, lengths);
  return CM_OK;
}

int cm_layout_piece(int layout, int64_t n, int p, int piece, int npieces, int64_t* offsets, int64_t* lengths) {
  if (p < 1) return fail(CM_ERR_INVALID_GROUP, "group size must be >= 1");
  if (n < 0) return fail(CM_ERR_SHAPE, "negative element count");
  if (layout != CM_LAYOUT_RING && layout != CM_LAYOUT_RHD) return fail(CM_ERR_CONFIG, "unknown layout");
  if (npieces < 1 || piece < 0 || piece >= npieces) return fail(CM_ERR_VALUE, "piece out of range");
  segments_of(n, p, layout, piece, npieces, offsets, lengths);
  return CM_OK;
}

int cm_layout(int layout, int64_t n, int p, int64_t* offsets, int64_t* lengths) {
  if (p < 1) return fail(CM_ERR_INVALID_GROUP, "group size must be >= 1");
  if (n < 0) return fail(CM_ERR_SHAPE, "negative element count");
  if (layout == CM_LAYOUT_RING) chunk_partition(n, p, offsets, lengths);
  else if (layout == CM_LAYOUT_RHD) rhd_layout(n, p, offsets, lengths);
  else return fail(CM_ERR_CONFIG, "unknown layout " + std::to_string(layout));
  return CM_OK;
}

static const char* algo_name(int a) {
  switch (a) {
    case CM_ALGO_AUTO: return "auto";
    case CM_ALGO_FLAT: return "flat";
    case CM_ALGO_RING: return "ring_rsa";
    case CM_ALGO_RHD: return "rhd_rsa";
    default: return nullptr;
  }
}

int cm_resolve_algorithm(int algo, int64_t nbytes, int64_t switch_bytes, int* concrete) {
  if (!algo_name(algo)) return fail(CM_ERR_CONFIG, "unknown algorithm " + std::to_string(algo));
  if (algo != CM_ALGO_AUTO) { *concrete = algo; return CM_OK; }
  if (switch_bytes <= 0) return fail(CM_ERR_CONFIG, "switch_bytes must be > 0 for auto dispatch");
  *concrete = nbytes < switch_bytes ? CM_ALGO_RHD : CM_ALGO_RING;   // collectives.py:247
  return CM_OK;
}

int cm_algo_stats(int algo, int p, int rank, int64_t n, int dtype, int64_t switch_bytes,
                  cm_stats_t* out) {
  const int64_t isz = (int64_t)dtype_size(dtype);
  if (!isz) return fail(CM_ERR_SHAPE, "unsupported dtype");
  if (p < 1 || rank < 0 || rank >= p) return fail(CM_ERR_INVALID_GROUP, "bad rank/size");
  int c;
  int st = cm_resolve_algorithm(algo, n * isz, switch_bytes, &c);
  if (st) return st;
  if (c == CM_ALGO_RING) *out = ring_stats(p, rank, n, isz);
  else if (c == CM_ALGO_RHD) *out = rhd_stats(p, rank, n, isz);
  else *out = flat_stats(p, rank, n, isz);
  return CM_OK;
}

int cm_rs_stats(int layout, int p, int rank, int64_t n, int dtype, cm_stats_t* out) {
  const int64_t isz = (int64_t)dtype_size(dtype);
  if (!isz) return fail(CM_ERR_SHAPE, "unsupported dtype");
  if (p < 1 || rank < 0 || rank >= p) return fail(CM_ERR_INVALID_GROUP, "bad rank/size");
  if (p == 1) { *out = mk(0, 0, 0); return CM_OK; }
  if (layout == CM_LAYOUT_RING) {          // collectives.py:128-139
    std::vector<int64_t> off(p), len(p);
    chunk_partition(n, p, off.data(), len.data());
    int64_t b = 0;
    for (int s = 0; s < p - 1; ++s) b += len[(rank + s + 1) % p];
    *out = mk(p - 1, p - 1, b * isz);
    return CM_OK;
  }
  if (layout != CM_LAYOUT_RHD) return fail(CM_ERR_CONFIG, "unknown layout");
  const RhdParams rp = rhd_params(p);     // fold (:180-192) + halving (:198-216)
  const int64_t rounds = rp.steps + (rp.excess ? 1 : 0);
  const int v = rhd_vrank(rank, p);
  if (v < 0) { *out = mk(rounds, 1, n * isz); return CM_OK; }
  std::vector<std::vector<int64_t>> sent;
  rhd_sent(n, p, sent);
  int64_t b = 0;
  for (int k = 0; k < rp.steps; ++k) b += sent[v][k];
  *out = mk(rounds, rp.steps, b * isz);
  return CM_OK;
}

int cm_ag_stats(int layout, int p, int rank, int64_t n, int dtype, cm_stats_t* out) {
  const int64_t isz = (int64_t)dtype_size(dtype);
  if (!isz) return fail(CM_ERR_SHAPE, "unsupported dtype");
  if (p < 1 || rank < 0 || rank >= p) return fail(CM_ERR_INVALID_GROUP, "bad rank/size");
  if (p == 1) { *out = mk(0, 0, 0); return CM_OK; }
  if (layout == CM_LAYOUT_RING) {          // collectives.py:142-150
    std::vector<int64_t> off(p), len(p);
    chunk_partition(n, p, off.data(), len.data());
    int64_t b = 0;
    for (int s = 0; s < p - 1; ++s) b += len[(rank + s) % p];
    *out = mk(p - 1, p - 1, b * isz);
    return CM_OK;
  }
  if (layout != CM_LAYOUT_RHD) return fail(CM_ERR_CONFIG, "unknown layout");
  const RhdParams rp = rhd_params(p);     // doubling (:219-229) + serve fold (:234-235)
  const int64_t rounds = rp.steps + (rp.excess ? 1 : 0);
  const int v = rhd_vrank(rank, p);
  if (v < 0) { *out = mk(rounds, 0, 0); return CM_OK; }
  std::vector<std::vector<int64_t>> sent;
  rhd_sent(n, p, sent);
  int64_t msgs = rp.steps, b = 0;
  for (int k = rp.steps; k < 2 * rp.steps; ++k) b += sent[v][k];
  if (rank < 2 * rp.excess) { msgs += 1; b += n; }
  *out = mk(rounds, msgs, b * isz);
  return CM_OK;
}

// aggregation.py:95-130 — greedy first-fit in the given order; a dtype change
// or overflowing the threshold closes the group; reaching it flushes.
int cm_fuse_plan(int n, const int64_t* nbytes, const int* dtypes, int64_t threshold,
                 int* group_of, int* n_groups) {
  if (threshold <= 0) return fail(CM_ERR_VALUE, "fusion threshold must be positive");
  int g = -1;
  int64_t cur = 0;
  bool open = false;
  int cur_dtype = -1;
  for (int i = 0; i < n; ++i) {
    if (open && (cur_dtype != dtypes[i] || cur + nbytes[i] > threshold)) { open = false; cur = 0; }
    if (!open) { ++g; open = true; cur_dtype = dtypes[i]; cur = 0; }
    group_of[i] = g;
    cur += nbytes[i];
    if (cur >= threshold) { open = false; cur = 0; }
  }
  *n_groups = g + 1;
  return CM_OK;
}

}  // extern "C"
