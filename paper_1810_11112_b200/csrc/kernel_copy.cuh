// diagnostic NVLink bandwidth kernel, batched copy (fusion pack) and TMA bulk copy
// (part of the sm_100a device code; see kernels.cuh for the overview)
#pragma once

#include "dev_common.cuh"

namespace cm {
namespace dev {
// ---- diagnostics: launch cost of an empty kernel with a small parameter block
// (cm_bench_p2p modes 16/17; modes 2 with 0 bytes gives the CollParams block)
static __global__ void __launch_bounds__(THREADS) empty_kernel(int x) {
  extern __shared__ char dyn[];
  if (x == 12345 && threadIdx.x == 0) dyn[0] = 1;
}

// launch-to-launch gap on the device (modes 18/19): every CTA spins `ns`, CTA 0
// stamps its start and end into out[2 i], out[2 i + 1]
template <class Param>
__device__ __forceinline__ void spin_body(unsigned long long* out, int i, long long ns) {
  const unsigned long long t0 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[2 * i] = t0;
  while ((long long)(gtimer() - t0) < ns) {
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[2 * i + 1] = gtimer();
}
static __global__ void __launch_bounds__(THREADS) spin_kernel_big(const __grid_constant__ CollParams P,
                                                                  unsigned long long* out, int i, long long ns) {
  if (P.p == 12345) out[0] = 0;
  spin_body<CollParams>(out, i, ns);
}
static __global__ void __launch_bounds__(THREADS) spin_kernel_small(unsigned long long* out, int i, long long ns) {
  spin_body<int>(out, i, ns);
}
// mode 20: the same under programmatic dependent launch (the next launch is
// scheduled while this one runs and waits in griddepcontrol.wait)
static __global__ void __launch_bounds__(THREADS, 1) spin_kernel_pdl(const __grid_constant__ CollParams P,
                                                                     unsigned long long* out, int i, long long ns) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ char spin_dyn[];
  if (P.p == 12345) { out[0] = 0; spin_dyn[threadIdx.x] = 1; }
  spin_body<CollParams>(out, i, ns);
}

// mode 21: PDL spin kernel whose CTA 0 first stores one word into the next
// peer's heap (a remote NVLink write in flight long before the grid ends);
// mode 22: the same with a remote load instead
static __global__ void __launch_bounds__(THREADS, 1) spin_kernel_remote(const __grid_constant__ CollParams P,
                                                                        unsigned long long* out, int i, long long ns,
                                                                        int load) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  auto* peer = reinterpret_cast<unsigned long long*>(P.heap[(P.rank + 1) % P.p] + P.staging_off) + 4096 + P.rank;
  __shared__ __align__(128) unsigned char tma_buf[1024];
  __shared__ __align__(8) unsigned long long tma_bar;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (load == 2) {     // mode 23: the remote load through the bulk-copy engine (TMA)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tma_bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tma_bar)), "r"(1024)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(tma_buf)),
                   "l"(reinterpret_cast<const char*>(peer) - 8 * P.rank), "r"(1024), "r"(smem_u32(&tma_bar))
                   : "memory");
      mbar_wait(&tma_bar, 0);
      out[4095] = tma_buf[5];
    } else if (load == 3) {   // mode 24: L1-bypassing load (ld.global.cg), as the allgather copies
      out[4095] = __ldcg(peer);
    } else if (load) {
      out[4095] = *reinterpret_cast<volatile unsigned long long*>(peer);
    } else {
      *reinterpret_cast<volatile unsigned long long*>(peer) = (unsigned long long)i;
    }
  }
  spin_body<CollParams>(out, i, ns);
}

// ---- diagnostics: raw NVLink read / write bandwidth between all ranks --------
// mode 0: pull — every rank reads `bytes` from each peer's staging into its own
// mode 1: push — every rank writes `bytes` into each peer's staging
// (all-to-all pattern of the two-shot phases; no synchronisation, data unused)
static __global__ void __launch_bounds__(THREADS) p2p_bw_kernel(const __grid_constant__ CollParams P, int mode,
                                                         long long bytes) {
  const int rank = P.rank, p = P.p, tid = threadIdx.x;
  const long long nv = bytes / 16;
  const long long per = (nv + gridDim.x - 1) / gridDim.x;
  const long long v0 = per * blockIdx.x, v1 = min(nv, v0 + per);
  char* mine = P.heap[rank] + P.staging_off;
  if (mode >= 2) {  // all peers concurrently from every thread
    const bool pull = mode == 2;
    for (long long j = v0 + tid; j < v1; j += THREADS) {
      uint4 v[MAXP];
#pragma unroll
      for (int i = 1; i < 8; ++i) {
        if (i < p) {
          const int q = (rank + i) % p;
          const uint4* src = reinterpret_cast<const uint4*>(
              pull ? P.heap[q] + P.staging_off + (long long)rank * bytes : mine + (long long)q * bytes);
          v[i] = src[j];
        }
      }
#pragma unroll
      for (int i = 1; i < 8; ++i) {
        if (i < p) {
          const int q = (rank + i) % p;
          uint4* dst = reinterpret_cast<uint4*>(pull ? mine + (long long)q * bytes
                                                     : P.heap[q] + P.staging_off + (long long)rank * bytes);
          dst[j] = v[i];
        }
      }
    }
    return;
  }
  for (int i = 1; i < p; ++i) {
    const int q = (rank + i) % p;
    char* peer = P.heap[q] + P.staging_off;
    const uint4* src = reinterpret_cast<const uint4*>(mode == 0 ? peer + (long long)rank * bytes
                                                                : mine + (long long)q * bytes);
    uint4* dst = reinterpret_cast<uint4*>(mode == 0 ? mine + (long long)q * bytes
                                                    : peer + (long long)rank * bytes);
    long long j = v0 + tid;
    for (; j + 3 * THREADS < v1; j += 4 * THREADS) {
      uint4 a = src[j], b = src[j + THREADS], c = src[j + 2 * THREADS], d = src[j + 3 * THREADS];
      dst[j] = a; dst[j + THREADS] = b; dst[j + 2 * THREADS] = c; dst[j + 3 * THREADS] = d;
    }
    for (; j < v1; j += THREADS) dst[j] = src[j];
  }
}

// ---- diagnostics: flag latency over NVLink ------------------------------------
// mode 10 (1 CTA): ping-pong between ranks 0 and 1 — iteration i: rank 0
//   stores i into rank 1's slot and waits for rank 1's answer; time per round trip
// mode 11 (every CTA): the start-barrier pattern — CTA b stores the iteration
//   into slot [b][rank] of every peer with st.release.sys, then waits for all
//   peers' slot [b][q] with ld.acquire.sys; time per barrier
// Slots live in the MID region (values only grow: base + i, base per call).
static __global__ void __launch_bounds__(THREADS, 1) flag_latency_kernel(const __grid_constant__ CollParams P,
                                                                         int mode, long long iters,
                                                                         unsigned long long base) {
  const int rank = P.rank, p = P.p, tid = threadIdx.x, b = blockIdx.x;
  char* mine = P.heap[rank];
  if (mode == 10) {
    if (tid != 0 || rank > 1) return;
    const int peer = 1 - rank;
    for (long long i = 1; i <= iters; ++i) {
      const unsigned long long v = base + (unsigned long long)i;
      if (rank == 0) {
        st_release_sys(mid_slot(P.heap[peer], 0, rank), v);
        while (ld_acquire_sys(mid_slot(mine, 0, peer)) < v) {
        }
      } else {
        while (ld_acquire_sys(mid_slot(mine, 0, peer)) < v) {
        }
        st_release_sys(mid_slot(P.heap[peer], 0, rank), v);
      }
    }
    return;
  }
  for (long long i = 1; i <= iters; ++i) {
    const unsigned long long v = base + (unsigned long long)i;
    if (mode == 11) {
      if (tid < p) st_release_sys(mid_slot(P.heap[tid], b, rank), v);
      if (tid < p)
        while (ld_acquire_sys(mid_slot(mine, b, tid)) < v) {
        }
    } else if (mode == 12) {   // relaxed stores and polls (no ordering; the raw path)
      if (tid < p) st_relaxed_sys(mid_slot(P.heap[tid], b, rank), v);
      if (tid < p)
        while (ld_relaxed_sys(mid_slot(mine, b, tid)) < v) {
        }
    } else {                   // 13: gpu-scope fence, relaxed store, relaxed poll
      if (tid < p) {
        __threadfence();
        st_relaxed_sys(mid_slot(P.heap[tid], b, rank), v);
      }
      if (tid < p)
        while (ld_relaxed_sys(mid_slot(mine, b, tid)) < v) {
        }
    }
    __syncthreads();
  }
}

// ---- batched copy (fusion pack / unfuse / cm_batched_copy) ---------------------
constexpr int MAXCOPY = 128;
struct CopyParams {
  const char* src[MAXCOPY];
  char* dst[MAXCOPY];          // absolute, or byte offset into staging[next parity] if staged
  long long start[MAXCOPY + 1];  // prefix sums of bytes
  int n;
  int staged;                  // dst is relative to own staging[(epoch+1)&1]
  char* heap;
  long long staging_bytes;
  long long staging_off;
};

// U: 16-byte loads in flight per thread (all issued before the stores)
template <int U>
__global__ void __launch_bounds__(THREADS) batched_copy_kernel(const __grid_constant__ CopyParams P) {
  pdl_begin();
  const long long total = P.start[P.n];
  const int b = blockIdx.x, nb = gridDim.x, tid = threadIdx.x;
  long long lo = (long long)(((__int128)total * b) / nb) & ~15ll;
  long long hi = b == nb - 1 ? total : ((long long)(((__int128)total * (b + 1)) / nb) & ~15ll);
  if (b == 0) lo = 0;
  char* base = nullptr;
  if (P.staged) {
    const unsigned long long e = epoch_read(P.heap, 0) + 1;
    base = P.heap + P.staging_off + (long long)(e & 1) * P.staging_bytes;
  }
  // find the first member overlapping [lo, hi)
  int k = 0;
  while (k < P.n && P.start[k + 1] <= lo) ++k;
  for (; k < P.n && P.start[k] < hi; ++k) {
    const long long a = lo > P.start[k] ? lo : P.start[k];
    const long long z = hi < P.start[k + 1] ? hi : P.start[k + 1];
    const char* s = P.src[k] + (a - P.start[k]);
    CM_CHECK(!P.staged || (long long)(uintptr_t)P.dst[k] + (P.start[k + 1] - P.start[k]) <= P.staging_bytes, nullptr);
    char* d = (P.staged ? base + (long long)(uintptr_t)P.dst[k] : P.dst[k]) + (a - P.start[k]);
    const long long nbytes = z - a;
    if ((((uintptr_t)s | (uintptr_t)d) & 15u) == 0) {
      const long long nv = nbytes >> 4;
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* d4 = reinterpret_cast<uint4*>(d);
      long long j = tid;
      for (; j + (U - 1) * THREADS < nv; j += U * THREADS) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = s4[j + u * THREADS];
#pragma unroll
        for (int u = 0; u < U; ++u) d4[j + u * THREADS] = r[u];
      }
      for (; j < nv; j += THREADS) d4[j] = s4[j];
      for (long long t = (nv << 4) + tid; t < nbytes; t += THREADS) d[t] = s[t];
    } else if ((((uintptr_t)s | (uintptr_t)d) & 3u) == 0) {
      const long long nw = nbytes >> 2;
      const uint32_t* s1 = reinterpret_cast<const uint32_t*>(s);
      uint32_t* d1 = reinterpret_cast<uint32_t*>(d);
      for (long long j = tid; j < nw; j += THREADS) d1[j] = s1[j];
      for (long long t = (nw << 2) + tid; t < nbytes; t += THREADS) d[t] = s[t];
    } else {
      for (long long t = tid; t < nbytes; t += THREADS) d[t] = s[t];
    }
  }
}

// ---- TMA bulk copy (same CopyParams; every member 16-byte aligned) ----------------
// One elected thread per CTA streams its contiguous byte range through a ring
// of BULK_STAGES shared-memory stages with the bulk-copy engine:
// cp.async.bulk global->shared (completion counted on an mbarrier), then
// cp.async.bulk shared->global (bulk group). Loads run BULK_STAGES-1 chunks
// ahead of the stores; no SM load/store instructions touch the payload.
constexpr int BULK_STAGES = 6;
constexpr int BULK_CHUNK = 16384;
constexpr int BULK_THREADS = 32;
constexpr size_t BULK_SMEM = (size_t)BULK_STAGES * BULK_CHUNK + BULK_STAGES * 8;

static __global__ void __launch_bounds__(BULK_THREADS) bulk_copy_kernel(const __grid_constant__ CopyParams P) {
  pdl_begin();
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  if (threadIdx.x != 0) return;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(bulk_smem + (size_t)BULK_STAGES * BULK_CHUNK);
  const long long total = P.start[P.n];
  const int b = blockIdx.x, nb = gridDim.x;
  long long lo = (long long)(((__int128)total * b) / nb) & ~15ll;
  long long hi = b == nb - 1 ? total : ((long long)(((__int128)total * (b + 1)) / nb) & ~15ll);
  if (b == 0) lo = 0;
  if (hi <= lo) return;
  char* base = nullptr;
  if (P.staged) {
    base = P.heap + P.staging_off + (long long)((epoch_read(P.heap, 0) + 1) & 1) * P.staging_bytes;
  }
  for (int s = 0; s < BULK_STAGES; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  // chunk cursor over [lo, hi): pieces of <= BULK_CHUNK bytes inside one member
  struct Cur {
    int k;
    long long pos;
  };
  auto first = [&](long long at) {
    Cur c{0, at};
    while (c.k < P.n && P.start[c.k + 1] <= at) ++c.k;
    return c;
  };
  auto piece = [&](const Cur& c, const char** src, char** dst) -> int {
    const long long mend = P.start[c.k + 1] < hi ? P.start[c.k + 1] : hi;
    long long len = mend - c.pos;
    if (len > BULK_CHUNK) len = BULK_CHUNK;
    const long long off = c.pos - P.start[c.k];
    *src = P.src[c.k] + off;
    *dst = (P.staged ? base + (long long)(uintptr_t)P.dst[c.k] : P.dst[c.k]) + off;
    return (int)len;
  };
  auto advance = [&](Cur& c, int len) {
    c.pos += len;
    while (c.k < P.n && P.start[c.k + 1] <= c.pos) ++c.k;
  };
  char* dsts[BULK_STAGES];
  int lens[BULK_STAGES];
  Cur ld = first(lo);
  int issued = 0;
  auto issue_load = [&](int i) {
    const int s = i % BULK_STAGES;
    const char* src;
    char* dst;
    const int len = piece(ld, &src, &dst);
    dsts[s] = dst;
    lens[s] = len;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(len)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(bulk_smem + (size_t)s * BULK_CHUNK)),
        "l"(src), "r"(len), "r"(smem_u32(&bar[s]))
        : "memory");
    advance(ld, len);
  };
  while (issued < BULK_STAGES && ld.pos < hi) issue_load(issued++);
  for (int i = 0; i < issued; ++i) {
    const int s = i % BULK_STAGES;
    const unsigned parity = (unsigned)((i / BULK_STAGES) & 1);
    unsigned ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(smem_u32(&bar[s])), "r"(parity)
          : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dsts[s]),
                 "r"(smem_u32(bulk_smem + (size_t)s * BULK_CHUNK)), "r"(lens[s])
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the previous stage's store has finished reading shared memory: refill it
    if (i >= 1 && ld.pos < hi) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue_load(issued++);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace dev
}  // namespace cm
