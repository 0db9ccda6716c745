// sm_100a kernels of the ICCL B200 path.  Nothing here is a contraction, so
// no tensor cores: these are byte movers bound by NVLink (peer destination)
// or HBM (local destination).
//
// K1  iccl_copy_tma   TMA-bulk P2P copy: one elected thread per CTA streams
//                     16 B-aligned tiles global -> smem (cp.async.bulk +
//                     mbarrier complete_tx) -> global (cp.async.bulk
//                     bulk_group), a ring of kStages smem stages; grid capped
//                     at sm_cap CTAs.  Used as the backup path of the
//                     primary-backup pair and as the SM transport.
// K4  stamps          %globaltimer t1 at the first CTA's start and t2 at the
//                     last CTA's end, written to a host-mapped KernelStamp
//                     the proxy turns into a monitor record;
//                     K1, K5 (sends) and K6 carry it, so every op the SM paths
//                     move yields a WR/WC record.
// K2  gather rows     MoE dispatch pack: dst[i] = src[idx[i]] (16 B vectors).
// K3  scatter rows    MoE combine unpack: dst[idx[i]] = src[i].
// K10 combine pull    fused MoE combine: the reverse alltoallv as NVLink loads
//                     from the expert ranks' tensors + K3's scatter.
// K9  backup attempt  the pre-enqueued backup of an armed transfer: CTS
//                     probe on request, K1 over the suffix after a switch.
// K8  dispatch push   fused MoE dispatch: K2's expand form storing every
//                     routed row straight into the owning rank's receive
//                     buffer (NVLink), with K6's ready / done handshake.
#include <cuda_runtime.h>
#include <stdint.h>

#include "iccl_internal.h"

namespace iccl {

namespace {

constexpr int kStages = 4;
constexpr int kTile = 32 * 1024;  // 4 x 32 KB stages: measured best of {4x32K, 8x16K} (probes/)
constexpr int kCopyThreads = 128;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void stamp_begin(KernelStamp* st) {
  if (st && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t = globaltimer();
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&st->t1), "l"(t) : "memory");
  }
}

// Last CTA to finish stamps t2 (system-scope release so the host sees data
// written before it).
__device__ __forceinline__ void stamp_end(KernelStamp* st) {
  if (!st) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned int prev = atomicAdd_system(&st->ctas_done, 1u);
    if (prev == gridDim.x - 1) {
      unsigned long long t = globaltimer();
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&st->t2), "l"(t) : "memory");
    }
  }
}

// Byte-granular copy for heads/tails and mutually misaligned buffers.
__device__ __forceinline__ void copy_bytes(const char* __restrict__ src, char* __restrict__ dst, size_t n,
                                           size_t tid, size_t nthreads) {
  for (size_t i = tid; i < n; i += nthreads) dst[i] = src[i];
}

// 16 B vector copy, grid-stride with 4 loads in flight per thread.
__device__ __forceinline__ void copy_vec16(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16,
                                           size_t tid, size_t nthreads) {
  size_t i = tid;
  for (; i + 3 * nthreads < n16; i += 4 * nthreads) {
    int4 v0, v1, v2, v3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w) : "l"(src + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w) : "l"(src + i + nthreads));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v2.x), "=r"(v2.y), "=r"(v2.z), "=r"(v2.w) : "l"(src + i + 2 * nthreads));
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v3.x), "=r"(v3.y), "=r"(v3.z), "=r"(v3.w) : "l"(src + i + 3 * nthreads));
    dst[i] = v0;
    dst[i + nthreads] = v1;
    dst[i + 2 * nthreads] = v2;
    dst[i + 3 * nthreads] = v3;
  }
  for (; i < n16; i += nthreads) dst[i] = src[i];
}

// The TMA ring of one CTA: tiles blockIdx.x, blockIdx.x + gridDim.x, ... of
// the 16 B-aligned body, global -> smem (cp.async.bulk + mbarrier
// complete_tx) -> global (bulk_group), kStages stages in flight, driven by
// thread 0; the < 16 B head and tail go with byte loads by warps 1..3 of
// CTA 0.  All bulk stores are complete (visible) when it returns.
__device__ __forceinline__ void tma_copy(const char* __restrict__ src, char* __restrict__ dst, size_t head,
                                         size_t body, size_t tail, char* smem, uint64_t* mbar) {
  if (blockIdx.x == 0 && threadIdx.x >= 32) {
    copy_bytes(src, dst, head, threadIdx.x - 32, blockDim.x - 32);
    copy_bytes(src + head + body, dst + head + body, tail, threadIdx.x - 32, blockDim.x - 32);
  }
  if (threadIdx.x == 0 && body > 0) {
    const char* s = src + head;
    char* d = dst + head;
    for (int i = 0; i < kStages; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t ntiles = (body + kTile - 1) / kTile;
    const size_t first = blockIdx.x;
    const size_t mine = first < ntiles ? (ntiles - first + gridDim.x - 1) / gridDim.x : 0;
    auto issue_load = [&](size_t j) {
      const size_t off = (first + j * gridDim.x) * (size_t)kTile;
      const uint32_t bytes = (uint32_t)min((size_t)kTile, body - off);
      const int st = (int)(j % kStages);
      const uint32_t mb = smem_u32(&mbar[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + (size_t)st * kTile)),
          "l"(s + off), "r"(bytes), "r"(mb)
          : "memory");
    };
    for (size_t j = 0; j < mine && j < (size_t)kStages; j++) issue_load(j);
    for (size_t j = 0; j < mine; j++) {
      const int st = (int)(j % kStages);
      const uint32_t mb = smem_u32(&mbar[st]);
      const uint32_t parity = (uint32_t)((j / kStages) & 1);
      uint32_t ready = 0;
      while (!ready)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ready)
            : "r"(mb), "r"(parity)
            : "memory");
      const size_t off = (first + j * gridDim.x) * (size_t)kTile;
      const uint32_t bytes = (uint32_t)min((size_t)kTile, body - off);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + off),
                   "r"(smem_u32(smem + (size_t)st * kTile)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (j + kStages < mine) {
        // the stage is reused once its store has read it out of smem
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue_load(j + kStages);
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// K1.  src/dst share the same alignment mod 16 (checked by the launcher).
__global__ void __launch_bounds__(kCopyThreads) iccl_copy_tma(const char* __restrict__ src, char* __restrict__ dst,
                                                              size_t head, size_t body, size_t tail,
                                                              KernelStamp* stamp, const uint32_t* resume,
                                                              uint32_t chunk) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[kStages];
  if (resume) {  // conditional chunk of a backup attempt: skip what the primary delivered
    uint32_t r;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(r) : "l"(resume) : "memory");
    if (chunk < r) return;
  }
  stamp_begin(stamp);
  tma_copy(src, dst, head, body, tail, smem, mbar);
  stamp_end(stamp);
}

// K9: the backup attempt of an armed transfer (iccl_internal.h BackupOp),
// one launch per transfer on the channel's backup stream behind a wait on
// `go`.  Thread 0 of CTA 0 is the controller: it spins on the watchdog's ctl
// word and the primary's p_fin until it can decide, runs the CTS probe when
// asked, and publishes the decision through w->dec, which the other CTAs
// poll.  A transfer that never fails costs one near-empty launch: the
// primary's end opens `go` with p_fin already set.
__device__ __forceinline__ uint32_t ld_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// K9a: the controller, one warp (lane 0 works), launched right behind the
// primary's enqueue on the backup stream: it waits for `go` inside the
// kernel rather than parking the stream on a stream-memory wait (a parked
// stream was measured to cost every other stream of the GPU ~50 us per op),
// then decides.  Polls back off with __nanosleep.
// The primary path can carry the CTS: not Down, or its gate open again.
__device__ __forceinline__ bool probe_path_open(const BackupOp& op) {
  const uint32_t g = ld_sys(&op.w->pgate);
  return g == 0 || ld_sys(op.gates + g - 1) != 0;
}

__global__ void __launch_bounds__(32) iccl_backup_ctl(const __grid_constant__ BackupOp op) {
  if (threadIdx.x != 0) return;
  ArmedWords* w = op.w;
  const unsigned long long t0 = globaltimer();
  uint32_t dec = kDecNone;
  bool probed = false;
  while (ld_sys(&w->go) == 0 && ld_sys(&w->ctl) != kCtlAbort) __nanosleep(256);
  while (dec == kDecNone) {
    const uint32_t ctl = ld_sys(&w->ctl);
    if (ctl == kCtlSwitch) {
      dec = kDecCopy;
    } else if (ctl == kCtlAbort) {
      dec = kDecExit;
    } else if (ld_sys(&w->p_fin)) {
      dec = ld_sys(&w->ctl) == kCtlSwitch ? kDecCopy : kDecExit;  // a switch racing the primary's end still copies
    } else if (ctl == kCtlProbe && !probed && probe_path_open(op)) {
      // the CTS crosses the primary path: lost while its gate is closed
      int4 v;
      asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(op.probe_src) : "memory");
      asm volatile("st.volatile.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(op.probe_dst), "r"(v.x), "r"(v.y),
                   "r"(v.z), "r"(v.w) : "memory");
      __threadfence_system();
      st_sys(&w->probe_done, 1u);
      probed = true;
    } else {
      __nanosleep(256);
    }
  }
  const uint32_t bg = ld_sys(&w->bgate);
  if (dec == kDecCopy && bg) {  // the backup path itself is Down: wait for it (or the abort)
    while (ld_sys(op.gates + bg - 1) == 0 && ld_sys(&w->ctl) != kCtlAbort) __nanosleep(256);
    if (ld_sys(&w->ctl) == kCtlAbort) dec = kDecExit;
  }
  (void)t0;
  // the copy grid reads the decision from this GPU's memory (a host-mapped
  // read by each of its CTAs cost ~12 us per armed op, profiles/r02 §4)
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(op.dec_dev), "r"((op.seq << 2) | dec) : "memory");
  st_sys(&w->dec, dec);
}

// K9b: the copy grid, behind K9a on the same stream, so the decision is
// final when it starts: nothing to do unless the watchdog switched.
__global__ void __launch_bounds__(kCopyThreads) iccl_backup_attempt(const __grid_constant__ BackupOp op) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[kStages];
  __shared__ uint32_t s_dec;
  ArmedWords* w = op.w;
  if (threadIdx.x == 0) {
    uint32_t v;
    do {  // K9a precedes on the stream: the word is final, the loop only guards the generation
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.dec_dev) : "memory");
    } while ((v >> 2) != (op.seq & 0x3fffffffu));
    s_dec = v & 3u;
  }
  __syncthreads();
  if (s_dec != kDecCopy) return;
  const uint32_t r = ld_sys(&w->resume);
  for (uint32_t k = r; k < op.nchunks; k++) {
    const size_t off = (size_t)k * op.chunk, n = min(op.chunk, op.bytes - off);
    const uintptr_t a = (uintptr_t)(op.src + off);
    size_t head = (16 - (a & 15)) & 15;
    if (head > n) head = n;
    const size_t body = (n - head) & ~(size_t)15, tail = n - head - body;
    KernelStamp* st = &op.ring[(op.stamp_base + k) % op.ring_slots];
    stamp_begin(st);
    tma_copy(op.src + off, op.dst + off, head, body, tail, smem, mbar);
    stamp_end(st);
  }
}

// K6: the direct path for mid-size messages.  Launched on the issuing
// side's own user stream by the side that arrived second at the rendezvous
// (no proxy, no side stream, no stream memop on this side): every CTA waits
// for the other side's ready flag (its user stream reached the op), moves its
// tiles straight between the two tensors (push or pull, zero-copy), and the
// last CTA releases both done flags.  Waits give up after 10 s (error flag).
__global__ void __launch_bounds__(kCopyThreads) iccl_direct_copy(DirectOp op) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[kStages];
  // one thread of CTA 0 polls the ready flag (host-mapped, or with device
  // flags a word in the peer GPU's memory read over NVLink); the other CTAs
  // wait on a word in this GPU's memory that it releases (gen-tagged, never
  // reset), so only one poller leaves the GPU
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    uint32_t v;
    if (blockIdx.x == 0) {
      do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(op.peer_ready) : "memory");
        if ((int32_t)(v - op.peer_ready_gen) < 0 && globaltimer() - t0 > 10000000000ull) {
          *op.error = 1;
          break;
        }
      } while ((int32_t)(v - op.peer_ready_gen) < 0);
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(op.go), "r"(op.my_done_gen) : "memory");
      if (op.stamp) {  // K4: the WR is posted once the other side is ready
        const unsigned long long t = globaltimer();
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t1), "l"(t) : "memory");
      }
    } else {
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.go) : "memory");
        if (v != op.my_done_gen && globaltimer() - t0 > 10000000000ull) {
          *op.error = 1;
          break;
        }
      } while (v != op.my_done_gen);
    }
  }
  __syncthreads();
  if (op.vec) {
    // small ops: every thread moves 16 B vectors straight between the two
    // tensors, no shared-memory round trip before the first store
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    copy_bytes(op.src, op.dst, op.head, tid, nt);
    copy_vec16((const int4*)(op.src + op.head), (int4*)(op.dst + op.head), op.body / 16, tid, nt);
    copy_bytes(op.src + op.head + op.body, op.dst + op.head + op.body, op.tail, tid, nt);
  } else {
    tma_copy(op.src, op.dst, op.head, op.body, op.tail, smem, mbar);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(op.counter, 1u) == gridDim.x - 1) {
      atomicExch(op.counter, 0u);
      __threadfence_system();
      if (op.stamp) {  // K4: the WC (every CTA's bulk stores are complete)
        const unsigned long long t = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t2), "l"(t) : "memory");
      }
      if (op.peer_done_dev)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.peer_done_dev), "r"(op.peer_done_gen) : "memory");
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.peer_done), "r"(op.peer_done_gen) : "memory");
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.my_done), "r"(op.my_done_gen) : "memory");
    }
  }
}

// Fallback for buffers whose addresses differ mod 16: byte copy.
__global__ void __launch_bounds__(512) iccl_copy_unaligned(const char* __restrict__ src, char* __restrict__ dst,
                                                           size_t n, KernelStamp* stamp, const uint32_t* resume,
                                                           uint32_t chunk) {
  if (resume) {
    uint32_t r;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(r) : "l"(resume) : "memory");
    if (chunk < r) return;
  }
  stamp_begin(stamp);
  copy_bytes(src, dst, n, blockIdx.x * (size_t)blockDim.x + threadIdx.x, (size_t)gridDim.x * blockDim.x);
  stamp_end(stamp);
}

__global__ void iccl_read_globaltimer(unsigned long long* out) {
  unsigned long long t = globaltimer();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(out), "l"(t) : "memory");
}

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// streaming store: evict-first in L2, so the rows being written do not push
// out data that is re-read (K2's token matrix is read k times)
__device__ __forceinline__ void st_cs(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// One warp moves one row: 16 B per lane per step (512 B coalesced per warp
// step), four independent loads in flight per lane before their stores.
__device__ __forceinline__ void warp_copy_row(const int4* __restrict__ s, int4* __restrict__ d, int64_t row16,
                                              int lane) {
  int64_t c = lane;
  for (; c + 96 < row16; c += 128) {
    const int4 v0 = ld_nc(s + c), v1 = ld_nc(s + c + 32), v2 = ld_nc(s + c + 64), v3 = ld_nc(s + c + 96);
    st_cs(d + c, v0);
    st_cs(d + c + 32, v1);
    st_cs(d + c + 64, v2);
    st_cs(d + c + 96, v3);
  }
  for (; c < row16; c += 32) st_cs(d + c, ld_nc(s + c));
}

// K2: dispatch pack, dst row r <- src row idx[r].
__global__ void __launch_bounds__(256) iccl_gather_rows(const int4* __restrict__ src, int4* __restrict__ dst,
                                                       const int64_t* __restrict__ idx, int64_t n_rows,
                                                       int64_t row16) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nwarps) warp_copy_row(src + idx[r] * row16, dst + r * row16, row16, lane);
}

// K2 (expand form): dispatch pack reading every token once: warp per token
// t, each 16 B column chunk loaded once and stored to its k packed rows
// dst[pos[t*k + j]].  DRAM traffic = T rows read + T*k rows written, versus
// T*k reads for the gather form (measured: the gather's re-reads miss L2,
// profiles/r01/ncu/k2k3_full_summary.csv).
// Each token row is split into `parts` column ranges, one warp each, so T
// tokens give T * parts warps (a whole-row warp left ~1/3 of the warp slots
// busy at T = 4096: ncu, profiles/r01/ncu/k2_expand_k3_summary.csv).
__global__ void __launch_bounds__(256) iccl_expand_rows(const int4* __restrict__ src, int4* __restrict__ dst,
                                                       const int64_t* __restrict__ pos, int64_t n_src, int k,
                                                       int64_t row16, int parts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t span = (row16 + parts - 1) / parts;
  for (int64_t w = warp; w < n_src * parts; w += nwarps) {
    const int64_t t = w / parts;
    const int64_t c0 = (w % parts) * span, c1 = min(row16, c0 + span);
    const int4* s = src + t * row16;
    const int64_t* p = pos + t * k;
    int64_t c = c0 + lane;
    for (; c + 96 < c1; c += 128) {
      const int4 v0 = ld_nc(s + c), v1 = ld_nc(s + c + 32), v2 = ld_nc(s + c + 64), v3 = ld_nc(s + c + 96);
      for (int j = 0; j < k; j++) {
        int4* d = dst + p[j] * row16;
        st_cs(d + c, v0);
        st_cs(d + c + 32, v1);
        st_cs(d + c + 64, v2);
        st_cs(d + c + 96, v3);
      }
    }
    for (; c < c1; c += 32) {
      const int4 v = ld_nc(s + c);
      for (int j = 0; j < k; j++) st_cs(dst + p[j] * row16 + c, v);
    }
  }
}

// K8: fused MoE dispatch (K2's expand form + the alltoallv push in one
// kernel, no staging buffer): each token row is read once and each of its k
// routed copies is stored straight into the receive buffer of the rank that
// owns the copy's packed position — over NVLink into an IPC mapping of the
// peer's tensor, or locally for the self segment (no
// intermediate buffer between the producer and the wire).
//
// Entry: the first CTA to arrive (a ticket, not blockIdx 0, so no CTA waits
// on one that is not resident yet) polls every destination's ready flag (its
// user stream reached the receive) and releases the others through a
// gen-tagged word in local HBM.  Body: a warp per (token, column part); lanes
// 0..k-1 resolve the k destination row pointers once (binary search of the
// packed row over the per-rank ranges, in shared memory) and the warp
// broadcasts them with shuffles.  Exit: the last CTA releases every
// destination's done flag and this rank's send-op done flags (system scope,
// after a system fence, like K6).
__device__ __forceinline__ int fused_dest_of(const int64_t* hi, int n, int64_t p) {
  int lo = 0, up = n - 1;  // first d with p < hi[d]
  while (lo < up) {
    const int mid = (lo + up) >> 1;
    if (p < hi[mid]) up = mid;
    else lo = mid + 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256, 5) iccl_dispatch_push(const __grid_constant__ DispatchOp op) {
  __shared__ int64_t s_lo[kMaxFusedRanks], s_hi[kMaxFusedRanks];
  __shared__ int4* s_seg[kMaxFusedRanks];
  for (int d = threadIdx.x; d < op.n; d += blockDim.x) {
    s_lo[d] = op.d[d].lo;
    s_hi[d] = op.d[d].hi;
    s_seg[d] = (int4*)op.d[d].seg;
  }
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    if (atomicAdd(op.ticket, 1u) == 0) {
      for (int d = 0; d < op.n; d++) {
        if (!op.d[d].ready) continue;
        uint32_t v;
        do {
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(op.d[d].ready) : "memory");
          if ((int32_t)(v - op.d[d].ready_gen) < 0 && globaltimer() - t0 > 10000000000ull) {
            *op.error = 1;
            break;
          }
        } while ((int32_t)(v - op.d[d].ready_gen) < 0);
      }
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(op.go), "r"(op.go_gen) : "memory");
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t1), "l"(t) : "memory");
      }
    } else {
      uint32_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.go) : "memory");
        if (v != op.go_gen && globaltimer() - t0 > 10000000000ull) {
          *op.error = 1;
          break;
        }
      } while (v != op.go_gen);
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t row16 = op.row16;
  const int64_t span = (row16 + op.parts - 1) / op.parts;
  for (int64_t w = warp; w < op.n_tokens * op.parts; w += nwarps) {
    const int64_t t = w / op.parts;
    const int64_t c0 = (w % op.parts) * span, c1 = min(row16, c0 + span);
    const int4* s = op.tokens + t * row16;
    int4* mine = nullptr;
    if (lane < op.k) {
      const int64_t p = op.pos[t * op.k + lane];
      const int d = fused_dest_of(s_hi, op.n, p);
      mine = s_seg[d] + (p - s_lo[d]) * row16;
    }
    // warp-uniform loops: every lane takes part in the pointer shuffles
    int64_t cb = c0;
    for (; cb + 128 <= c1; cb += 128) {
      const int64_t c = cb + lane;
      const int4 v0 = ld_nc(s + c), v1 = ld_nc(s + c + 32), v2 = ld_nc(s + c + 64), v3 = ld_nc(s + c + 96);
      for (int j = 0; j < op.k; j++) {
        int4* d = (int4*)__shfl_sync(0xffffffffu, (unsigned long long)mine, j);
        st_cs(d + c, v0);
        st_cs(d + c + 32, v1);
        st_cs(d + c + 64, v2);
        st_cs(d + c + 96, v3);
      }
    }
    for (; cb < c1; cb += 32) {
      const int64_t c = cb + lane;
      const int4 v = c < c1 ? ld_nc(s + c) : int4{0, 0, 0, 0};
      for (int j = 0; j < op.k; j++) {
        int4* d = (int4*)__shfl_sync(0xffffffffu, (unsigned long long)mine, j);
        if (c < c1) st_cs(d + c, v);
      }
    }
  }
  __threadfence_system();  // every thread's row stores, before the CTA's arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(op.counter, 1u) == gridDim.x - 1) {
      atomicExch(op.counter, 0u);
      atomicExch(op.ticket, 0u);
      __threadfence_system();
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t2), "l"(t) : "memory");
      }
      for (int d = 0; d < op.n; d++) {
        if (op.d[d].done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].done), "r"(op.d[d].done_gen) : "memory");
        if (op.d[d].my_done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].my_done), "r"(op.d[d].my_done_gen)
                       : "memory");
      }
    }
  }
}

// K10: fused MoE combine (iccl_internal.h CombineOp).  The mirror of K8:
// the receiving (token) rank runs it and pulls — each warp loads one column
// part of a packed row from the expert rank's tensor over NVLink (four
// 16-byte loads in flight per lane) and stores it at the row's (token, k)
// slot; same entry ticket / exit counter handshake as K8, with the roles of
// the flags swapped (it waits for the sources' ready flags and releases their
// done flags).
__global__ void __launch_bounds__(256, 5) iccl_combine_pull(const __grid_constant__ CombineOp op) {
  __shared__ int64_t s_lo[kMaxFusedRanks], s_hi[kMaxFusedRanks];
  __shared__ const int4* s_seg[kMaxFusedRanks];
  for (int d = threadIdx.x; d < op.n; d += blockDim.x) {
    s_lo[d] = op.d[d].lo;
    s_hi[d] = op.d[d].hi;
    s_seg[d] = (const int4*)op.d[d].seg;
  }
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    if (atomicAdd(op.ticket, 1u) == 0) {
      for (int d = 0; d < op.n; d++) {
        if (!op.d[d].ready) continue;
        uint32_t v;
        do {
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(op.d[d].ready) : "memory");
          if ((int32_t)(v - op.d[d].ready_gen) < 0 && globaltimer() - t0 > 10000000000ull) {
            *op.error = 1;
            break;
          }
        } while ((int32_t)(v - op.d[d].ready_gen) < 0);
      }
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(op.go), "r"(op.go_gen) : "memory");
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t1), "l"(t) : "memory");
      }
    } else {
      uint32_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.go) : "memory");
        if (v != op.go_gen && globaltimer() - t0 > 10000000000ull) {
          *op.error = 1;
          break;
        }
      } while (v != op.go_gen);
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t row16 = op.row16;
  const int64_t span = (row16 + op.parts - 1) / op.parts;
  for (int64_t w = warp; w < op.n_rows * op.parts; w += nwarps) {
    // rows visited in a stride permutation (stride coprime to n_rows): the
    // warps in flight at any moment pull from every source segment at once,
    // so the local copy of the self segment overlaps the NVLink loads
    const int64_t r = (int64_t)(((unsigned long long)(w / op.parts) * op.stride) % (unsigned long long)op.n_rows);
    const int64_t c0 = (w % op.parts) * span, c1 = min(row16, c0 + span);
    const int d = fused_dest_of(s_hi, op.n, r);
    const int4* src = s_seg[d] + (r - s_lo[d]) * row16;
    int4* dst = op.out + op.order[r] * row16;
    int64_t c = c0 + lane;
    for (; c + 96 < c1; c += 128) {
      const int4 v0 = ld_nc(src + c), v1 = ld_nc(src + c + 32), v2 = ld_nc(src + c + 64), v3 = ld_nc(src + c + 96);
      st_cs(dst + c, v0);
      st_cs(dst + c + 32, v1);
      st_cs(dst + c + 64, v2);
      st_cs(dst + c + 96, v3);
    }
    for (; c < c1; c += 32) st_cs(dst + c, ld_nc(src + c));
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(op.counter, 1u) == gridDim.x - 1) {
      atomicExch(op.counter, 0u);
      atomicExch(op.ticket, 0u);
      __threadfence_system();
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t2), "l"(t) : "memory");
      }
      for (int d = 0; d < op.n; d++) {
        if (op.d[d].done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].done), "r"(op.d[d].done_gen) : "memory");
        if (op.d[d].my_done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].my_done), "r"(op.d[d].my_done_gen)
                       : "memory");
      }
    }
  }
}

// K2, TMA form: one warp per CTA.  Lane 0 streams each (token, tile) item
// into a ring of kExpStages shared-memory stages (cp.async.bulk
// global->shared, mbarrier complete_tx); lanes 0..k-1 then each issue one
// bulk store of the stage to their packed row (cp.async.bulk shared->global,
// one bulk group per lane per item).  No register copies at all: the copy
// engines of the SM (TMA) move the bytes; the pos entries of the next item
// are loaded one item ahead.  Rows are split into tiles of <= tile bytes
// (16-byte multiples).
constexpr int kExpStages = 4;
__global__ void __launch_bounds__(32) iccl_expand_tma(const char* __restrict__ src, char* __restrict__ dst,
                                                      const int64_t* __restrict__ pos, int64_t n_src, int k,
                                                      int64_t row_bytes, int64_t tile, int64_t ntile) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[kExpStages];
  const int lane = threadIdx.x;
  const int64_t items = n_src * ntile;
  const int64_t first = blockIdx.x;
  const int64_t mine = first < items ? (items - first + gridDim.x - 1) / gridDim.x : 0;
  if (lane == 0) {
    for (int i = 0; i < kExpStages; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue_load = [&](int64_t j) {
    const int64_t it = first + j * gridDim.x, t = it / ntile, off = (it % ntile) * tile;
    const uint32_t bytes = (uint32_t)min(tile, row_bytes - off);
    const int st = (int)(j % kExpStages);
    const uint32_t mb = smem_u32(&mbar[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (size_t)st * tile)),
        "l"(src + t * row_bytes + off), "r"(bytes), "r"(mb)
        : "memory");
  };
  if (lane == 0)
    for (int64_t j = 0; j < mine && j < kExpStages; j++) issue_load(j);
  int64_t p_next = (mine > 0 && lane < k) ? pos[(first / ntile) * k + lane] : 0;
  for (int64_t j = 0; j < mine; j++) {
    const int64_t it = first + j * gridDim.x, t = it / ntile, off = (it % ntile) * tile;
    const uint32_t bytes = (uint32_t)min(tile, row_bytes - off);
    const int64_t p = p_next;
    if (j + 1 < mine && lane < k) p_next = pos[((first + (j + 1) * gridDim.x) / ntile) * k + lane];
    const int st = (int)(j % kExpStages);
    const uint32_t mb = smem_u32(&mbar[st]);
    const uint32_t parity = (uint32_t)((j / kExpStages) & 1);
    uint32_t ready = 0;
    while (!ready)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ready)
          : "r"(mb), "r"(parity)
          : "memory");
    if (lane < k) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + p * row_bytes + off),
                   "r"(smem_u32(smem + (size_t)st * tile)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (j + kExpStages < mine) {
      // the stage is reloaded once every lane's store has read it out of smem
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      if (lane == 0) issue_load(j + kExpStages);
    }
    (void)t;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K8, TMA form: K2's TMA ring (iccl_expand_tma) with K8's destinations and
// handshake: lane 0 of the first CTA to arrive polls every destination's
// ready flag and releases the others; lanes 0..k-1 resolve their packed
// row's owner (binary search over the per-rank ranges) and bulk-store the
// stage straight into that rank's receive buffer (NVLink for a peer); the
// last CTA releases the done flags after its bulk stores completed.
__global__ void __launch_bounds__(32) iccl_dispatch_tma(const __grid_constant__ DispatchOp op, int64_t tile,
                                                        int64_t ntile) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[kExpStages];
  __shared__ int64_t s_lo[kMaxFusedRanks], s_hi[kMaxFusedRanks];
  __shared__ char* s_seg[kMaxFusedRanks];
  const int lane = threadIdx.x;
  for (int d = lane; d < op.n; d += 32) {
    s_lo[d] = op.d[d].lo;
    s_hi[d] = op.d[d].hi;
    s_seg[d] = op.d[d].seg;
  }
  if (lane == 0) {
    const unsigned long long t0 = globaltimer();
    if (atomicAdd(op.ticket, 1u) == 0) {
      for (int d = 0; d < op.n; d++) {
        if (!op.d[d].ready) continue;
        uint32_t v;
        do {
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(op.d[d].ready) : "memory");
          if ((int32_t)(v - op.d[d].ready_gen) < 0 && globaltimer() - t0 > 10000000000ull) {
            *op.error = 1;
            break;
          }
        } while ((int32_t)(v - op.d[d].ready_gen) < 0);
      }
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(op.go), "r"(op.go_gen) : "memory");
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t1), "l"(t) : "memory");
      }
    } else {
      uint32_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.go) : "memory");
        if (v != op.go_gen && globaltimer() - t0 > 10000000000ull) {
          *op.error = 1;
          break;
        }
      } while (v != op.go_gen);
    }
    for (int i = 0; i < kExpStages; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const char* src = (const char*)op.tokens;
  const int64_t row_bytes = op.row16 * 16;
  const int64_t items = op.n_tokens * ntile;
  const int64_t first = blockIdx.x;
  const int64_t mine = first < items ? (items - first + gridDim.x - 1) / gridDim.x : 0;
  auto issue_load = [&](int64_t j) {
    const int64_t it = first + j * gridDim.x, t = it / ntile, off = (it % ntile) * tile;
    const uint32_t bytes = (uint32_t)min(tile, row_bytes - off);
    const int st = (int)(j % kExpStages);
    const uint32_t mb = smem_u32(&mbar[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (size_t)st * tile)),
        "l"(src + t * row_bytes + off), "r"(bytes), "r"(mb)
        : "memory");
  };
  if (lane == 0)
    for (int64_t j = 0; j < mine && j < kExpStages; j++) issue_load(j);
  int64_t p_next = (mine > 0 && lane < op.k) ? op.pos[(first / ntile) * op.k + lane] : 0;
  for (int64_t j = 0; j < mine; j++) {
    const int64_t it = first + j * gridDim.x, off = (it % ntile) * tile;
    const uint32_t bytes = (uint32_t)min(tile, row_bytes - off);
    const int64_t p = p_next;
    if (j + 1 < mine && lane < op.k) p_next = op.pos[((first + (j + 1) * gridDim.x) / ntile) * op.k + lane];
    const int st = (int)(j % kExpStages);
    const uint32_t mb = smem_u32(&mbar[st]);
    const uint32_t parity = (uint32_t)((j / kExpStages) & 1);
    uint32_t ready = 0;
    while (!ready)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ready)
          : "r"(mb), "r"(parity)
          : "memory");
    if (lane < op.k) {
      const int d = fused_dest_of(s_hi, op.n, p);
      char* dp = s_seg[d] + (p - s_lo[d]) * row_bytes + off;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dp),
                   "r"(smem_u32(smem + (size_t)st * tile)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (j + kExpStages < mine) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      if (lane == 0) issue_load(j + kExpStages);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // this lane's stores performed
  __threadfence_system();
  __syncwarp();
  if (lane == 0) {
    if (atomicAdd(op.counter, 1u) == gridDim.x - 1) {
      atomicExch(op.counter, 0u);
      atomicExch(op.ticket, 0u);
      __threadfence_system();
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t2), "l"(t) : "memory");
      }
      for (int d = 0; d < op.n; d++) {
        if (op.d[d].done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].done), "r"(op.d[d].done_gen) : "memory");
        if (op.d[d].my_done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].my_done), "r"(op.d[d].my_done_gen)
                       : "memory");
      }
    }
  }
}

// K10, TMA form: lane 0 of each one-warp CTA bulk-loads (row, tile) items
// straight from the source rank's tensor (NVLink for a peer) into a ring of
// shared-memory stages and bulk-stores each to its out row; rows are visited
// in K10's coprime-stride order.  Same handshake as K10.
__global__ void __launch_bounds__(32) iccl_combine_tma(const __grid_constant__ CombineOp op, int64_t tile,
                                                       int64_t ntile) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[kExpStages];
  __shared__ int64_t s_lo[kMaxFusedRanks], s_hi[kMaxFusedRanks];
  __shared__ const char* s_seg[kMaxFusedRanks];
  const int lane = threadIdx.x;
  for (int d = lane; d < op.n; d += 32) {
    s_lo[d] = op.d[d].lo;
    s_hi[d] = op.d[d].hi;
    s_seg[d] = op.d[d].seg;
  }
  if (lane == 0) {
    const unsigned long long t0 = globaltimer();
    if (atomicAdd(op.ticket, 1u) == 0) {
      for (int d = 0; d < op.n; d++) {
        if (!op.d[d].ready) continue;
        uint32_t v;
        do {
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(op.d[d].ready) : "memory");
          if ((int32_t)(v - op.d[d].ready_gen) < 0 && globaltimer() - t0 > 10000000000ull) {
            *op.error = 1;
            break;
          }
        } while ((int32_t)(v - op.d[d].ready_gen) < 0);
      }
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(op.go), "r"(op.go_gen) : "memory");
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t1), "l"(t) : "memory");
      }
    } else {
      uint32_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.go) : "memory");
        if (v != op.go_gen && globaltimer() - t0 > 10000000000ull) {
          *op.error = 1;
          break;
        }
      } while (v != op.go_gen);
    }
    for (int i = 0; i < kExpStages; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane == 0) {
    const int64_t row_bytes = op.row16 * 16;
    const int64_t items = op.n_rows * ntile;
    const int64_t first = blockIdx.x;
    const int64_t mine = first < items ? (items - first + gridDim.x - 1) / gridDim.x : 0;
    auto item = [&](int64_t j, int64_t* r, int64_t* off) {
      const int64_t it = first + j * gridDim.x;
      *r = (int64_t)(((unsigned long long)(it / ntile) * op.stride) % (unsigned long long)op.n_rows);
      *off = (it % ntile) * tile;
    };
    int64_t orow_ring[kExpStages];  // out rows of the items in flight (loaded with the tile: latency hidden)
    auto issue_load = [&](int64_t j) {
      int64_t r, off;
      item(j, &r, &off);
      orow_ring[j % kExpStages] = op.order[r];
      const int d = fused_dest_of(s_hi, op.n, r);
      const uint32_t bytes = (uint32_t)min(tile, row_bytes - off);
      const int st = (int)(j % kExpStages);
      const uint32_t mb = smem_u32(&mbar[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + (size_t)st * tile)),
          "l"(s_seg[d] + (r - s_lo[d]) * row_bytes + off), "r"(bytes), "r"(mb)
          : "memory");
    };
    for (int64_t j = 0; j < mine && j < kExpStages; j++) issue_load(j);
    for (int64_t j = 0; j < mine; j++) {
      int64_t r, off;
      item(j, &r, &off);
      const int64_t orow = orow_ring[j % kExpStages];
      const uint32_t bytes = (uint32_t)min(tile, row_bytes - off);
      const int st = (int)(j % kExpStages);
      const uint32_t mb = smem_u32(&mbar[st]);
      const uint32_t parity = (uint32_t)((j / kExpStages) & 1);
      uint32_t ready = 0;
      while (!ready)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ready)
            : "r"(mb), "r"(parity)
            : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)op.out + orow * row_bytes + off),
                   "r"(smem_u32(smem + (size_t)st * tile)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (j + kExpStages < mine) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue_load(j + kExpStages);
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __threadfence_system();
    if (atomicAdd(op.counter, 1u) == gridDim.x - 1) {
      atomicExch(op.counter, 0u);
      atomicExch(op.ticket, 0u);
      __threadfence_system();
      if (op.stamp) {
        const unsigned long long t = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&op.stamp->t2), "l"(t) : "memory");
      }
      for (int d = 0; d < op.n; d++) {
        if (op.d[d].done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].done), "r"(op.d[d].done_gen) : "memory");
        if (op.d[d].my_done)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(op.d[d].my_done), "r"(op.d[d].my_done_gen)
                       : "memory");
      }
    }
  }
}

// K3: inverse permutation (combine unpack), dst row idx[r] <- src row r.
__global__ void __launch_bounds__(256) iccl_scatter_rows(const int4* __restrict__ src, int4* __restrict__ dst,
                                                        const int64_t* __restrict__ idx, int64_t n_rows,
                                                        int64_t row16) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += nwarps) warp_copy_row(src + r * row16, dst + idx[r] * row16, row16, lane);
}

// K5: LL eager path.  Block b serves op b of the batch.  A send writes every
// 4-byte word of its payload as an 8-byte {word, seq} line into the peer's
// slot (one 8-byte store: data and flag become visible together, no fence);
// a recv polls each of its lines until the flag equals seq, stores the word,
// and when the whole block is done returns the slot's credit to the sender.
// Credits are per slot (credit[(seq-1) % kLLSlots] = seq): the CTAs of one
// launch finish in any order, so a single "last consumed" word could run
// backwards and let a sender overwrite a slot whose previous message was not
// read yet.  Waits give up after 10 s (error flag) instead of hanging the GPU.
__device__ __forceinline__ bool ll_timed_out(unsigned long long t0) {
  return globaltimer() - t0 > 10000000000ull;
}

constexpr int kLLUnroll = 8;

// The 4-byte word i of an LL message (byte-wise at a misaligned / short end).
__device__ __forceinline__ uint32_t ll_load_word(const char* buf, size_t bytes, size_t i) {
  const size_t off = i * 4;
  if (off + 4 <= bytes && ((uintptr_t)(buf + off) & 3) == 0) return *(const uint32_t*)(buf + off);
  uint32_t w = 0;
  for (int k = 0; k < 4 && off + k < bytes; k++) w |= (uint32_t)(unsigned char)buf[off + k] << (8 * k);
  return w;
}
__device__ __forceinline__ void ll_store_word(char* buf, size_t bytes, size_t i, uint32_t w) {
  const size_t off = i * 4;
  if (off + 4 <= bytes && ((uintptr_t)(buf + off) & 3) == 0) {
    *(uint32_t*)(buf + off) = w;
    return;
  }
  for (int k = 0; k < 4 && off + k < bytes; k++) buf[off + k] = (char)(w >> (8 * k));
}

__global__ void __launch_bounds__(256) iccl_ll_group(LLBatch b) {
  __shared__ int s_op;
  if (threadIdx.x == 0) {
    int op = 0;
    while (op + 1 < b.n && blockIdx.x >= b.d[op + 1].first_blk) op++;
    s_op = op;
  }
  __syncthreads();
  const LLDesc& d = b.d[s_op];
  const uint32_t part = blockIdx.x - d.first_blk;
  const unsigned long long t0 = globaltimer();
  const size_t lines = (d.bytes + 3) / 4;
  const size_t lo = lines * part / d.nblk, hi = lines * (part + 1) / d.nblk;
  uint2* slot = (uint2*)d.slot;
  __shared__ bool s_last;
  if (d.kind == 0) {
    if (d.seq > (uint32_t)kLLSlots) {
      if (threadIdx.x == 0) {
        const uint32_t need = d.seq - kLLSlots;
        const unsigned int* cw = d.credit + (d.seq - 1) % kLLSlots;
        uint32_t c;
        do {
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(c) : "l"(cw) : "memory");
          if (ll_timed_out(t0)) {
            *b.error = 1;
            break;
          }
        } while ((int32_t)(c - need) < 0);
      }
      __syncthreads();
    }
    if (d.stamp && part == 0 && threadIdx.x == 0) {  // K4: WR posted (the slot is free)
      const unsigned long long t = globaltimer();
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&d.stamp->t1), "l"(t) : "memory");
    }
    // kLLUnroll source words loaded before their line stores: the loads of
    // one thread are in flight together instead of one latency per line
    for (size_t i0 = lo + threadIdx.x; i0 < hi; i0 += kLLUnroll * blockDim.x) {
      uint32_t w[kLLUnroll];
#pragma unroll
      for (int j = 0; j < kLLUnroll; j++) {
        const size_t i = i0 + (size_t)j * blockDim.x;
        w[j] = i < hi ? ll_load_word(d.buf, d.bytes, i) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kLLUnroll; j++) {
        const size_t i = i0 + (size_t)j * blockDim.x;
        if (i < hi)
          asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(slot + i), "r"(w[j]), "r"(d.seq) : "memory");
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // last CTA of the op: every CTA read its part of the source
      s_last = d.nblk == 1 || atomicAdd(d.counter, 1u) == d.nblk - 1;
      if (s_last && d.nblk > 1) atomicExch(d.counter, 0u);
      if (s_last && d.stamp) {  // K4: every line of the op is out
        __threadfence_system();
        const unsigned long long t = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&d.stamp->t2), "l"(t) : "memory");
      }
      if (s_last && d.done_flag)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(d.done_flag), "r"(d.done_gen) : "memory");
    }
  } else {
    // kLLUnroll lines polled at once (their first loads in flight together);
    // a line not there yet is re-polled on its own
    for (size_t i0 = lo + threadIdx.x; i0 < hi; i0 += kLLUnroll * blockDim.x) {
      uint32_t w[kLLUnroll], f[kLLUnroll];
#pragma unroll
      for (int j = 0; j < kLLUnroll; j++) {
        const size_t i = i0 + (size_t)j * blockDim.x;
        f[j] = d.seq;
        if (i < hi)
          asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(w[j]), "=r"(f[j]) : "l"(slot + i) : "memory");
      }
#pragma unroll
      for (int j = 0; j < kLLUnroll; j++) {
        const size_t i = i0 + (size_t)j * blockDim.x;
        if (i >= hi) continue;
        while (f[j] != d.seq) {
          if (ll_timed_out(t0)) {
            *b.error = 1;
            break;
          }
          asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(w[j]), "=r"(f[j]) : "l"(slot + i) : "memory");
        }
        ll_store_word(d.buf, d.bytes, i, w[j]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = d.nblk == 1 || atomicAdd(d.counter, 1u) == d.nblk - 1;
      if (s_last) {
        if (d.nblk > 1) {
          atomicExch(d.counter, 0u);
          __threadfence();  // the other CTAs' payload stores are ordered before the credit / done
        }
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(d.credit + (d.seq - 1) % kLLSlots), "r"(d.seq)
                     : "memory");
        if (d.done_flag)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(d.done_flag), "r"(d.done_gen) : "memory");
      }
    }
  }
}

bool smem_configured = false;
// Dynamic shared memory of the TMA-ring kernels (K1, K1 chunks, K6), once.
cudaError_t configure_smem() {
  if (smem_configured) return cudaSuccess;
  const void* fns[] = {(const void*)iccl_copy_tma, (const void*)iccl_direct_copy, (const void*)iccl_backup_attempt};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kTile);
    if (e != cudaSuccess) return e;
  }
  smem_configured = true;
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_ll(const LLBatch& b, cudaStream_t st) {
  if (b.n <= 0) return cudaSuccess;
  const unsigned blocks = b.d[b.n - 1].first_blk + b.d[b.n - 1].nblk;
  iccl_ll_group<<<blocks, 256, 0, st>>>(b);
  return cudaGetLastError();
}

// K7.  One thread polls each done flag in turn (the flags live in the
// host-mapped control block); the stream continues when the kernel exits.
__global__ void __launch_bounds__(32) iccl_wait_flags(WaitList wl) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = globaltimer();
  for (int i = 0; i < wl.n; i++) {
    uint32_t v;
    unsigned polls = 0;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(wl.addr[i]) : "memory");
      if ((int32_t)(v - wl.gen[i]) >= 0) break;
      if (wl.alt[i] && (++polls & 63) == 0)
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(wl.alt[i]) : "memory");
      if ((int32_t)(v - wl.gen[i]) < 0 && globaltimer() - t0 > 10000000000ull) {
        *wl.error = 1;
        return;
      }
    } while ((int32_t)(v - wl.gen[i]) < 0);
  }
}

cudaError_t launch_wait(const WaitList& wl, cudaStream_t st) {
  if (wl.n <= 0) return cudaSuccess;
  iccl_wait_flags<<<1, 32, 0, st>>>(wl);
  return cudaGetLastError();
}

cudaError_t launch_direct(DirectOp op, size_t bytes, int ctas, cudaStream_t st, int* grid_out) {
  const uintptr_t s = (uintptr_t)op.src, d = (uintptr_t)op.dst;
  if (((s ^ d) & 15) != 0) return cudaErrorInvalidValue;  // caller routes mutually misaligned pairs elsewhere
  op.head = (16 - (s & 15)) & 15;
  if (op.head > bytes) op.head = bytes;
  op.body = (bytes - op.head) & ~(size_t)15;
  op.tail = bytes - op.head - op.body;
  const size_t tile = op.vec ? (size_t)kCopyThreads * 16 * 4 : (size_t)kTile;  // vec: one unrolled pass per CTA
  const size_t ntiles = (op.body + tile - 1) / tile;
  int grid = (int)min((size_t)ctas, ntiles > 0 ? ntiles : (size_t)1);
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid;
  iccl_direct_copy<<<grid, kCopyThreads, op.vec ? 0 : kStages * kTile, st>>>(op);
  return cudaGetLastError();
}

cudaError_t launch_backup(const BackupOp& op, int ctas, cudaStream_t st, int* grid_out) {
  if (grid_out) *grid_out = 0;
  if ((((uintptr_t)op.src ^ (uintptr_t)op.dst) & 15) != 0 || (op.chunk & 15) || op.nchunks == 0)
    return cudaErrorInvalidValue;
  if (cudaError_t e = configure_smem()) return e;
  const size_t ntiles = (min(op.chunk, op.bytes) + kTile - 1) / kTile;
  int grid = (int)min((size_t)max(ctas, 16), ntiles > 0 ? ntiles : (size_t)1);
  if (ctas > 0) grid = (int)min((size_t)ctas, ntiles > 0 ? ntiles : (size_t)1);
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid + 1;
  iccl_backup_ctl<<<1, 32, 0, st>>>(op);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || ctas == 0) return e;  // ctas 0: the controller alone (attribution runs)
  // attribution runs only (ctas < 0): -1 = the copy grid without its shared
  // memory (it must not copy), -2 = a one-CTA copy grid
  if (ctas == -1) {
    iccl_backup_attempt<<<grid, kCopyThreads, 0, st>>>(op);
    return cudaGetLastError();
  }
  iccl_backup_attempt<<<ctas == -2 ? 1 : grid, kCopyThreads, kStages * kTile, st>>>(op);
  return cudaGetLastError();
}

cudaError_t launch_copy(const void* src, void* dst, size_t bytes, int ctas, KernelStamp* stamp, cudaStream_t st,
                        int* grid_out, const uint32_t* resume, uint32_t chunk) {
  if (grid_out) *grid_out = 0;
  if (bytes == 0) return cudaSuccess;
  const uintptr_t s = (uintptr_t)src, d = (uintptr_t)dst;
  if (((s ^ d) & 15) != 0) {
    int grid = (int)min((size_t)ctas, (bytes + 512 * 16 - 1) / (512 * 16));
    if (grid < 1) grid = 1;
    if (grid_out) *grid_out = grid;
    iccl_copy_unaligned<<<grid, 512, 0, st>>>((const char*)src, (char*)dst, bytes, stamp, resume, chunk);
    return cudaGetLastError();
  }
  size_t head = (16 - (s & 15)) & 15;
  if (head > bytes) head = bytes;
  size_t body = (bytes - head) & ~(size_t)15;
  size_t tail = bytes - head - body;
  if (cudaError_t e = configure_smem()) return e;
  size_t ntiles = (body + kTile - 1) / kTile;
  int grid = (int)min((size_t)ctas, ntiles > 0 ? ntiles : (size_t)1);
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid;
  iccl_copy_tma<<<grid, kCopyThreads, kStages * kTile, st>>>((const char*)src, (char*)dst, head, body, tail, stamp,
                                                             resume, chunk);
  return cudaGetLastError();
}

// Load every kernel of this module now.  With CUDA lazy loading the first
// launch of a kernel loads its module, and a load issued while one of our
// streams is parked on a stream-memop wait blocked the launching thread on
// B200 (probes/p2p_probe4 test 1).  The proxy must never block, so
// iccl_comm_init_rank calls this before any wait is enqueued.
cudaError_t preload_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)iccl_copy_tma, (const void*)iccl_direct_copy,   (const void*)iccl_copy_unaligned,
                       (const void*)iccl_read_globaltimer, (const void*)iccl_gather_rows,
                       (const void*)iccl_scatter_rows, (const void*)iccl_expand_rows,
                       (const void*)iccl_ll_group, (const void*)iccl_wait_flags, (const void*)iccl_dispatch_push,
                       (const void*)iccl_backup_attempt, (const void*)iccl_backup_ctl,
                       (const void*)iccl_combine_pull, (const void*)iccl_expand_tma,
                       (const void*)iccl_dispatch_tma, (const void*)iccl_combine_tma};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  if (cudaError_t e = configure_smem()) return e;
  return cudaSuccess;
}

cudaError_t launch_read_globaltimer(unsigned long long* out, cudaStream_t st) {
  iccl_read_globaltimer<<<1, 1, 0, st>>>(out);
  return cudaGetLastError();
}


static int rows_grid(int64_t n_rows, int ctas) {
  int64_t warps_needed = n_rows;
  int64_t blocks = (warps_needed + 7) / 8;
  if (blocks > ctas) blocks = ctas;
  return (int)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_gather_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                               int ctas, cudaStream_t st) {
  if (n_rows == 0) return cudaSuccess;
  if ((row_bytes & 15) || ((uintptr_t)src & 15) || ((uintptr_t)dst & 15)) return cudaErrorInvalidValue;
  iccl_gather_rows<<<rows_grid(n_rows, ctas), 256, 0, st>>>((const int4*)src, (int4*)dst, idx, n_rows,
                                                            row_bytes / 16);
  return cudaGetLastError();
}

cudaError_t launch_dispatch(const DispatchOp& op, int ctas, cudaStream_t st, int* grid_out) {
  if (grid_out) *grid_out = 0;
  // launched even with no rows: its last CTA writes the done flags
  if (op.k < 1 || op.k > 32 || op.n > kMaxFusedRanks || (op.row16 <= 0) || ((uintptr_t)op.tokens & 15)) return cudaErrorInvalidValue;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  static const bool tma = getenv("ICCL_K8_TMA") ? atoi(getenv("ICCL_K8_TMA")) != 0 : false;  // measured no faster (profiles/r02 §5)
  if (tma) {
    const int64_t row_bytes = op.row16 * 16;
    const int64_t ntile = (row_bytes + 32768 - 1) / 32768;
    const int64_t tile = ((row_bytes + ntile - 1) / ntile + 15) / 16 * 16;
    const int smem = (int)(kExpStages * tile);
    static bool configured = false;
    if (!configured) {
      cudaError_t e = cudaFuncSetAttribute(iccl_dispatch_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    const int per_sm = (int)max((int64_t)1, min((int64_t)8, (int64_t)(200 * 1024) / (smem + 2048)));
    int64_t grid = ctas > 0 ? ctas : (int64_t)per_sm * sms;
    if (grid > op.n_tokens * ntile) grid = op.n_tokens * ntile;
    if (grid < 1) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    iccl_dispatch_tma<<<(int)grid, 32, smem, st>>>(op, tile, ntile);
    return cudaGetLastError();
  }
  const int64_t warps = op.n_tokens * op.parts;
  int64_t grid = (warps + 7) / 8;
  const int64_t cap = ctas > 0 ? ctas : 5 * (int64_t)sms;  // one wave: 5 x 256-thread CTAs per SM (48 registers)
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = (int)grid;
  iccl_dispatch_push<<<(int)grid, 256, 0, st>>>(op);
  return cudaGetLastError();
}

cudaError_t launch_combine(const CombineOp& op, int ctas, cudaStream_t st, int* grid_out) {
  if (grid_out) *grid_out = 0;
  // launched even with no rows: its last CTA writes the done flags
  if (op.n > kMaxFusedRanks || op.row16 <= 0 || ((uintptr_t)op.out & 15)) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const bool tma = getenv("ICCL_K10_TMA") ? atoi(getenv("ICCL_K10_TMA")) != 0 : true;
  if (tma) {
    const int64_t row_bytes = op.row16 * 16;
    const int64_t ntile = (row_bytes + 32768 - 1) / 32768;
    const int64_t tile = ((row_bytes + ntile - 1) / ntile + 15) / 16 * 16;
    const int smem = (int)(kExpStages * tile);
    static bool configured = false;
    if (!configured) {
      cudaError_t e = cudaFuncSetAttribute(iccl_combine_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    const int per_sm = (int)max((int64_t)1, min((int64_t)8, (int64_t)(200 * 1024) / (smem + 2048)));
    int64_t grid = ctas > 0 ? ctas : (int64_t)per_sm * sms;
    if (grid > op.n_rows * ntile) grid = op.n_rows * ntile;
    if (grid < 1) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    iccl_combine_tma<<<(int)grid, 32, smem, st>>>(op, tile, ntile);
    return cudaGetLastError();
  }
  int64_t grid = (op.n_rows * op.parts + 7) / 8;
  const int64_t cap = ctas > 0 ? ctas : 5 * (int64_t)sms;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = (int)grid;
  iccl_combine_pull<<<(int)grid, 256, 0, st>>>(op);
  return cudaGetLastError();
}

cudaError_t launch_expand_rows(const void* src, void* dst, const int64_t* pos, int64_t n_src, int k,
                               int64_t row_bytes, int ctas, cudaStream_t st) {
  if (n_src == 0 || k == 0) return cudaSuccess;
  if ((row_bytes & 15) || ((uintptr_t)src & 15) || ((uintptr_t)dst & 15)) return cudaErrorInvalidValue;
  static const bool tma = getenv("ICCL_K2_TMA") ? atoi(getenv("ICCL_K2_TMA")) != 0 : false;  // measured slower (profiles/r02 §5)
  if (tma && k <= 32) {
    // TMA form: tiles of <= 32 KB, kExpStages stages per one-warp CTA
    const int64_t ntile = (row_bytes + 32768 - 1) / 32768;
    const int64_t tile = ((row_bytes + ntile - 1) / ntile + 15) / 16 * 16;
    const int smem = (int)(kExpStages * tile);
    static int configured = 0;
    if (configured < smem) {
      cudaError_t e = cudaFuncSetAttribute(iccl_expand_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
      if (e != cudaSuccess) return e;
      configured = 4 * 32768;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = (int)max((int64_t)1, min((int64_t)8, (int64_t)(220 * 1024) / (smem + 1024)));
    int64_t grid = ctas > 0 ? ctas : (int64_t)per_sm * sms;
    if (grid > n_src * ntile) grid = n_src * ntile;
    iccl_expand_tma<<<(int)grid, 32, smem, st>>>((const char*)src, (char*)dst, pos, n_src, k, row_bytes, tile,
                                                 ntile);
    return cudaGetLastError();
  }
  const int64_t row16 = row_bytes / 16;
  const int parts = (int)max((int64_t)1, min((int64_t)8, row16 / 128));  // >= 4 int4 per lane per part
  if (ctas <= 0) {  // 8 x 256-thread CTAs per SM (62 registers: 4 resident, two waves) measured best
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ctas = 8 * sms;
  }
  iccl_expand_rows<<<rows_grid(n_src * parts, ctas), 256, 0, st>>>((const int4*)src, (int4*)dst, pos, n_src, k,
                                                                   row16, parts);
  return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                                int ctas, cudaStream_t st) {
  if (n_rows == 0) return cudaSuccess;
  if ((row_bytes & 15) || ((uintptr_t)src & 15) || ((uintptr_t)dst & 15)) return cudaErrorInvalidValue;
  iccl_scatter_rows<<<rows_grid(n_rows, ctas), 256, 0, st>>>((const int4*)src, (int4*)dst, idx, n_rows,
                                                             row_bytes / 16);
  return cudaGetLastError();
}

}  // namespace iccl
