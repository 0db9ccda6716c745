// Internal declarations shared by the runtime, the host arithmetic and the
// kernels of libiccl_b200.so.  Not part of the ABI (see include/iccl_b200.h).
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda.h>
#include <cuda_runtime_api.h>

#include "iccl_b200.h"

namespace iccl {

// Thread-local detailed message for iccl_get_last_error.
void set_last_error(const std::string& msg);
const char* last_error();

#define ICCL_CHECK_CUDA(expr)                                                              \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      ::iccl::set_last_error(std::string(#expr) + ": " + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                   \
      return ICCL_ERR_CUDA;                                                                \
    }                                                                                      \
  } while (0)

#define ICCL_CHECK_CU(expr)                                                                 \
  do {                                                                                      \
    CUresult r_ = (expr);                                                                   \
    if (r_ != CUDA_SUCCESS) {                                                               \
      const char* s_ = "?";                                                                 \
      if (::iccl::driver()) ::iccl::driver()->cuGetErrorString(r_, &s_);                    \
      ::iccl::set_last_error(std::string(#expr) + ": " + s_ + " at " + __FILE__ + ":" +     \
                             std::to_string(__LINE__));                                     \
      return ICCL_ERR_CUDA;                                                                 \
    }                                                                                       \
  } while (0)

#define ICCL_RETURN_IF(cond, code, msg)   \
  do {                                    \
    if (cond) {                           \
      ::iccl::set_last_error(msg);        \
      return code;                        \
    }                                     \
  } while (0)

uint64_t now_ns();  // CLOCK_MONOTONIC

// Monitor slot the SM copy kernel stamps with %globaltimer (K4).  Lives in
// host-mapped pinned memory; the proxy turns it into an iccl_mon_rec_t.
struct alignas(64) KernelStamp {
  unsigned long long t1;        // first CTA start
  unsigned long long t2;        // last CTA end
  unsigned int ctas_done;       // arrival counter for the last-CTA election
  unsigned int pad;
};

// Kernel launchers (iccl_kernels.cu).  All return cudaError_t of the launch.
// K1: copy `bytes` from src to dst (dst may be an IPC-mapped peer pointer)
// with at most `ctas` CTAs; TMA bulk body + vector head/tail.  `stamp` may be
// null.
// `resume` (host-mapped, may be null) makes the launch conditional: it copies
// only if chunk >= *resume when the kernel starts (the pre-enqueued backup
// attempt of an armed transfer skips the chunks the primary delivered).
cudaError_t launch_copy(const void* src, void* dst, size_t bytes, int ctas, KernelStamp* stamp, cudaStream_t st,
                        int* grid_out = nullptr, const uint32_t* resume = nullptr, uint32_t chunk = 0);
// Host-mapped words of one armed transfer (iccl_runtime.cpp armed_launch).
// Device writes come from stream memops and the backup kernel (K9); the
// watchdog thread only loads and stores them.
enum ArmedCtl : uint32_t { kCtlNone = 0, kCtlProbe = 1, kCtlSwitch = 2, kCtlAbort = 3 };
enum ArmedDec : uint32_t { kDecNone = 0, kDecExit = 1, kDecCopy = 2 };
struct alignas(64) ArmedWords {
  uint32_t prog;        // primary chunks landed (a memop after each primary chunk)
  uint32_t go;          // K9 may start: the primary finished, or the watchdog needs it (probe / switch)
  uint32_t resume;      // once switched, K9 copies chunks [resume, nchunks)
  uint32_t ctl;         // watchdog -> K9 (ArmedCtl)
  uint32_t probe_done;  // K9's CTS probe crossed the primary path
  uint32_t ns;          // no switch (1): the primary writes the done flags itself
  uint32_t p_fin;       // the primary attempt's copies (stale ones included) all landed
  uint32_t b_fin;       // the backup attempt drained
  uint32_t fin;         // the primary passed its done writes (the slot may be reused)
  uint32_t dec;         // K9's decision (ArmedDec), which its CTAs follow
  uint32_t pgate;       // 1 + the gate word the primary waits on (its path is Down), or 0: the probe is lost while it is closed
  uint32_t bgate;       // 1 + the gate word of a Down backup path, or 0
  uint32_t pad[4];
};
// K9: the backup attempt of an armed transfer, one launch per transfer,
// started once `go` opens.  CTA 0 decides: the primary finished with no
// switch -> every CTA exits; the watchdog asked for a probe -> a 16-byte CTS
// store over the primary path (unless that path's fault gate is closed) and
// probe_done; switched -> K1 over chunks [resume, nchunks) with a K4 stamp per
// chunk (ring[(stamp_base + k) % ring_slots]).
struct BackupOp {
  const char* src;
  char* dst;
  size_t bytes, chunk;
  uint32_t nchunks, ring_slots, stamp_base, pad;
  KernelStamp* ring;
  ArmedWords* w;
  const uint32_t* gates;   // the gate words (w->pgate / w->bgate index them)
  const char* probe_src;   // 16 bytes moved by the probe (over the primary path's direction)
  char* probe_dst;
  unsigned int* error;     // host-mapped: set if the decision wait exceeds 60 s
  unsigned int* dec_dev;   // K9a -> K9b decision word in GPU memory: (seq << 2) | decision
  uint32_t seq;            // this transfer's generation of dec_dev (30 bits)
};
cudaError_t launch_backup(const BackupOp& op, int ctas, cudaStream_t st, int* grid_out = nullptr);
// K6: direct zero-copy of a mid-size message by the side that arrived second
// at the rendezvous, on its own user stream (see rzv_post).
struct DirectOp {
  const char* src;
  char* dst;
  size_t head, body, tail;          // filled by launch_direct
  const uint32_t* peer_ready;       // the other side's ready flag (host-mapped control block)
  uint32_t peer_ready_gen;
  uint32_t* peer_done;              // the other side's done flag
  uint32_t peer_done_gen;
  uint32_t* my_done;                // this side's done flag (request bookkeeping)
  uint32_t my_done_gen;
  uint32_t* peer_done_dev;          // the other side's done word in its GPU memory (device flags), or null
  int vec;                          // 1: register copy (16 B vectors, no smem stage) instead of the TMA ring
  unsigned int* counter;            // CTA arrival counter (0 between uses)
  unsigned int* go;                 // CTA 0 -> other CTAs: the peer is ready (device memory, gen-tagged)
  unsigned int* error;              // host-mapped: set to 1 if the wait timed out
  KernelStamp* stamp;               // monitor on: %globaltimer t1 (peer ready seen) / t2 (last CTA done), or null
};
cudaError_t launch_direct(DirectOp op, size_t bytes, int ctas, cudaStream_t st, int* grid_out = nullptr);
// K7: the other side of a direct (K6-class) op waits for its done flags in a
// one-warp kernel (ld.acquire.sys polling) instead of a stream memop wait.
constexpr int kWaitMax = 32;
struct WaitList {
  const uint32_t* addr[kWaitMax];
  const uint32_t* alt[kWaitMax];  // device flags: addr is a word in this GPU's memory and alt the
                                  // host-mapped flag, read every 64th poll (paths that only write it)
  uint32_t gen[kWaitMax];
  int n;
  unsigned int* error;  // host-mapped: set to 1 if a wait timed out (10 s)
};
cudaError_t launch_wait(const WaitList& wl, cudaStream_t st);
// Force-load every kernel (see iccl_kernels.cu: lazy loading vs parked streams).
cudaError_t preload_kernels();
// K5: low-latency (LL) eager path for small and mid-size messages.  8-byte
// lines {4 B payload, 4 B sequence flag} written straight into a per-pair
// slot ring in the receiver's GPU memory; one fused kernel per stream
// progresses every LL op of a group concurrently, each op on 1..kLLMaxBlk
// CTAs scaled by its size (kLLLinesPerBlk lines per CTA), so group members
// never wait on each other through stream order.  The last CTA of an op
// (per-op arrival counter, reset by that CTA) writes its done flag and, on
// the receive side, returns the slot's credit.
constexpr int kLLSlots = 4;                 // slots per ordered pair (flow-control window)
constexpr size_t kLLMaxBytes = 1024 * 1024;  // largest LL message (the slot ring holds it; sm_small_bytes routes)
constexpr size_t kLLLines = kLLMaxBytes / 4;
constexpr int kLLMaxOps = 64;               // LL ops per launch
constexpr int kLLMaxBlk = 64;               // CTAs per op (16 -> 64: 256 KiB 18.3 -> 27.3 GB/s, profiles/r02)
constexpr size_t kLLLinesPerBlk = 1024;     // 4 lines per thread at 256 threads
constexpr int kLLMaxBlocksPerLaunch = 1024;
constexpr int kLLCounters = 4096;           // per-op arrival counters (ring)
struct LLDesc {
  int kind;               // 0 send, 1 recv
  uint32_t seq;           // 1-based message number on this ordered pair
  uint64_t bytes;
  char* buf;              // send: source; recv: destination
  void* slot;             // uint2[kLLLines]: peer's slot (send) / my slot (recv)
  unsigned int* credit;   // kLLSlots per-slot credit words (slot s: seq of the last message
                          // read from it); send: mine for the peer (local), recv: the
                          // sender's words for me (peer-mapped)
  unsigned int* done_flag;  // op's done slot in the control block (host-mapped)
  uint32_t done_gen;
  uint32_t first_blk;     // first CTA of this op in the launch
  uint32_t nblk;          // CTAs of this op
  unsigned int* counter;  // arrival counter of this op (local HBM, 0 between uses)
  KernelStamp* stamp;     // send, monitor on: %globaltimer t1 (first CTA starts) / t2 (last CTA done), or null
};
struct LLBatch {
  int n;
  unsigned int* error;    // host-mapped: set to 1 if a wait timed out
  LLDesc d[kLLMaxOps];
};
cudaError_t launch_ll(const LLBatch& b, cudaStream_t st);

// Calibration: write %globaltimer into *out (host-mapped).
cudaError_t launch_read_globaltimer(unsigned long long* out, cudaStream_t st);
// K2 / K3: row gather / scatter of `row_bytes`-byte rows (MoE dispatch pack /
// combine unpack).  dst_rows[i] <- src_rows[idx[i]]  (gather),
// dst_rows[idx[i]] <- src_rows[i] (scatter).  Rows are 16-byte multiples.
cudaError_t launch_gather_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                               int ctas, cudaStream_t st);
// K2 expand form: dst_rows[pos[t*k + j]] <- src_rows[t] for j < k (each source row read once).
cudaError_t launch_expand_rows(const void* src, void* dst, const int64_t* pos, int64_t n_src, int k,
                               int64_t row_bytes, int ctas, cudaStream_t st);
// K8: fused MoE dispatch (K2 expand form + the alltoallv push, no staging).
// Packed row p (the send layout: rows grouped by destination rank) goes to
// the rank d with lo[d] <= p < hi[d], as row p - lo[d] of seg (that rank's
// receive segment for this source: IPC-mapped, or local for the self one).
constexpr int kMaxFusedRanks = 64;
struct FusedDest {
  char* seg;
  int64_t lo, hi;
  const uint32_t* ready;  // the destination's recv-op ready flag (host-mapped), null for the self segment
  uint32_t ready_gen;
  uint32_t done_gen;
  uint32_t* done;         // the destination's recv-op done flag, or null
  uint32_t* my_done;      // this rank's send-op done flag, or null
  uint32_t my_done_gen;
  uint32_t pad;
};
struct DispatchOp {
  const int4* tokens;
  const int64_t* pos;  // [n_tokens * k]: packed row of (token, j)
  int64_t n_tokens;
  int32_t k, n;        // top-k (<= 32), ranks
  int64_t row16;
  int32_t parts;       // column parts per token row (one warp each)
  uint32_t go_gen;
  unsigned int* ticket;   // entry ticket (0 between uses): the first CTA polls the ready flags
  unsigned int* counter;  // exit counter (0 between uses)
  unsigned int* go;       // poller -> other CTAs (gen-tagged)
  unsigned int* error;    // host-mapped: set to 1 if a wait timed out
  KernelStamp* stamp;
  FusedDest d[kMaxFusedRanks];
};
cudaError_t launch_dispatch(const DispatchOp& op, int ctas, cudaStream_t st, int* grid_out = nullptr);
// K10: fused MoE combine (the reverse alltoallv + K3 in one kernel, no
// staging): packed row r (rows grouped by the expert rank d that holds them,
// lo[d] <= r < hi[d]) is loaded from row r - lo[d] of seg[d] — this rank's
// segment in rank d's expert-output tensor, IPC-mapped (NVLink loads) or
// local — and stored at out row order[r].
struct FusedSrc {
  const char* seg;
  int64_t lo, hi;
  const uint32_t* ready;  // the source's send-op ready flag (host-mapped), null for the self segment
  uint32_t ready_gen;
  uint32_t done_gen;
  uint32_t* done;         // the source's send-op done flag, or null
  uint32_t* my_done;      // this rank's recv-op done flag, or null
  uint32_t my_done_gen;
  uint32_t pad;
};
struct CombineOp {
  int4* out;
  const int64_t* order;  // [n_rows]: out row of packed row r
  int64_t n_rows;
  int64_t stride;        // visiting order of the rows: r = (i * stride) mod n_rows, gcd(stride, n_rows) = 1
  int32_t n, parts;
  int64_t row16;
  uint32_t go_gen, pad;
  unsigned int* ticket;
  unsigned int* counter;
  unsigned int* go;
  unsigned int* error;
  KernelStamp* stamp;
  FusedSrc d[kMaxFusedRanks];
};
cudaError_t launch_combine(const CombineOp& op, int ctas, cudaStream_t st, int* grid_out = nullptr);
cudaError_t launch_scatter_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                                int ctas, cudaStream_t st);
}  // namespace iccl

namespace iccl {
// CUDA driver entry points, resolved at first use through cudart
// (cudaGetDriverEntryPoint) so libiccl_b200.so loads on hosts without a GPU
// driver (the CPU test suite checks its exports there).
struct Driver {
  CUresult (*cuGetErrorString)(CUresult, const char**);
  CUresult (*cuInit)(unsigned int);
  CUresult (*cuDeviceGet)(CUdevice*, int);
  CUresult (*cuDeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  CUresult (*cuStreamWriteValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  CUresult (*cuStreamWaitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  CUresult (*cuStreamBatchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);
  CUresult (*cuMemcpyDtoDAsync)(CUdeviceptr, CUdeviceptr, size_t, CUstream);
  CUresult (*cuMemGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  CUresult (*cuPointerGetAttribute)(void*, CUpointer_attribute, CUdeviceptr);
  bool ok;
};
// Returns null (and sets the last error) if the driver is unavailable.
const Driver* driver();
}  // namespace iccl
