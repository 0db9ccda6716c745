// ICCL B200 runtime: communicator bootstrap, the stream-ordered P2P API and
// the per-rank proxy thread that drives the copy engines.
//
// Mapping of the reference design (§3.2-3.4, SPEC.md verbs /
// transport / monitor) onto one 8xB200 NVSwitch box:
//
//   paper / SPEC                          here
//   ------------------------------------  --------------------------------------------
//   CPU proxy thread   one std::thread per communicator (proxy_loop)
//   hostFunc #1 / #2   driver()->cuStreamWriteValue32(ready) / WaitValue(done)
//                                         on the caller's stream: 0 SMs, no callbacks
//   User Buffer Registration (:410-412)   IPC export of the caller's allocation, cached
//                                         by CU_POINTER_ATTRIBUTE_BUFFER_ID
//   CTS / RTS               each side's posting (buffer IPC handle, op slot)
//                                         in the pair's rendezvous ring (shm); the side
//                                         that arrives second issues the copies from its
//                                         own API call: push by the sender, pull by the
//                                         receiver
//   WR post / WC        chunk copy enqueue / device-written progress
//                                         word observed by the proxy
//   primary QP / backup QP (:461)         copy-engine path / SM-kernel path (K1)
//   six pointers        Xfer::next_issue (posted=transmitted),
//                                         Xfer::completed (acked = receiver done)
//   switch_qp           switch_path(): resume at receiver done
//   RNIC port down         injected gate: cuStreamWaitValue32 on a host
//                                         word placed before chunks on the primary path
//
// Data moves zero-copy: a copy engine (or K1) moves the bytes straight from
// the sender's tensor into the receiver's tensor through an IPC mapping — no
// FIFO, no staging copy.
//
// Why the API thread issues the copies (and the proxy only observes, monitors
// and re-issues on failover): while any thread of the process sits in a
// synchronous CUDA call (e.g. a pageable cudaMemcpy) on a stream parked behind
// one of our ops, every other CUDA call of the process blocks — memcpy,
// kernel launch, stream memop, event record alike (probes/p2p_probe6).  A
// proxy that still had to enqueue the copy would deadlock with such a user;
// all device work an op needs is therefore enqueued before the API returns.
#include <errno.h>
#include <fcntl.h>
#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <sys/syscall.h>
#include <unistd.h>

#include "iccl_internal.h"

namespace iccl {

// ICCL_DEBUG=1: the proxy traces every device call it makes (stderr), so a
// stuck proxy shows the call it is blocked in.
static const bool g_debug = getenv("ICCL_DEBUG") && atoi(getenv("ICCL_DEBUG")) > 0;
#define ICCL_TRACE(...)                                                          \
  do {                                                                           \
    if (::iccl::g_debug) {                                                       \
      char b_[512];                                                              \
      snprintf(b_, sizeof(b_), __VA_ARGS__);                                     \
      fprintf(stderr, "[iccl %.6f %d] %s\n", (double)::iccl::now_ns() * 1e-9,     \
              (int)syscall(SYS_gettid), b_);                                     \
    }                                                                            \
  } while (0)

// Under ICCL_DEBUG every device call is also timed: one that blocks for more
// than 50 us (a full command queue, a lock another thread holds in the
// driver) is traced with the call and the calling thread.
#define ICCL_TIMED_(expr, R_)                                                                     \
  [&]() {                                                                                         \
    const uint64_t t0_ = ::iccl::g_debug ? ::iccl::now_ns() : 0;                                  \
    R_ v_ = (expr);                                                                               \
    if (::iccl::g_debug) {                                                                        \
      const uint64_t d_ = ::iccl::now_ns() - t0_;                                                 \
      if (d_ > 50000) ICCL_TRACE("slow device call %.1f us at line %d: %s", d_ * 1e-3, __LINE__, #expr); \
    }                                                                                             \
    return v_;                                                                                    \
  }()
#undef ICCL_CHECK_CUDA
#define ICCL_CHECK_CUDA(expr)                                                              \
  do {                                                                                     \
    cudaError_t e_ = ICCL_TIMED_(expr, cudaError_t);                                       \
    if (e_ != cudaSuccess) {                                                               \
      ::iccl::set_last_error(std::string(#expr) + ": " + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                   \
      return ICCL_ERR_CUDA;                                                                \
    }                                                                                      \
  } while (0)
#undef ICCL_CHECK_CU
#define ICCL_CHECK_CU(expr)                                                              \
  do {                                                                                   \
    CUresult r_ = ICCL_TIMED_(expr, CUresult);                                           \
    if (r_ != CUDA_SUCCESS) {                                                            \
      const char* s_ = "?";                                                              \
      if (::iccl::driver()) ::iccl::driver()->cuGetErrorString(r_, &s_);                 \
      ::iccl::set_last_error(std::string(#expr) + ": " + s_ + " at " + __FILE__ + ":" +  \
                             std::to_string(__LINE__));                                  \
      return ICCL_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)

constexpr uint64_t kMagic = 0x3030324242434349ull;  // "ICCLB200"
constexpr int kSlots = 4096;                        // op slots per rank (ready/done flags)
constexpr int kRzvDepth = 1024;                     // rendezvous entries per ordered pair
constexpr int kMaxRanks = 64;
// Gate words (fault gates, probe gates): a closed gate is never recycled; a
// released one only after the whole ring went round (16K allocations — at a
// probe per 200 us, > 3 s — so every device wait on it has long executed).
constexpr int kGateWords = 16384;
constexpr int kStampSlots = 4096;
constexpr int kArmedSlots = 1024;  // armed transfers in flight per rank
constexpr size_t kScratchBytes = 4096;
constexpr int kProxyNapUs = 20;  // proxy back-off when a pass moved nothing
// How long a send waits for its receiver's half before posting its own (so
// that it arrives second and pushes, see rzv_post): single ops / a group.
// ICCL_SEND_WAIT_US / ICCL_GROUP_SEND_WAIT_US override them.
static uint64_t env_us(const char* name, uint64_t dflt) {
  const char* v = getenv(name);
  return v && *v ? strtoull(v, nullptr, 10) : dflt;
}
static const uint64_t kSendWaitUs = env_us("ICCL_SEND_WAIT_US", 20);
static const uint64_t kGroupSendWaitUs = env_us("ICCL_GROUP_SEND_WAIT_US", 1000);

// ---------------------------------------------------------------- shared control block
struct alignas(64) ShmHeader {
  uint64_t magic;
  int32_t nranks;
  std::atomic<int32_t> attached;
  std::atomic<int32_t> bar_count;
  std::atomic<int32_t> bar_sense;
  std::atomic<int32_t> abort;
};

struct alignas(64) RankInfo {
  int32_t pid;
  int32_t dev;
  char bus_id[32];
  cudaIpcMemHandle_t scratch_handle;
  cudaIpcMemHandle_t ll_handle;
  cudaIpcMemHandle_t relay_handle;  // staging slots of this rank as a relay (valid if relay_slot_bytes)
  uint64_t relay_slot_bytes;
  std::atomic<uint64_t> op_count;  // opCount
};

// Six-pointer view of one op, published by the sender's
// proxy into both endpoints' slots so either side's iccl_req_state sees it.
struct XferPub {
  uint32_t gen;       // op generation this record belongs to
  int32_t kind;       // 0 send, 1 recv (written by the owner's API thread)
  int32_t total;      // chunks
  int32_t posted;     // sender posted == transmitted (handed to an engine)
  int32_t done;       // contiguous delivered prefix: receiver done == sender acked
  int32_t path;
  int32_t switches;
  int32_t pad;
  uint64_t bytes;
};

struct alignas(64) RankFlags {
  uint32_t ready[kSlots];  // written by the owner's user stream
  uint32_t done[kSlots];   // written by the copy stream that completes the op
  XferPub pub[kSlots];
};

// One side's posting of the k-th op of an ordered pair (RTS from the sender,
// CTS from the receiver).
struct RzvSide {
  uint64_t bytes;
  uint64_t buffer_id;    // CU_POINTER_ATTRIBUTE_BUFFER_ID of the allocation (0: self pair, use direct_ptr)
  uint64_t base_offset;  // offset of the tensor inside that allocation
  uint64_t direct_ptr;   // the tensor's pointer in its owner's address space
  uint32_t slot, gen;    // the owner's op slot: ready / done flags and six-pointer record
  uint64_t stream;       // the owner's user stream (a self pair compares it: same stream => ordered)
  cudaIpcMemHandle_t handle;
};

// Rendezvous of the k-th send and the k-th recv of an ordered pair: each side
// writes its half, then bumps `arrivals` (the side that sees 2g+1, g = k /
// depth, arrived second); the transfer is issued by whoever wins `claimed`.
struct alignas(64) RzvEntry {
  std::atomic<uint64_t> arrivals;
  std::atomic<uint64_t> claimed;  // generations whose transfer has an issuer (CAS g -> g + 1)
  RzvSide side[2];  // 0 sender, 1 receiver
};

// Per ordered pair src->dst: the active path (shared by whichever side
// issues), how many fault-script entries name the pair, and the routing of
// its small (LL-size) ops.
//
// Small ops have no rendezvous: the k-th LL send of a pair meets the k-th LL
// recv because both sides classify by size.  A pair that is armed for
// failover (a fault script names it) or runs on its backup path must take
// the rendezvous / chunked path instead, where gates, the watchdog,
// switch_qp and the monitor apply — and both sides
// must agree op by op.  So the route is a history of segments over the
// pair's small-op index: a change appended under `route_lock` starts at
// max(ops the sender classified, ops the receiver classified), i.e. after
// every op either side has already routed, and each side routes its q-th
// small op by the segment containing q.
constexpr int kRouteSegs = 512;  // route changes remembered per pair (a side may lag the other by all of them)
struct alignas(64) PairState {
  std::atomic<int32_t> active_path, switches;
  std::atomic<int32_t> faults_armed;  // fault-script entries naming the pair (both endpoints' scripts)
  std::atomic<uint32_t> route_lock;
  uint64_t small_ops[2];              // small ops routed so far: [0] sender side, [1] receiver side
  int32_t route_rdv;                  // current route of new small ops: 1 = rendezvous, 0 = LL
  int32_t route_base;                 // route of ops older than every retained segment
  uint32_t nseg;                      // segments appended so far (ring of kRouteSegs)
  uint32_t pad;
  uint64_t seg_start[kRouteSegs];
  int32_t seg_rdv[kRouteSegs];
};

// Buffers src exported to dst (a new CU_POINTER_ATTRIBUTE_BUFFER_ID in one of
// its halves): dst's proxy opens them ahead of need (premap_peer_buffers).
constexpr int kAnnDepth = 64;
struct AnnEntry {
  uint64_t buffer_id;
  uint64_t retire;  // 1: the owner deregistered the buffer — close its mapping
  cudaIpcMemHandle_t handle;
};
struct alignas(64) Announce {
  std::atomic<uint64_t> head, tail;  // head: src's API thread, tail: dst's proxy
  AnnEntry e[kAnnDepth];
};

struct alignas(64) RzvRing {
  PairState st;
  Announce ann;
  RzvEntry e[kRzvDepth];
};

// GPU-relay backup path (SURVEY.md §2.3 N9, §8e "Relay backup"): source s
// pushes a piece into its staging slot on relay GPU r (hop 1, s's copy
// engine), r's proxy forwards it into the destination's buffer (hop 2, r's
// copy engine).  Per relay r and source s: two staging slots, a request ring
// written by s's proxy, and two device-written piece counters.
constexpr int kRelayDepth = 64;  // requests in flight per (relay, source)
constexpr int kRelaySlots = 2;   // staging slots per (relay, source)

struct alignas(64) RelayReq {
  std::atomic<uint64_t> seq;  // 1-based piece number from this source; published last
  int32_t dst;
  uint32_t slot;
  uint64_t bytes;
  uint64_t buffer_id;    // destination allocation (owned by rank dst)
  uint64_t base_offset;  // piece offset inside that allocation
  cudaIpcMemHandle_t handle;
};

struct alignas(64) RelayCounter {
  uint32_t v;  // cyclic piece counter, written by a copy stream (WriteValue), waited on with GEQ
  uint32_t pad[15];
};

struct ShmLayout {
  size_t off_ranks, off_flags, off_rings, off_relay, relay_box, total;
  explicit ShmLayout(int n) {
    size_t o = 4096;
    off_ranks = o;
    o += sizeof(RankInfo) * n;
    o = (o + 4095) & ~(size_t)4095;
    off_flags = o;
    o += sizeof(RankFlags) * n;
    o = (o + 4095) & ~(size_t)4095;
    off_rings = o;
    o += sizeof(RzvRing) * n * n;
    o = (o + 4095) & ~(size_t)4095;
    // per relay rank: in[n], out[n] counters, then req[n][kRelayDepth]
    off_relay = o;
    relay_box = sizeof(RelayCounter) * 2 * n + sizeof(RelayReq) * n * kRelayDepth;
    relay_box = (relay_box + 4095) & ~(size_t)4095;
    o += relay_box * n;
    total = (o + 4095) & ~(size_t)4095;
  }
};

struct UidBlob {
  uint64_t magic;
  char shm_name[64];
};

static inline bool cyc_geq(uint32_t a, uint32_t b) { return (int32_t)(a - b) >= 0; }

// ---------------------------------------------------------------- proxy-side structures
// ENG_CE_GROUP: the rank's two group streams — one for the pushes, one for
// the pulls of a group (alltoallv, batch_isend_irecv) — see rzv_post.
enum Engine { ENG_CE = 0, ENG_SM = 1, ENG_RELAY = 2, ENG_CE_GROUP = 3 };

struct OpDesc {
  int kind;  // 0 send, 1 recv
  int peer;
  const char* src;
  size_t bytes;
  uint32_t slot, gen;
  uint64_t op_seq;
  bool ll = false;   // small message on the LL kernel path (K5)
  uint32_t ll_seq = 0;
  bool direct = false;   // mid-size message: the side arriving second runs K6 on its user stream
  bool issued_direct = false;  // ... and that side is this one: K6 replaces this op's stream markers
  bool issued_instream = false;  // this side issued the copy on its own user stream (no markers)
  bool markers_elided = false;   // self pair, both halves on one stream in one group: no markers at all
  bool fused = false;            // a send of a fused dispatch (K8 stores the rows; iccl_dispatch_rows)
  bool pull = false;             // a recv of a fused combine (K10 loads the rows; iccl_combine_rows)
  DirectOp dop{};        // K6 parameters when issued_direct
  int kstamp = -1;       // monitor on: K5 send / K6 stamp slot (K4), turned into a record by the proxy
};

struct ChunkRec {
  int stream = -1;  // index into Channel::stream table
  cudaEvent_t ev = nullptr;   // recorded after the chunk on its copy stream: the WC
  cudaEvent_t tev = nullptr;  // monitor on, copy-engine path: timing event on the channel's
                              // monitor stream right behind ev (the WC then; the chunk's t2)
  cudaEvent_t t1ev = nullptr;  // monitor: timing event marking the chunk's start (not owned)
  uint64_t t1 = 0;
  int path = 0;
  int stamp = -1;
  bool done = false;
  uint32_t relay_q = 0;  // relay path: the chunk's last piece number (its WC: relay out >= relay_q)
};

struct Xfer {
  uint64_t op_seq = 0;   // the issuer's op number (monitor records)
  uint64_t pair_seq = 0;  // k: the k-th op of the ordered pair src_rank -> dst_rank
  int src_rank = 0, dst_rank = 0;
  int chan = -1;  // issuing channel (2 * peer + dir)
  const char* src = nullptr;  // sender's tensor (local, or IPC-mapped when the receiver pulls)
  char* dst = nullptr;        // receiver's tensor (local, or IPC-mapped when the sender pushes)
  size_t bytes = 0;
  uint32_t s_slot = 0, s_gen = 0;  // sender's op slot
  uint32_t r_ready_slot = 0, r_ready_gen = 0, r_done_slot = 0, r_done_gen = 0;  // receiver's
  int nchunks = 0;
  size_t chunk = 0;
  // receiver's buffer as exported in its CTS (the relay forwards into it)
  uint64_t dst_buffer_id = 0, dst_base_offset = 0;
  cudaIpcMemHandle_t dst_handle{};
  int relay_r = -1;          // relay GPU carrying pieces of this op, if any
  uint32_t relay_last_q = 0;  // last piece pushed through it (completion waits for its hop 2)
  int next_issue = 0;  // sender posted == transmitted (chunks handed to an engine)
  int completed = 0;   // contiguous prefix observed delivered: acked == receiver done
  int path = 0;
  std::vector<int> waited[2];  // per path: streams that already waited on the ready flags
  bool group_stream = false;   // remote copy of a group: the rank's group stream of its direction
  int group_lane = 0;          // which of the direction's group streams (ICCL_GROUP_LANES)
  bool done_enqueued = false;
  bool eligible = false;
  uint64_t last_progress = 0;
  int switches = 0;
  int fault_ops_index = -1;
  std::vector<ChunkRec> rec;
  std::vector<cudaEvent_t> fences;  // events the completion must also wait for
  // monitor on the copy-engine path: per stream, the last timing event this
  // op recorded there (a chunk starts where the previous one on its stream
  // ended, or at the op's anchor recorded right after the ready waits)
  std::vector<std::pair<int, cudaEvent_t>> last_ev;
  std::vector<cudaEvent_t> anchors;  // owned timing events (returned at retire)
  // issued from this side's API call: the issuing user stream's position at
  // the op, recorded right there; the copy streams wait on it instead of
  // polling this side's host-mapped ready flag (same process, same GPU)
  cudaEvent_t own_ready = nullptr;
  int own_side = -1;  // 0: stands for the sender's ready flag, 1: the receiver's
  // In-stream issue (a healthy, unarmed pair): the issuing side enqueued every
  // chunk on its own user stream behind a wait on the other side's ready
  // flag, and the done writes behind the last chunk.  Such a transfer is not
  // migrated by switch_qp; it completes where it was posted.
  cudaStream_t ustream = nullptr;
  bool instream = false;
  bool gated = false;          // this attempt placed a chunk behind a closed fault gate
  bool done_deferred = false;  // ... so its last chunk carries no done writes: the attempt that
                               // completes the op releases both sides (device writes after the
                               // fences, or the proxy's host writes once every chunk landed)
  // Armed transfer (armed_launch): both attempts are on the device from the
  // start; the watchdog thread drives the failover with host stores only.
  bool armed = false;
  int aw = -1;                   // ArmedWords slot
  std::vector<int> bstamp;       // K4 stamp slot of each backup chunk (its WC)
  cudaEvent_t p_end = nullptr;   // the primary attempt's end (the backup's fence)
  bool switched = false;         // the backup attempt carries chunks [resume, N)
  bool probing = false, probe_ok = false;
  uint64_t probe_t = 0;
  uint64_t t_obs = 0;            // host time of the last primary-progress observation (monitor t1)
};

struct StreamCtx {
  cudaStream_t s = nullptr;
  uint32_t ticket = 0;
  volatile uint32_t* prog = nullptr;  // host-mapped, written by the stream after each chunk
  cudaEvent_t ev = nullptr;
  int engine = ENG_CE;
};

struct FaultState {
  bool down = false;
  int gate = -1;        // gate word index while down
  uint64_t down_at = 0;  // ns
};

// One direction of traffic with one peer, as seen by the issuing side:
// dir 0 = push (I send to peer), dir 1 = pull (peer sends to me).  The
// transfers I issue for that ordered pair live here.
struct Channel {
  int peer = -1;
  int dir = 0;
  int src = -1, dst = -1;  // ranks of the ordered pair
  std::deque<Xfer> xfers;    // issued by this rank, in issue order
  std::vector<int> path_streams[2];
  int probe_stream = -1;
  int mon_stream = -1;            // monitor timing events (kept off the copy streams)
  cudaEvent_t bridge = nullptr;   // untimed event copy stream -> monitor stream (op anchors)
  // on the backup because the primary failed (watchdog + probe): only then
  // does monitor_failed_link probe the primary to switch back;
  // an API switch_qp is sticky until the next API switch
  bool failed_over = false;
  FaultState fault[2];
  // probe state
  bool probe_out = false;
  uint32_t probe_ticket_expect = 0;
  uint64_t probe_sent = 0;
  int probe_path = 0;
  uint64_t last_probe = 0;
  uint64_t fault_seq_base = 0;  // pair op count at iccl_fault_set (chunk-triggered faults count from here)
  char* peer_scratch = nullptr;  // 16 B probe target on the peer
  int relay_rank = -1;  // relay GPU of the backup path: lowest rank not an endpoint (topology.py:140-151 tie-break)
  // armed transfers (owned by the watchdog thread)
  int b_si = -1;                   // the channel's backup-attempt stream, created on first use
  int p_si = -1;                   // the channel's progress-word stream (armed primaries), created on first use
  std::deque<Xfer> armed;
  bool armed_failed_over = false;  // the watchdog moved the pair to its backup path
  uint64_t armed_last_probe = 0;
};

struct Fault {
  iccl_fault_t f;
  bool fired = false;
};

}  // namespace iccl

using namespace iccl;

struct iccl_comm {
  int rank = 0, nranks = 0, dev = 0;
  iccl_config_t cfg{};
  // shm
  std::string shm_name;
  void* shm = nullptr;
  size_t shm_bytes = 0;
  ShmHeader* hdr = nullptr;
  RankInfo* ranks = nullptr;
  RankFlags* flags = nullptr;
  RzvRing* rings = nullptr;
  int bar_sense = 0;
  // private pinned host memory (progress words, gates, probe words, stamps)
  uint32_t* pinned = nullptr;
  size_t pinned_bytes = 0;
  volatile uint32_t* gate_words = nullptr;
  std::vector<uint8_t> gate_closed;  // 1 while a gate is allocated and not yet released (gate_mu)
  std::mutex gate_mu;                // leaf lock: gate allocation / release
  std::atomic<int> next_gate{0};
  KernelStamp* stamps = nullptr;
  std::atomic<int> next_stamp{0};
  unsigned long long* gtimer = nullptr;
  int64_t gtimer_offset = 0;  // host_ns - globaltimer_ns
  char* scratch = nullptr;    // device scratch (probe target), exported to peers
  // LL path (K5): slot rings for every source rank + credit words, in my HBM
  char* ll_region = nullptr;
  std::vector<char*> peer_ll;
  std::vector<uint32_t> ll_sent, ll_recvd;
  unsigned int* ll_error = nullptr;  // host-mapped
  unsigned int* ll_counters = nullptr;  // kLLCounters per-op arrival counters (device)
  uint32_t ll_ctr_next = 0;
  // GPU relay (backup_kind RELAY, >= 3 ranks)
  char* relay_buf = nullptr;         // my staging: [source][kRelaySlots] x relay_slot_bytes
  size_t relay_slot_bytes = 0;
  std::vector<char*> peer_relay;     // staging of relay rank r, mapped on first use
  std::vector<uint32_t> relay_sent;  // pieces I pushed through relay r
  std::vector<uint64_t> relay_next;  // next request I (as relay) expect from source s
  std::vector<int> relay_serve;      // my forwarding stream per source (index into streams)
  // API state
  uint64_t op_seq = 0;
  std::vector<uint64_t> pair_sends, pair_recvs;  // non-LL ops posted per peer (rendezvous index k)
  std::vector<std::unordered_map<uint64_t, char*>> peer_ipc;  // per peer: its buffer id -> mapped base
  std::vector<char*> peer_scratch_base;                       // IPC-opened peer scratch blocks
  int group_depth = 0;
  std::vector<std::pair<OpDesc, cudaStream_t>> group_ops;
  struct GroupJob {
    int kind, peer;
    uint64_t k, op_seq;
    RzvSide side[2];      // both halves, copied before the claim (the entry may be reused after it)
    cudaStream_t stream;  // this side's user stream
  };
  std::vector<GroupJob> group_jobs;  // copy-engine transfers this side issues for the open group
  // fused MoE dispatch (iccl_dispatch_rows) in the open group: its sends
  // rendezvous at group_end, then K8 runs on `stream` between the group's
  // ready markers and its done waits
  bool in_dispatch = false;   // ops posted now belong to a dispatch: no LL, K7 done waits
  bool dispatch_fused = false;
  cudaStream_t dispatch_stream = nullptr;
  DispatchOp dispatch_op{};
  // fused MoE combine (iccl_combine_rows): its recvs rendezvous at group_end
  // (each waits for the sender's half and pulls), then K10 runs on the stream
  bool in_combine = false;
  bool combine_fused = false;
  cudaStream_t combine_stream = nullptr;
  CombineOp combine_op{};
  char* dispatch_stage = nullptr;  // staging of the unfused fallback (an armed pair), grown on demand
  size_t dispatch_stage_bytes = 0;
  int direct_ctas = 32;       // K6 grid (>= 16 CTAs keep NVLink busy, kernels bench)
  int dispatch_ctas = 0;      // K8 grid cap (0: 4 CTAs per SM; ICCL_DISPATCH_CTAS)
  bool kernel_waits = true;   // K7 for the done waits of direct-class ops (ICCL_KERNEL_WAITS=0: memop waits)
  size_t k6_vec_bytes = 0;    // K6 copies ops up to this size with registers (ICCL_K6_VEC_KIB)
  bool device_flags = false;  // direct-class ready/done words also in GPU memory (ICCL_DEVICE_FLAGS=1; slower)
  bool event_ready = false;   // same-process ready wait as a CUDA event (ICCL_EVENT_READY=1; mixed result)
  int group_lanes = 1;        // group streams per direction (ICCL_GROUP_LANES)
  std::unordered_map<uint64_t, cudaIpcMemHandle_t> export_cache;
  std::vector<std::unordered_set<uint64_t>> announced;  // per peer: buffer ids announced to it
  // proxy
  std::vector<Channel> ch;  // 2 per peer: [2 * peer + dir]
  std::vector<StreamCtx> streams;
  // per-rank side streams shared by every channel (so N = 8 needs ~22 streams,
  // under CUDA_DEVICE_MAX_CONNECTIONS = 32): the backup SM-kernel stream, the
  // CTS probe stream, one monitor stream per direction (push / pull) and the
  // relay hop-1 stream
  int sm_si = -1, probe_si = -1, mon_si[2] = {-1, -1}, relay_si = -1;
  // a group's self copy (alltoallv's own segment, a local HBM copy) runs on
  // self_si, forked from and joined back into the user stream by events, so
  // it overlaps the group's NVLink copies instead of queueing in front of them
  int self_si = -1;
  cudaEvent_t self_fork = nullptr, self_join = nullptr;
  bool self_overlap = true;  // ICCL_SELF_OVERLAP=0: the self copy stays in the user stream's order
  // K7 (a one-warp polling kernel) instead of a stream-memory wait for the
  // copy-engine path's done waits (ICCL_K7_CE) / the issuer's wait on the
  // other side's ready flag (ICCL_K7_READY): a parked stream slows the GPU's
  // other streams
  bool k7_ce = false, k7_ready = false;
  int a2a_pieces = 1;  // ICCL_A2A_PIECES: pieces per remote alltoallv segment (see iccl_alltoallv)
  int a2a_order = 0;   // ICCL_A2A_ORDER: 0 rotated, 1 largest segment first
  size_t ll_lines_per_blk = kLLLinesPerBlk;  // K5 CTAs per op: lines per CTA (ICCL_LL_LINES_PER_BLK) ...
  int ll_max_blk = kLLMaxBlk;                // ... up to this many (ICCL_LL_MAX_BLK)
  bool instream_ce = true;  // healthy pairs: the issuer enqueues the copy on its own user stream (ICCL_INSTREAM=0: off)
  bool armed_backup = true;  // attribution only (ICCL_ARMED_BACKUP=0): armed transfers enqueue no backup attempt
  int k9_mode = 0;           // attribution only (ICCL_K9_MODE): 1 = K9a alone, 2 = b_fin memop alone,
                             // 3 = K9b launched without its shared memory, 4 = a one-CTA K9b
  bool prog_events = true;   // armed primaries' progress words from a side stream (ICCL_PROG_EVENTS=0: in-stream memops)
  // monitor records of ops the proxy does not track (K5 sends, K6): their
  // %globaltimer stamps (K4), turned into records once t2 lands
  struct KRec {
    int stamp;
    uint64_t bytes, op_seq;
    int peer, dir;
  };
  std::deque<KRec> krecs;  // mon_mu
  std::atomic<uint64_t> krecs_pending{0};  // krecs.size(), readable without mon_mu (proxy nap, stats)
  std::thread proxy;
  std::atomic<bool> stop{false};
  std::mutex qmu;
  std::condition_variable qcv;
  std::vector<Xfer> handoff;  // issued by the API thread, tracked by the proxy
  // the watchdog thread (armed transfers): no CUDA calls, so a user thread
  // blocked in a synchronous CUDA call behind a failing op can never stall
  // the failover that would release it
  std::thread watchdog;
  std::mutex amu;
  std::vector<Xfer> ahandoff;  // armed transfers issued by the API thread
  ArmedWords* armed_words = nullptr;
  std::vector<uint8_t> armed_used;  // API thread sets, watchdog clears (atomic byte ops)
  uint32_t armed_next = 0;
  uint32_t armed_seq = 1;  // generations of the K9 decision words
  std::mutex mon_mu;
  std::deque<iccl_mon_rec_t> mon;
  std::deque<iccl_switch_event_t> sw_events;
  std::atomic<int> monitor_enabled{0};
  std::atomic<int> async_err{ICCL_SUCCESS};
  std::string async_msg;
  std::mutex fault_mu;  // fault script + per-channel fault / gate state (API thread and proxy)
  std::mutex ev_mu;     // event pools (API thread and proxy)
  std::mutex relay_mu;  // relay piece counters (API thread and proxy)
  std::mutex ipc_mu;    // peer_ipc (API thread, relay server, premapping proxy)
  std::mutex open_mu;   // serialises cudaIpcOpenMemHandle (map_peer_allocation)
  std::vector<Fault> faults;
  uint64_t faults_t0 = 0;
  std::atomic<int> time_faults_pending{0};  // unfired time-triggered entries naming this rank
  std::atomic<uint64_t> tf_last{0};          // last fire_time_faults pass (rate limit)
  std::atomic<int> path_req[2 * kMaxRanks];  // API-requested switches per channel: -1 none, else target path
  std::atomic<uint64_t> pending_xfers{0};
  std::atomic<uint64_t> kernels_launched{0}, ctas_launched{0}, copies_issued{0}, bytes_issued{0};
  std::atomic<uint64_t> pulls_issued{0}, cts_timeouts{0};  // rendezvous outcomes (rzv_post)
  std::vector<cudaEvent_t> event_pool;  // proxy-owned: chunk WC events
  std::vector<cudaEvent_t> tevent_pool;  // proxy-owned: timing-enabled WC / anchor events (monitor)
  std::vector<cudaEvent_t> all_events;
  // Device time base of the timing events: base_abs_ns is base_ev's time on
  // the CLOCK_MONOTONIC scale; re-based to a recent anchor every second so
  // cudaEventElapsedTime's float ms keeps sub-100 ns precision.
  cudaEvent_t base_ev = nullptr;
  int64_t base_abs_ns = 0;
  std::deque<cudaEvent_t> old_bases;
};

namespace iccl {

static RankFlags* flags_of(iccl_comm* c, int r) { return &c->flags[r]; }
static RzvRing* ring_of(iccl_comm* c, int src, int dst) { return &c->rings[src * c->nranks + dst]; }
static PairState& pair_of(iccl_comm* c, int src, int dst) { return ring_of(c, src, dst)->st; }

// A pair needs the failover-capable (rendezvous, chunked) path when a fault
// script names it or it runs on its backup path.
static bool pair_armed(PairState& ps) {
  return ps.faults_armed.load(std::memory_order_acquire) > 0 || ps.active_path.load(std::memory_order_acquire) != 0;
}

struct RouteLock {
  PairState& ps;
  explicit RouteLock(PairState& p) : ps(p) {
    uint32_t z = 0;
    while (!ps.route_lock.compare_exchange_weak(z, 1u, std::memory_order_acquire)) {
      z = 0;
      sched_yield();
    }
  }
  ~RouteLock() { ps.route_lock.store(0, std::memory_order_release); }
};

// Re-evaluate the pair's small-op route after its fault count or active path
// changed: a new segment starts after every op either side already routed.
static void route_update(PairState& ps) {
  RouteLock lk(ps);
  const int32_t want = pair_armed(ps) ? 1 : 0;
  if (want == ps.route_rdv) return;
  const uint32_t n = ps.nseg;
  if (n >= (uint32_t)kRouteSegs) ps.route_base = ps.seg_rdv[n % kRouteSegs];  // evicted segment
  ps.seg_start[n % kRouteSegs] = std::max(ps.small_ops[0], ps.small_ops[1]);
  ps.seg_rdv[n % kRouteSegs] = want;
  ps.nseg = n + 1;
  ps.route_rdv = want;
}

// Route this side's next small op of the pair: true = rendezvous.
static bool route_small(PairState& ps, int side) {
  RouteLock lk(ps);
  const uint64_t q = ps.small_ops[side]++;
  const uint32_t n = ps.nseg, lo = n > (uint32_t)kRouteSegs ? n - kRouteSegs : 0;
  for (uint32_t i = n; i-- > lo;)
    if (ps.seg_start[i % kRouteSegs] <= q) return ps.seg_rdv[i % kRouteSegs] != 0;
  return ps.route_base != 0;
}

static void set_async(iccl_comm* c, iccl_result_t e, const std::string& msg) {
  int expected = ICCL_SUCCESS;
  if (c->async_err.compare_exchange_strong(expected, e)) {
    c->async_msg = msg;
    // like NCCL's WARN: the first asynchronous error of a communicator is
    // printed once, since the API thread may be blocked on the stream
    fprintf(stderr, "[iccl_b200 rank %d] async error %s: %s\n", c->rank, iccl_get_error_string(e), msg.c_str());
  }
}

// sense-reversing barrier over the shm header
static iccl_result_t shm_barrier(iccl_comm* c, double timeout_s = 120.0) {
  c->bar_sense ^= 1;
  int s = c->bar_sense;
  if (c->hdr->bar_count.fetch_add(1) + 1 == c->nranks) {
    c->hdr->bar_count.store(0);
    c->hdr->bar_sense.store(s);
    return ICCL_SUCCESS;
  }
  uint64_t t0 = now_ns();
  while (c->hdr->bar_sense.load() != s) {
    if (c->hdr->abort.load()) return ICCL_ERR_ABORTED;
    if ((now_ns() - t0) * 1e-9 > timeout_s) {
      set_last_error("bootstrap barrier timed out");
      return ICCL_ERR_TIMEOUT;
    }
    usleep(50);
  }
  return ICCL_SUCCESS;
}

// ---------------------------------------------------------------- proxy helpers
static iccl_result_t memop_write(cudaStream_t s, volatile void* addr, uint32_t v) {
  ICCL_TRACE("write %p <- %u on %p", (void*)addr, v, (void*)s);
  ICCL_CHECK_CU(driver()->cuStreamWriteValue32((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT));
  return ICCL_SUCCESS;
}
static iccl_result_t memop_wait(cudaStream_t s, volatile void* addr, uint32_t v) {
  ICCL_TRACE("wait %p >= %u on %p", (void*)addr, v, (void*)s);
  ICCL_CHECK_CU(driver()->cuStreamWaitValue32((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ));
  return ICCL_SUCCESS;
}

static cudaEvent_t get_event(iccl_comm* c) {
  std::lock_guard<std::mutex> g(c->ev_mu);
  if (c->event_pool.empty()) {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    c->all_events.push_back(e);
    return e;
  }
  cudaEvent_t e = c->event_pool.back();
  c->event_pool.pop_back();
  return e;
}

static cudaEvent_t get_tevent(iccl_comm* c) {
  std::lock_guard<std::mutex> g(c->ev_mu);
  if (c->tevent_pool.empty()) {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    c->all_events.push_back(e);
    return e;
  }
  cudaEvent_t e = c->tevent_pool.back();
  c->tevent_pool.pop_back();
  return e;
}

static void put_events(iccl_comm* c, Xfer& x) {
  std::lock_guard<std::mutex> g(c->ev_mu);
  for (ChunkRec& r : x.rec) {
    if (r.ev) c->event_pool.push_back(r.ev);
    if (r.tev) c->tevent_pool.push_back(r.tev);
    r.ev = r.tev = nullptr;
  }
  for (cudaEvent_t e : x.anchors) c->tevent_pool.push_back(e);
  x.anchors.clear();
  if (x.own_ready) c->event_pool.push_back(x.own_ready);
  x.own_ready = nullptr;
  x.last_ev.clear();
}

// Absolute (CLOCK_MONOTONIC-scale) ns of a completed timing event.
static uint64_t event_abs_ns(iccl_comm* c, cudaEvent_t e) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->base_ev, e) != cudaSuccess) return 0;
  return (uint64_t)(c->base_abs_ns + (int64_t)((double)ms * 1e6));
}

static void publish_one(XferPub& p, uint32_t gen, const Xfer& x) {
  p.total = x.nchunks;
  p.posted = x.next_issue;
  p.done = x.completed;
  p.path = x.path;
  p.switches = x.switches;
  p.bytes = x.bytes;
  __atomic_store_n(&p.gen, gen, __ATOMIC_RELEASE);
}

// Mirror the transfer's pointers into the sender's and the receiver's op slot.
static void publish(iccl_comm* c, const Xfer& x) {
  publish_one(flags_of(c, x.src_rank)->pub[x.s_slot], x.s_gen, x);
  publish_one(flags_of(c, x.dst_rank)->pub[x.r_done_slot], x.r_done_gen, x);
}

static int alloc_gate(iccl_comm* c) {
  std::lock_guard<std::mutex> lk(c->gate_mu);
  int g = c->next_gate++ % kGateWords;
  for (int tries = 0; c->gate_closed[g] && tries < kGateWords; tries++) g = c->next_gate++ % kGateWords;
  c->gate_closed[g] = 1;
  c->gate_words[g] = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return g;
}

static void release_gate(iccl_comm* c, int g) {
  if (g < 0) return;
  std::lock_guard<std::mutex> lk(c->gate_mu);
  __atomic_store_n((uint32_t*)&c->gate_words[g], 1u, __ATOMIC_SEQ_CST);
  c->gate_closed[g] = 0;
}

static void push_switch_event(iccl_comm* c, int peer, int to, int resume, int trigger, uint64_t detect_ns) {
  std::lock_guard<std::mutex> g(c->mon_mu);
  iccl_switch_event_t e{now_ns(), peer, to, resume, trigger, detect_ns};
  c->sw_events.push_back(e);
  if (c->sw_events.size() > 65536) c->sw_events.pop_front();
}

// Base of rank `owner`'s allocation `buffer_id` in my address space, opened
// over CUDA IPC once and cached (the analog of User Buffer Registration,
// PAPER.md:410-412).  Shared by the API thread and the relay server.
static iccl_result_t map_peer_allocation(iccl_comm* c, int owner, uint64_t buffer_id, cudaIpcMemHandle_t handle,
                                         char** base) {
  {
    std::lock_guard<std::mutex> g(c->ipc_mu);
    auto& cache = c->peer_ipc[owner];
    auto it = cache.find(buffer_id);
    if (it != cache.end()) {
      *base = it->second;
      return ICCL_SUCCESS;
    }
  }
  // opened under open_mu only (it can take tens of ms): a thread looking up
  // an already-open buffer never waits for it
  std::lock_guard<std::mutex> og(c->open_mu);
  {
    std::lock_guard<std::mutex> g(c->ipc_mu);
    auto& cache = c->peer_ipc[owner];
    auto it = cache.find(buffer_id);
    if (it != cache.end()) {  // another thread opened it meanwhile
      *base = it->second;
      return ICCL_SUCCESS;
    }
  }
  void* p = nullptr;
  ICCL_CHECK_CUDA(cudaIpcOpenMemHandle(&p, handle, cudaIpcMemLazyEnablePeerAccess));
  std::lock_guard<std::mutex> g(c->ipc_mu);
  c->peer_ipc[owner].emplace(buffer_id, (char*)p);
  *base = (char*)p;
  return ICCL_SUCCESS;
}

// Opening a peer allocation costs 0.3-55 ms (cudaIpcOpenMemHandle of a
// caching-allocator segment, 4-rank alltoallv trace), during which the
// opening thread issues nothing.  Whichever side reaches a rendezvous second
// maps the other side's tensor, so a pair that has only ever pushed meets
// that cost again the first time it pulls — and a host stalled for 45 ms
// makes every peer's send stop waiting for it and post first, i.e. more
// pulls (a 10-step alltoallv ran at 3-6 ms/step instead of 1.5, profiles/r01).
// So each new buffer is announced to the peer on first use, and the peer's
// proxy opens it in the background.
static bool announce_entry(iccl_comm* c, int peer, const AnnEntry& en) {
  Announce& a = ring_of(c, c->rank, peer)->ann;
  const uint64_t h = a.head.load(std::memory_order_relaxed);
  if (h - a.tail.load(std::memory_order_acquire) >= (uint64_t)kAnnDepth) return false;  // best effort
  a.e[h % kAnnDepth] = en;
  a.head.store(h + 1, std::memory_order_release);
  return true;
}

static void announce_buffer(iccl_comm* c, int peer, const RzvSide& s) {
  if (!c->announced[peer].insert(s.buffer_id).second) return;
  announce_entry(c, peer, AnnEntry{s.buffer_id, 0, s.handle});
}

// Peer side of iccl_deregister: drop (and close) the mapping of a buffer its
// owner retired.  Buffer ids are never reused, so a stale entry could only
// leak the mapping; closing it lets the owner's memory go.
static void unmap_peer_allocation(iccl_comm* c, int owner, uint64_t buffer_id) {
  std::lock_guard<std::mutex> og(c->open_mu);
  char* base = nullptr;
  {
    std::lock_guard<std::mutex> g(c->ipc_mu);
    auto& cache = c->peer_ipc[owner];
    auto it = cache.find(buffer_id);
    if (it == cache.end()) return;
    base = it->second;
    cache.erase(it);
  }
  cudaIpcCloseMemHandle(base);
}

// Proxy: open what peers announced (errors are ignored: the owner may have
// freed the buffer since; the issuing side maps on demand anyway).
static bool premap_peer_buffers(iccl_comm* c) {
  bool any = false;
  for (int q = 0; q < c->nranks; q++) {
    if (q == c->rank) continue;
    Announce& a = ring_of(c, q, c->rank)->ann;
    uint64_t t = a.tail.load(std::memory_order_relaxed);
    const uint64_t h = a.head.load(std::memory_order_acquire);
    for (; t < h; t++) {
      const AnnEntry en = a.e[t % kAnnDepth];
      if (en.retire) {
        unmap_peer_allocation(c, q, en.buffer_id);
        a.tail.store(t + 1, std::memory_order_release);
        any = true;
        continue;
      }
      char* base = nullptr;
      const uint64_t t0 = now_ns();
      if (map_peer_allocation(c, q, en.buffer_id, en.handle, &base) != ICCL_SUCCESS) cudaGetLastError();
      ICCL_TRACE("premapped buffer %llu of rank %d in %.1f us", (unsigned long long)en.buffer_id, q,
                 (now_ns() - t0) * 1e-3);
      a.tail.store(t + 1, std::memory_order_release);
      any = true;
    }
  }
  return any;
}

// The other side's tensor in my address space: its own pointer for a self
// pair, else inside its IPC-mapped allocation.
static iccl_result_t open_peer_buffer(iccl_comm* c, Channel& chn, const RzvSide& e, char** out) {
  if (chn.peer == c->rank) {
    *out = (char*)(uintptr_t)e.direct_ptr;
    return ICCL_SUCCESS;
  }
  char* base = nullptr;
  iccl_result_t r = map_peer_allocation(c, chn.peer, e.buffer_id, e.handle, &base);
  if (r) return r;
  *out = base + e.base_offset;
  return ICCL_SUCCESS;
}

static int engine_for(iccl_comm* c, size_t bytes) {
  if (c->cfg.transport == ICCL_TRANSPORT_SM) return ENG_SM;
  if (c->cfg.transport == ICCL_TRANSPORT_CE) return ENG_CE;
  return bytes <= c->cfg.sm_small_bytes ? ENG_SM : ENG_CE;
}

// Path p of a channel: primary (0) uses the configured engine; backup (1)
// the other one — or, for a copy-engine primary with backup_kind RELAY and a
// third GPU available, two copy-engine hops through the relay GPU.
static int path_engine(iccl_comm* c, const Channel& chn, int path, size_t bytes) {
  int prim = engine_for(c, bytes);
  if (path == 0) return prim;
  if (prim == ENG_CE && c->cfg.backup_kind == ICCL_BACKUP_RELAY && chn.relay_rank >= 0 && c->relay_buf)
    return ENG_RELAY;
  return prim == ENG_CE ? ENG_SM : ENG_CE;
}

// ---------------------------------------------------------------- GPU relay
static RelayCounter* relay_in(iccl_comm* c, int r, int src) {
  ShmLayout L(c->nranks);
  return (RelayCounter*)((char*)c->shm + L.off_relay + L.relay_box * r) + src;
}
static RelayCounter* relay_out(iccl_comm* c, int r, int src) { return relay_in(c, r, src) + c->nranks; }
static RelayReq* relay_req(iccl_comm* c, int r, int src, uint64_t q) {
  ShmLayout L(c->nranks);
  RelayReq* base = (RelayReq*)((char*)c->shm + L.off_relay + L.relay_box * r + sizeof(RelayCounter) * 2 * c->nranks);
  return base + (size_t)src * kRelayDepth + (size_t)((q - 1) % kRelayDepth);
}

static size_t relay_pieces(iccl_comm* c, size_t n) { return (n + c->relay_slot_bytes - 1) / c->relay_slot_bytes; }

// Hop 1 of one chunk: piece by piece into my staging slots on relay rr, each
// followed by its in-counter write, plus a forwarding request for rr's proxy.
// Returns ICCL_ERR_IN_PROGRESS (nothing issued) if rr's request ring is full.
static iccl_result_t relay_push(iccl_comm* c, Channel& chn, Xfer& x, size_t off, size_t n, cudaStream_t s,
                                ChunkRec& rc) {
  std::lock_guard<std::mutex> g(c->relay_mu);
  const int rr = chn.relay_rank, me = c->rank;
  const uint32_t out_now = __atomic_load_n(&relay_out(c, rr, me)->v, __ATOMIC_ACQUIRE);
  if ((int32_t)(c->relay_sent[rr] + (uint32_t)relay_pieces(c, n) - out_now) > kRelayDepth) return ICCL_ERR_IN_PROGRESS;
  if (!c->peer_relay[rr]) {
    void* p = nullptr;
    ICCL_CHECK_CUDA(cudaIpcOpenMemHandle(&p, c->ranks[rr].relay_handle, cudaIpcMemLazyEnablePeerAccess));
    c->peer_relay[rr] = (char*)p;
  }
  const size_t slot_bytes = c->relay_slot_bytes;
  for (size_t p = 0; p < n; p += slot_bytes) {
    const size_t m = std::min(slot_bytes, n - p);
    const uint32_t q = ++c->relay_sent[rr];
    const uint32_t slot = (q - 1) % kRelaySlots;
    // the slot is free once hop 2 of piece q - kRelaySlots has read it
    if (q > (uint32_t)kRelaySlots) {
      iccl_result_t r = memop_wait(s, &relay_out(c, rr, me)->v, q - kRelaySlots);
      if (r) return r;
    }
    char* stage = c->peer_relay[rr] + ((size_t)me * kRelaySlots + slot) * slot_bytes;
    ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)stage, (CUdeviceptr)(x.src + off + p), m, (CUstream)s));
    iccl_result_t r = memop_write(s, &relay_in(c, rr, me)->v, q);
    if (r) return r;
    RelayReq* rq = relay_req(c, rr, me, q);
    rq->dst = chn.peer;
    rq->slot = slot;
    rq->bytes = m;
    rq->buffer_id = x.dst_buffer_id;
    rq->base_offset = x.dst_base_offset + off + p;
    rq->handle = x.dst_handle;
    rq->seq.store(q, std::memory_order_release);
    rc.relay_q = q;
    c->copies_issued += 1;
  }
  x.relay_r = rr;
  x.relay_last_q = rc.relay_q;
  return ICCL_SUCCESS;
}

// Hop 2, on the relay: forward every published piece from every source into
// its destination buffer, in order per source, on that source's stream.
static iccl_result_t serve_relays(iccl_comm* c, bool* busy) {
  if (!c->relay_buf) return ICCL_SUCCESS;
  for (int src = 0; src < c->nranks; src++) {
    if (src == c->rank) continue;
    for (;;) {
      const uint64_t q = c->relay_next[src];
      RelayReq* rq = relay_req(c, c->rank, src, q);
      if (rq->seq.load(std::memory_order_acquire) != q) break;
      char* dbase = nullptr;
      iccl_result_t r0 = map_peer_allocation(c, rq->dst, rq->buffer_id, rq->handle, &dbase);
      if (r0) return r0;
      cudaStream_t st = c->streams[c->relay_serve[src]].s;
      const char* stage = c->relay_buf + ((size_t)src * kRelaySlots + rq->slot) * c->relay_slot_bytes;
      iccl_result_t r = memop_wait(st, &relay_in(c, c->rank, src)->v, (uint32_t)q);
      if (r) return r;
      ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)(dbase + rq->base_offset), (CUdeviceptr)stage,
                                                rq->bytes, (CUstream)st));
      r = memop_write(st, &relay_out(c, c->rank, src)->v, (uint32_t)q);
      if (r) return r;
      c->relay_next[src] = q + 1;
      c->copies_issued += 1;
      *busy = true;
    }
  }
  return ICCL_SUCCESS;
}

static bool waited_on(const Xfer& x, int path, int si) {
  return std::find(x.waited[path].begin(), x.waited[path].end(), si) != x.waited[path].end();
}

// The stream a chunk of `engine` goes to on path `path`.  The channel owns its
// copy-engine streams (which also carry a small-message pair's K1 primary);
// the backup K1 stream and the relay hop-1 stream are per rank, shared by all
// channels; ENG_CE_GROUP picks one of the rank's group streams (lane k).
static int stream_for(iccl_comm* c, Channel& chn, int path, int engine, int k) {
  if (engine == ENG_SM && path == 1) return c->sm_si;
  if (engine == ENG_RELAY) return c->relay_si;
  std::vector<int> cand;
  for (int si : chn.path_streams[path])
    if (c->streams[si].engine == (engine == ENG_CE_GROUP ? ENG_CE_GROUP : ENG_CE)) cand.push_back(si);
  return cand[k % cand.size()];
}

static void fault_up(iccl_comm* c, FaultState& fs) {
  ICCL_TRACE("gate %d opens", fs.gate);
  fs.down = false;
  release_gate(c, fs.gate);
  fs.gate = -1;
}

// A fault on directed path src -> dst applies on both endpoints (either may
// issue the pair's next transfer): on every channel of this rank that can
// issue over that path (one push or one pull channel; both for a self pair).
static void apply_fault(iccl_comm* c, FaultState& fs, bool up, uint64_t t) {
  if (!up && !fs.down) {
    fs.down = true;
    fs.gate = alloc_gate(c);
    fs.down_at = t;
  } else if (up && fs.down) {
    fault_up(c, fs);
  }
}

static void fire_time_faults(iccl_comm* c) {
  // the watchdog and the proxy call this on every pass while they spin: with
  // nothing pending they must not touch fault_mu at all, or the API thread —
  // which takes it once per chunk it issues — starves (an armed 128-chunk
  // issue took 44 ms, profiles/r02/raw/p_ac5_debug_n2.log)
  if (c->time_faults_pending.load(std::memory_order_acquire) == 0) return;
  const uint64_t now = now_ns();  // and at most every 10 us between the two threads
  uint64_t last = c->tf_last.load(std::memory_order_relaxed);
  if (now - last < 10000 || !c->tf_last.compare_exchange_strong(last, now)) return;
  std::lock_guard<std::mutex> g(c->fault_mu);
  uint64_t t = now_ns();
  for (auto& f : c->faults) {
    if (f.fired || f.f.trigger_kind != 0) continue;
    if (f.f.src != c->rank && f.f.dst != c->rank) continue;
    if (t - c->faults_t0 < f.f.t_us * 1000ull) continue;
    f.fired = true;
    c->time_faults_pending.fetch_sub(1);
    ICCL_TRACE("time fault %s path %d of %d->%d fires at +%.1f us", f.f.up ? "Up" : "Down", f.f.path, f.f.src, f.f.dst,
               (t - c->faults_t0) * 1e-3);
    for (Channel& chn : c->ch)
      if (chn.src == f.f.src && chn.dst == f.f.dst) apply_fault(c, chn.fault[f.f.path & 1], f.f.up, t);
  }
}

// Chunk-triggered: fires when this rank issues chunk `chunk` of the
// op_index-th transfer of the pair (counted from iccl_fault_set).  Caller
// holds fault_mu.
static void fire_chunk_faults(iccl_comm* c, Channel& chn, int op_index, int chunk, int path) {
  for (auto& f : c->faults) {
    if (f.fired || f.f.trigger_kind != 1 || f.f.src != chn.src || f.f.dst != chn.dst) continue;
    if (f.f.op_index != op_index || f.f.chunk != chunk || (f.f.path & 1) != path) continue;
    f.fired = true;
    ICCL_TRACE("chunk fault %s path %d of %d->%d fires at chunk %d (+%.1f us)", f.f.up ? "Up" : "Down", path, chn.src,
               chn.dst, chunk, (now_ns() - c->faults_t0) * 1e-3);
    FaultState& fs = chn.fault[path];
    if (!f.f.up && !fs.down) {
      fs.down = true;
      fs.gate = alloc_gate(c);
      fs.down_at = now_ns();
    } else if (f.f.up && fs.down) {
      fault_up(c, fs);
    }
  }
}

static int chunk_stream(iccl_comm* c, Channel& chn, const Xfer& x, int path, int eng, int k) {
  return (eng == ENG_CE && x.group_stream) ? stream_for(c, chn, path, ENG_CE_GROUP, x.group_lane)
                                            : stream_for(c, chn, path, eng, k);
}

// The ready waits of a transfer's first chunk, enqueued ahead of time (a
// group's pushes, see iccl_group_end).
// hostFunc#1 analog: a copy stream may start the op only once both user
// streams reached it
static iccl_result_t wait_both_ready(iccl_comm* c, cudaStream_t s, const Xfer& x) {
  if (x.own_ready && x.own_side == 0) {
    ICCL_CHECK_CUDA(cudaStreamWaitEvent(s, x.own_ready, 0));
  } else {
    iccl_result_t r = memop_wait(s, &flags_of(c, x.src_rank)->ready[x.s_slot], x.s_gen);
    if (r) return r;
  }
  if (x.own_ready && x.own_side == 1) {
    ICCL_CHECK_CUDA(cudaStreamWaitEvent(s, x.own_ready, 0));
    return ICCL_SUCCESS;
  }
  return memop_wait(s, &flags_of(c, x.dst_rank)->ready[x.r_ready_slot], x.r_ready_gen);
}

static iccl_result_t ready_waits(iccl_comm* c, Channel& chn, Xfer& x) {
  const int eng = path_engine(c, chn, x.path, x.bytes);
  if (eng != ENG_CE) return ICCL_SUCCESS;
  const int si = chunk_stream(c, chn, x, x.path, eng, 0);
  if (waited_on(x, x.path, si)) return ICCL_SUCCESS;
  iccl_result_t r = wait_both_ready(c, c->streams[si].s, x);
  if (r) return r;
  x.waited[x.path].push_back(si);
  return ICCL_SUCCESS;
}

static iccl_result_t issue_chunk(iccl_comm* c, Channel& chn, Xfer& x, int k) {
  const int path = x.path;
  const int eng = path_engine(c, chn, path, x.bytes);
  const size_t off = (size_t)k * x.chunk;
  const size_t n = std::min(x.chunk, x.bytes - off);
  const int si = chunk_stream(c, chn, x, path, eng, k);
  StreamCtx& sc = c->streams[si];
  RankFlags* sender = flags_of(c, x.src_rank);
  RankFlags* receiver = flags_of(c, x.dst_rank);
  if (!waited_on(x, path, si)) {
    iccl_result_t r = wait_both_ready(c, sc.s, x);
    if (r) return r;
    x.waited[path].push_back(si);
  }
  {
    bool anchored = false;
    for (auto& le : x.last_ev) anchored |= le.first == si;
    if (!anchored && eng == ENG_CE && c->monitor_enabled.load(std::memory_order_relaxed)) {
      // monitor anchor (the op's start on this stream): an untimed event on
      // the copy stream bridged to a timing event on the monitor stream
      cudaEvent_t a = get_tevent(c);
      x.anchors.push_back(a);
      cudaStream_t ms = c->streams[chn.mon_stream].s;
      ICCL_CHECK_CUDA(cudaEventRecord(chn.bridge, sc.s));
      ICCL_CHECK_CUDA(cudaStreamWaitEvent(ms, chn.bridge, 0));
      ICCL_CHECK_CUDA(cudaEventRecord(a, ms));
      x.last_ev.emplace_back(si, a);
    }
  }
  {
    std::lock_guard<std::mutex> g(c->fault_mu);
    if (x.fault_ops_index >= 0) fire_chunk_faults(c, chn, x.fault_ops_index, k, path);
    if (chn.fault[path].down) {
      iccl_result_t r = memop_wait(sc.s, &c->gate_words[chn.fault[path].gate], 1);
      if (r) return r;
      x.gated = true;
    }
  }
  ChunkRec& rc = x.rec[k];
  rc.t1 = now_ns();
  rc.relay_q = 0;
  rc.path = path;
  rc.stream = si;
  rc.done = false;
  rc.stamp = -1;
  // Monitor on, SM path: K1 itself stamps the chunk's WR/WC pair with
  // %globaltimer (K4 epilogue) and the t2 stamp doubles as the WC the proxy
  // polls.  Copy-engine path: the WC is an untimed event after the chunk;
  // with the monitor on, the channel's monitor stream waits for it and
  // records a timing event, whose device time (and the previous one, the
  // chunk's start) give t1/t2 with no kernel — the path stays at 0 SMs — and
  // without a timing event between copies (2.7 us of copy-engine stall per
  // chunk, profiles/r01/probe5b.txt).  A stream memop there would cost a full
  // copy-engine drain per chunk (probes/p2p_probe3).
  const bool mon = c->monitor_enabled.load(std::memory_order_relaxed);
  KernelStamp* st = nullptr;
  if (mon && eng == ENG_SM) {
    rc.stamp = c->next_stamp.fetch_add(1) % kStampSlots;
    st = &c->stamps[rc.stamp];
    memset((void*)st, 0, sizeof(KernelStamp));
  }
  rc.t1ev = nullptr;
  if (mon && eng == ENG_CE) {
    for (auto& le : x.last_ev)
      if (le.first == si) rc.t1ev = le.second;
  }
  if (eng == ENG_CE) {
    ICCL_TRACE("copy op %llu chunk %d: %zu B on %p", (unsigned long long)x.op_seq, k, n, (void*)sc.s);
    ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)(x.dst + off), (CUdeviceptr)(x.src + off), n, (CUstream)sc.s));
    ICCL_TRACE("copy issued");
    c->copies_issued += 1;
  } else if (eng == ENG_RELAY) {
    // two copy-engine hops through the relay GPU; the WC is the relay's
    // out-counter reaching the chunk's last piece (no event, no kernel)
    iccl_result_t r = relay_push(c, chn, x, off, n, sc.s, rc);
    if (r) return r;
  } else {
    ICCL_TRACE("K1 op %llu chunk %d: %zu B on %p", (unsigned long long)x.op_seq, k, n, (void*)sc.s);
    int grid = 0;
    ICCL_CHECK_CUDA(launch_copy(x.src + off, x.dst + off, n, c->cfg.sm_cap, st, sc.s, &grid));
    c->ctas_launched += grid;
    c->copies_issued += 1;
  }
  c->kernels_launched += eng == ENG_SM ? 1 : 0;
  c->bytes_issued += n;
  if (!st && eng != ENG_RELAY) {
    if (!rc.ev) rc.ev = get_event(c);
    ICCL_TRACE("event record");
    ICCL_CHECK_CUDA(cudaEventRecord(rc.ev, sc.s));
    ICCL_TRACE("event recorded");
    if (mon && eng == ENG_CE) {
      if (!rc.tev) rc.tev = get_tevent(c);
      cudaStream_t ms = c->streams[chn.mon_stream].s;
      ICCL_CHECK_CUDA(cudaStreamWaitEvent(ms, rc.ev, 0));
      ICCL_CHECK_CUDA(cudaEventRecord(rc.tev, ms));
      for (auto& le : x.last_ev)
        if (le.first == si) le.second = rc.tev;
    } else if (rc.tev) {
      std::lock_guard<std::mutex> g(c->ev_mu);
      c->tevent_pool.push_back(rc.tev);
      rc.tev = nullptr;
    }
  }
  iccl_result_t r = ICCL_SUCCESS;
  if (k == x.nchunks - 1 && x.gated) {
    // Some chunk of this attempt waits behind a closed gate: a switch will
    // release that gate at once (a parked stream stalls unrelated streams),
    // so done writes queued here would fire after the flushed stale copies —
    // while the re-issued suffix is still writing the receiver's buffer and
    // reading the sender's.  The attempt that completes the op writes them.
    x.done_deferred = true;
  } else if (k == x.nchunks - 1) {
    // completion (hostFunc#2 analog): join every stream that carried chunks of
    // this op, plus the fences of paths abandoned by a switch, then release
    // both user streams.
    for (int p = 0; p < 2; p++) {
      for (int sj : chn.path_streams[p]) {
        if (sj == si || !waited_on(x, p, sj)) continue;
        StreamCtx& o = c->streams[sj];
        ICCL_CHECK_CUDA(cudaEventRecord(o.ev, o.s));
        ICCL_CHECK_CUDA(cudaStreamWaitEvent(sc.s, o.ev, 0));
      }
    }
    for (cudaEvent_t fe : x.fences) ICCL_CHECK_CUDA(cudaStreamWaitEvent(sc.s, fe, 0));
    if (x.relay_r >= 0) {
      // every piece that went through the relay must have been forwarded
      r = memop_wait(sc.s, &relay_out(c, x.relay_r, c->rank)->v, x.relay_last_q);
      if (r) return r;
    }
    r = memop_write(sc.s, &receiver->done[x.r_done_slot], x.r_done_gen);
    if (r) return r;
    r = memop_write(sc.s, &sender->done[x.s_slot], x.s_gen);
    if (r) return r;
    x.done_enqueued = true;
  }
  return ICCL_SUCCESS;
}

// switch_qp: receiver-driven breakpoint.  The receiver's
// done (contiguous delivered prefix) is where retransmission resumes; posted
// and transmitted retreat to it; stale in-flight work on the abandoned path is
// fenced so completion waits for it.
//
// Which transfers move: a watchdog switch (trigger 1: the path stalled)
// migrates every unfinished transfer on the pair.  A voluntary switch (an API
// switch_qp, trigger 0, or the switch back after a successful probe, trigger
// 2) leaves a transfer whose done writes are already queued behind its last
// chunk on a healthy path to finish there — re-issuing it would let those
// writes release both user streams while the re-issued copies still run —
// and moves the rest from their next chunk on, without retreat.  In-stream
// transfers are never moved (their copies sit on the user's stream).
static iccl_result_t switch_path(iccl_comm* c, Channel& chn, int to, int trigger) {
  PairState& ps = pair_of(c, chn.src, chn.dst);
  const bool voluntary = trigger != 1;
  auto movable = [&](const Xfer& x) {
    return x.path != to && !x.instream && !(voluntary && x.done_enqueued && !x.gated);
  };
  bool moves = false;
  for (Xfer& x : chn.xfers) moves |= movable(x);
  if (!moves && ps.active_path.load() == to) return ICCL_SUCCESS;
  const int from = to ^ 1;
  std::unique_lock<std::mutex> lk(c->fault_mu);
  uint64_t detect = chn.fault[from].down ? now_ns() - chn.fault[from].down_at : 0;
  int resume = -1;
  int stale_gate = chn.fault[from].down ? chn.fault[from].gate : -1;
  for (Xfer& x : chn.xfers) {
    if (!movable(x)) continue;
    if (voluntary && !x.gated) {
      // healthy path: chunks already queued there complete there; the rest
      // (and the done writes, which join every stream the op used) go on the
      // new path
      if (resume < 0) resume = x.next_issue;
      x.path = to;
      x.switches++;
      x.last_progress = now_ns();
      publish(c, x);
      continue;
    }
    // fence: an event after everything already queued on the abandoned path
    bool had_work = x.next_issue > x.completed || x.done_enqueued;
    if (had_work) {
      for (int sj : chn.path_streams[from]) {
        if (!waited_on(x, from, sj)) continue;
        cudaEvent_t fe;
        ICCL_CHECK_CUDA(cudaEventCreateWithFlags(&fe, cudaEventDisableTiming));
        ICCL_CHECK_CUDA(cudaEventRecord(fe, c->streams[sj].s));
        x.fences.push_back(fe);
      }
    }
    if (resume < 0) resume = x.completed;
    // retreat: posted = transmitted = acked = done
    x.next_issue = x.completed;
    x.path = to;
    x.done_enqueued = false;
    x.gated = false;
    x.done_deferred = false;
    x.switches++;
    x.last_progress = now_ns();
    publish(c, x);
  }
  if (stale_gate >= 0) {
    // Future work on the still-Down path waits on a fresh gate epoch; the old
    // gate is released right away: its copies are flushed (SPEC.md:285's
    // Flushed WCs) — they rewrite the bytes the new path delivers, and the
    // op's completion waits for them through the fences above.  Leaving a
    // stream parked would also stall every stream sharing its hardware queue
    // (a failover step took 1.29 s that way, profiles/r01/README.md).
    chn.fault[from].gate = alloc_gate(c);
    release_gate(c, stale_gate);
  }
  lk.unlock();
  chn.failed_over = (to == 1 && trigger == 1);
  ps.active_path.store(to);
  ps.switches.fetch_add(1);
  route_update(ps);
  chn.probe_out = false;  // abandon the outstanding probe
  chn.last_probe = now_ns();
  ICCL_TRACE("switch pair %d->%d to path %d at chunk %d (trigger %d, detect %llu ns)", chn.src, chn.dst, to, resume,
             trigger, (unsigned long long)detect);
  push_switch_event(c, chn.peer, to, resume, trigger, detect);
  return ICCL_SUCCESS;
}

static void retire_probe(iccl_comm* c, Channel& chn) {
  (void)c;
  chn.probe_out = false;
}

// The CTS probe of check_receiver_timeout / monitor_failed_link
// (SPEC.md:246-273).  Over an injected-Down path it is lost: nothing is
// enqueued (a probe parked on the device would stall every stream sharing its
// hardware queue) and the proxy sees no completion within delta.
static iccl_result_t send_probe(iccl_comm* c, Channel& chn, int path) {
  const int si = chn.probe_stream;
  StreamCtx& sc = c->streams[si];
  bool down;
  {
    std::lock_guard<std::mutex> g(c->fault_mu);
    down = chn.fault[path].down;
  }
  chn.probe_out = true;
  chn.probe_sent = now_ns();
  chn.probe_path = path;
  if (down) {
    chn.probe_ticket_expect = sc.ticket + 0x40000000u;  // never reached
    return ICCL_SUCCESS;
  }
  // a 16-byte CTS over the suspect path: into the peer's scratch (push
  // channel) or out of it (pull channel)
  if (chn.dir == 0)
    ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)chn.peer_scratch, (CUdeviceptr)c->scratch, 16, (CUstream)sc.s));
  else
    ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)(c->scratch + 2048 + 16 * chn.peer),
                                              (CUdeviceptr)chn.peer_scratch, 16, (CUstream)sc.s));
  chn.probe_ticket_expect = ++sc.ticket;
  return memop_write(sc.s, sc.prog, chn.probe_ticket_expect);
}

static void record_monitor(iccl_comm* c, Channel& chn, Xfer& x, int k, uint64_t t2_host) {
  ChunkRec& rc = x.rec[k];
  iccl_mon_rec_t m{};
  m.t1_ns = rc.t1;
  m.t2_ns = t2_host;
  if (rc.tev && rc.t1ev) {
    // copy-engine path: device times of the chunk's start / end events
    uint64_t a = event_abs_ns(c, rc.t1ev), b = event_abs_ns(c, rc.tev);
    if (a && b && b >= a) {
      m.t1_ns = a;
      m.t2_ns = b;
    }
    // keep the float-ms elapsed time short: re-base once a second
    if (b > (uint64_t)c->base_abs_ns + 1000000000ull) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, c->base_ev, rc.tev) == cudaSuccess) {
        cudaEvent_t nb = rc.tev;  // ownership moves to the time base
        rc.tev = nullptr;
        // a later chunk of this op may still name the old base as its start
        // event: recycle it only two re-bases (>= 2 s) later
        c->old_bases.push_back(c->base_ev);
        if (c->old_bases.size() > 2) {
          std::lock_guard<std::mutex> g(c->ev_mu);
          c->tevent_pool.push_back(c->old_bases.front());
          c->old_bases.pop_front();
        }
        c->base_ev = nb;
        c->base_abs_ns += (int64_t)((double)ms * 1e6);
      }
    }
  } else if (rc.stamp >= 0) {
    KernelStamp* st = &c->stamps[rc.stamp];
    unsigned long long t1 = st->t1, t2 = st->t2;
    if (t1 && t2 && t2 > t1) {
      m.t1_ns = (uint64_t)((int64_t)t1 + c->gtimer_offset);
      m.t2_ns = (uint64_t)((int64_t)t2 + c->gtimer_offset);
    }
  }
  m.bytes = std::min(x.chunk, x.bytes - (size_t)k * x.chunk);
  m.peer = chn.peer;
  m.path = rc.path;
  m.chunk = k;
  m.dir = chn.dir;
  m.op_seq = x.op_seq;
  std::lock_guard<std::mutex> g(c->mon_mu);
  c->mon.push_back(m);
  if (c->mon.size() > (1u << 20)) c->mon.pop_front();
}

// One proxy pass over a channel: completions, retirement, re-issue after a
// path switch, watchdog.  Sets *busy if anything moved.
static iccl_result_t progress_channel(iccl_comm* c, Channel& chn, bool* busy) {
  iccl_result_t r;
  if (chn.xfers.empty()) return ICCL_SUCCESS;
  // 2. completions: advance each xfer's contiguous delivered prefix (acked / done)
  const uint64_t tnow = now_ns();
  for (Xfer& x : chn.xfers) {
    while (x.completed < x.next_issue) {
      ChunkRec& rc = x.rec[x.completed];
      if (rc.relay_q) {
        if (!cyc_geq(__atomic_load_n(&relay_out(c, x.relay_r, c->rank)->v, __ATOMIC_ACQUIRE), rc.relay_q)) break;
      } else if (rc.stamp >= 0) {
        if (__atomic_load_n(&c->stamps[rc.stamp].t2, __ATOMIC_ACQUIRE) == 0) break;
      } else {
        cudaError_t q = cudaEventQuery(rc.tev ? rc.tev : rc.ev);
        if (q == cudaErrorNotReady) break;
        if (q != cudaSuccess) {
          set_last_error(std::string("chunk completion: ") + cudaGetErrorString(q));
          return ICCL_ERR_CUDA;
        }
      }
      rc.done = true;
      if (c->monitor_enabled.load(std::memory_order_relaxed)) record_monitor(c, chn, x, x.completed, tnow);
      x.completed++;
      x.last_progress = tnow;
      *busy = true;
    }
    if (x.done_deferred && !x.done_enqueued && x.completed == x.nchunks) {
      // every chunk of a gated attempt landed (its gate opened): release both
      // user streams from the host once the fenced stale copies (if any) and
      // the relay's forwarding drained
      bool drained = !(x.relay_r >= 0 && !cyc_geq(__atomic_load_n(&relay_out(c, x.relay_r, c->rank)->v,
                                                                  __ATOMIC_ACQUIRE), x.relay_last_q));
      for (cudaEvent_t fe : x.fences) drained = drained && cudaEventQuery(fe) == cudaSuccess;
      if (drained) {
        __atomic_store_n(&flags_of(c, x.dst_rank)->done[x.r_done_slot], x.r_done_gen, __ATOMIC_SEQ_CST);
        __atomic_store_n(&flags_of(c, x.src_rank)->done[x.s_slot], x.s_gen, __ATOMIC_SEQ_CST);
        x.done_enqueued = true;
        *busy = true;
      }
    }
    publish(c, x);
  }
  // 3. retire completed xfers (their done writes are queued on the device)
  while (!chn.xfers.empty()) {
    Xfer& x = chn.xfers.front();
    if (!(x.completed == x.nchunks && x.done_enqueued)) break;
    if (!x.fences.empty()) {
      // fences may only be destroyed after the device consumed them; the
      // done flag write follows them on the same stream
      if (!cyc_geq(flags_of(c, x.src_rank)->done[x.s_slot], x.s_gen)) break;
      for (cudaEvent_t fe : x.fences) cudaEventDestroy(fe);
      x.fences.clear();
    }
    ICCL_TRACE("retire op %llu (pair %d->%d #%llu)", (unsigned long long)x.op_seq, x.src_rank, x.dst_rank,
               (unsigned long long)x.pair_seq);
    put_events(c, x);
    chn.xfers.pop_front();
    c->pending_xfers.fetch_sub(1);
    *busy = true;
  }
  // 4. re-issue after a path switch (posted - acked <= window); the API
  // thread issued every chunk of the original attempt itself
  int outstanding = 0;
  for (Xfer& x : chn.xfers) outstanding += x.next_issue - x.completed;
  for (Xfer& x : chn.xfers) {
    bool stalled = false;
    while (x.next_issue < x.nchunks && outstanding < c->cfg.window) {
      r = issue_chunk(c, chn, x, x.next_issue);
      if (r == ICCL_ERR_IN_PROGRESS) {  // relay ring full: retry on a later pass
        stalled = true;
        break;
      }
      if (r) return r;
      x.next_issue++;
      outstanding++;
      *busy = true;
      publish(c, x);
    }
    if (stalled || x.next_issue < x.nchunks) break;
  }
  // 5. watchdog + probe (check_receiver_timeout); in-stream
  // transfers cannot be migrated, so they are not watched
  if (!chn.xfers.empty() && !chn.xfers.front().instream) {
    Xfer& x = chn.xfers.front();
    bool elig = cyc_geq(flags_of(c, x.src_rank)->ready[x.s_slot], x.s_gen) &&
                cyc_geq(flags_of(c, x.dst_rank)->ready[x.r_ready_slot], x.r_ready_gen);
    if (!elig) {
      x.last_progress = tnow;  // innocent stall upstream: the sender's data is not ready
    } else if (!x.eligible) {
      x.eligible = true;
      x.last_progress = tnow;
    }
    const uint64_t delta = c->cfg.delta_us * 1000ull;
    if (elig && x.completed < x.next_issue && tnow - x.last_progress > delta) {
      if (!chn.probe_out) {
        r = send_probe(c, chn, x.path);
        if (r) return r;
      } else if (chn.probe_path == x.path) {
        StreamCtx& ps = c->streams[chn.probe_stream];
        if (cyc_geq(*ps.prog, chn.probe_ticket_expect)) {
          retire_probe(c, chn);  // CTS ok: innocent link
          x.last_progress = tnow;
        } else if (tnow - chn.probe_sent > delta) {
          // CTS failed: trigger the switch
          r = switch_path(c, chn, x.path ^ 1, 1);
          if (r) return r;
          *busy = true;
        }
      }
    }
  }
  return ICCL_SUCCESS;
}

// monitor_failed_link: while on the backup, probe the
// primary every probe period; a probe that completes switches back.
static iccl_result_t monitor_failed_link(iccl_comm* c, Channel& chn) {
  if (!chn.failed_over || pair_of(c, chn.src, chn.dst).active_path.load() != 1) return ICCL_SUCCESS;
  const uint64_t t = now_ns();
  StreamCtx& ps = c->streams[chn.probe_stream];
  if (chn.probe_out) {
    if (cyc_geq(*ps.prog, chn.probe_ticket_expect)) {
      const bool primary_ok = chn.probe_path == 0;  // the probe crossed the primary path
      retire_probe(c, chn);
      if (primary_ok) return switch_path(c, chn, 0, 2);
    } else if (t - chn.probe_sent > c->cfg.delta_us * 1000ull) {
      retire_probe(c, chn);  // probe lost: the primary is still down
      chn.last_probe = t;
    }
    return ICCL_SUCCESS;
  }
  if (t - chn.last_probe >= c->cfg.probe_period_us * 1000ull) {
    chn.last_probe = t;
    return send_probe(c, chn, 0);
  }
  return ICCL_SUCCESS;
}

// Monitor records of K5 sends and K6 ops (the proxy does not track them as
// transfers): emitted once the kernel's t2 stamp lands, in completion order.
static bool drain_kstamps(iccl_comm* c) {
  std::lock_guard<std::mutex> g(c->mon_mu);
  bool any = false;
  for (auto it = c->krecs.begin(); it != c->krecs.end();) {
    KernelStamp* st = &c->stamps[it->stamp];
    const unsigned long long t2 = __atomic_load_n(&st->t2, __ATOMIC_ACQUIRE);
    if (!t2) {
      ++it;
      continue;
    }
    const unsigned long long t1 = __atomic_load_n(&st->t1, __ATOMIC_ACQUIRE);
    iccl_mon_rec_t m{};
    m.t1_ns = (uint64_t)((int64_t)(t1 ? t1 : t2) + c->gtimer_offset);
    m.t2_ns = (uint64_t)((int64_t)t2 + c->gtimer_offset);
    m.bytes = it->bytes;
    m.peer = it->peer;
    m.path = ICCL_PATH_PRIMARY;
    m.chunk = 0;
    m.dir = it->dir;
    m.op_seq = it->op_seq;
    c->mon.push_back(m);
    if (c->mon.size() > (1u << 20)) c->mon.pop_front();
    it = c->krecs.erase(it);
    c->krecs_pending.fetch_sub(1);
    any = true;
  }
  return any;
}

static void proxy_loop(iccl_comm* c) {
  cudaSetDevice(c->dev);
  if (c->cfg.proxy_cpu >= 0) {
    cpu_set_t set;
    CPU_ZERO(&set);
    CPU_SET(c->cfg.proxy_cpu, &set);
    pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
  }
  std::vector<Xfer> batch;
  uint64_t idle_since = now_ns();
  while (!c->stop.load(std::memory_order_relaxed)) {
    bool busy = false;
    {
      std::unique_lock<std::mutex> lk(c->qmu);
      if (c->handoff.empty() && c->pending_xfers.load() == 0 && c->krecs_pending.load() == 0 &&
          now_ns() - idle_since > 200000) {
        // a relay GPU has no transfers of its own: nap shorter so its
        // forwarding (hop 2) starts within ~50 us of a request
        c->qcv.wait_for(lk, std::chrono::microseconds(c->relay_buf ? 50 : 500));
      }
      batch.swap(c->handoff);
    }
    for (Xfer& x : batch) {
      Channel& chn = c->ch[x.chan];
      chn.xfers.push_back(std::move(x));
      busy = true;
    }
    batch.clear();
    if (c->async_err.load() != ICCL_SUCCESS) {
      usleep(100);
      continue;
    }
    fire_time_faults(c);
    busy |= premap_peer_buffers(c);
    busy |= drain_kstamps(c);
    for (int ci = 0; ci < 2 * c->nranks; ci++) {
      Channel& chn = c->ch[ci];
      int req = c->path_req[ci].exchange(-1);
      iccl_result_t r = ICCL_SUCCESS;
      if (req >= 0) r = switch_path(c, chn, req, 0);
      if (!r) r = progress_channel(c, chn, &busy);
      if (!r) r = monitor_failed_link(c, chn);
      if (r) {
        set_async(c, r, std::string("proxy: ") + last_error());
        break;
      }
    }
    {
      iccl_result_t r = serve_relays(c, &busy);
      if (r) set_async(c, r, std::string("relay: ") + last_error());
    }
    if (c->hdr->abort.load()) set_async(c, ICCL_ERR_ABORTED, "communicator aborted");
    if (c->ll_error && __atomic_load_n(c->ll_error, __ATOMIC_ACQUIRE))
      set_async(c, ICCL_ERR_TIMEOUT, "LL / direct kernel wait exceeded 10 s (peer never posted the matching op)");
    if (busy) {
      idle_since = now_ns();
    } else {
      // Nothing moved: back off before the next pass.  Every cudaEventQuery
      // takes the context lock the API thread needs to enqueue transfers, so
      // a spinning proxy would slow the issuing thread down; completion is
      // not latency-critical here (the device writes the done flags itself).
      std::this_thread::sleep_for(std::chrono::microseconds(kProxyNapUs));
    }
  }
}

// Reserve the next op slot; a slot is reused only after its previous op completed.
static iccl_result_t next_slot(iccl_comm* c, uint32_t* slot, uint32_t* gen, uint64_t* seq) {
  uint64_t s = c->op_seq++;
  *seq = s;
  *slot = (uint32_t)(s % kSlots);
  *gen = (uint32_t)(s + 1);
  if (s >= (uint64_t)kSlots) {
    uint32_t prev = (uint32_t)(s + 1 - kSlots);
    uint64_t t0 = now_ns();
    while (!cyc_geq(flags_of(c, c->rank)->done[*slot], prev)) {
      if (c->async_err.load() != ICCL_SUCCESS) return (iccl_result_t)c->async_err.load();
      if (now_ns() - t0 > 60ull * 1000000000ull) {
        set_last_error("more than 4096 ops in flight for 60 s");
        return ICCL_ERR_TIMEOUT;
      }
      sched_yield();
    }
  }
  // ready is written by the stream; clear stale content is not needed (cyclic gens)
  return ICCL_SUCCESS;
}

}  // namespace iccl

// Export the allocation holding `buf` over CUDA IPC (cached by buffer id) so
// the peer can map it: the zero-copy registration of SPEC.md:126-129.
static iccl_result_t export_buffer(iccl_comm* c, const void* buf, RzvSide* side) {
  CUdeviceptr base = 0;
  size_t asize = 0;
  ICCL_CHECK_CU(driver()->cuMemGetAddressRange(&base, &asize, (CUdeviceptr)buf));
  unsigned long long bid = 0;
  ICCL_CHECK_CU(driver()->cuPointerGetAttribute(&bid, CU_POINTER_ATTRIBUTE_BUFFER_ID, (CUdeviceptr)buf));
  auto it = c->export_cache.find(bid);
  if (it == c->export_cache.end()) {
    cudaIpcMemHandle_t h;
    cudaError_t err = cudaIpcGetMemHandle(&h, (void*)base);
    if (err != cudaSuccess) {
      set_last_error(std::string("cannot export the buffer for zero-copy (") + cudaGetErrorString(err) +
                     "); allocate it with cudaMalloc / the torch caching allocator without expandable segments");
      return ICCL_ERR_UNREGISTERED_REGION;
    }
    it = c->export_cache.emplace(bid, h).first;
  }
  side->handle = it->second;
  side->buffer_id = bid;
  side->base_offset = (uint64_t)((CUdeviceptr)buf - base);
  return ICCL_SUCCESS;
}

static RzvEntry& rzv_entry(iccl_comm* c, int kind, int peer, uint64_t k) {
  const int src = kind == 0 ? c->rank : peer, dst = kind == 0 ? peer : c->rank;
  return ring_of(c, src, dst)->e[k % kRzvDepth];
}

static bool rzv_claim(RzvEntry& e, uint64_t k) {
  uint64_t g = k / kRzvDepth;
  return e.claimed.compare_exchange_strong(g, g + 1, std::memory_order_acq_rel);
}

// The entry holds op k's halves once both sides arrived for its previous
// generation and that transfer was claimed (its halves were copied out).
static bool rzv_free(const RzvEntry& e, uint64_t k) {
  const uint64_t g = k / kRzvDepth;
  return e.arrivals.load(std::memory_order_acquire) >= 2 * g && e.claimed.load(std::memory_order_acquire) >= g;
}

// Count my arrival at op k (my half is already in e.side): the side that
// arrives second copies both halves out and claims the transfer; true then.
static bool rzv_arrive(RzvEntry& e, uint64_t k, RzvSide snap[2]) {
  const uint64_t g = k / kRzvDepth;
  if (e.arrivals.fetch_add(1, std::memory_order_acq_rel) != 2 * g + 1) return false;
  snap[0] = e.side[0];  // before the claim: after it a peer kRzvDepth ops ahead may reuse the entry
  snap[1] = e.side[1];
  return rzv_claim(e, k);  // cannot fail: the first side never claims
}

// Build the transfer of rendezvous entry k of the pair (as `kind`: 0 = push
// by the sender, 1 = pull by the receiver) from the entry's two halves
// `side`, copied out of the shared entry before the claim (after the claim a
// peer up to kRzvDepth ops ahead may already reuse it); no device work yet.
static iccl_result_t rzv_build(iccl_comm* c, int kind, int peer, uint64_t k, uint64_t op_seq, bool group,
                               const RzvSide* side, Xfer* out) {
  const int src = kind == 0 ? c->rank : peer, dst = kind == 0 ? peer : c->rank;
  const RzvSide& snd = side[0];
  const RzvSide& rcv = side[1];
  if (snd.bytes != rcv.bytes) {
    // release both streams so nothing hangs, and report the mismatch
    __atomic_store_n(&flags_of(c, src)->done[snd.slot], snd.gen, __ATOMIC_SEQ_CST);
    __atomic_store_n(&flags_of(c, dst)->done[rcv.slot], rcv.gen, __ATOMIC_SEQ_CST);
    std::string msg = "send of " + std::to_string(snd.bytes) + " B from rank " + std::to_string(src) +
                      " matched a recv of " + std::to_string(rcv.bytes) + " B on rank " + std::to_string(dst);
    set_async(c, ICCL_ERR_SIZE_MISMATCH, msg);
    set_last_error(msg);
    return ICCL_ERR_SIZE_MISMATCH;
  }
  const int ci = 2 * peer + kind;
  Channel& chn = c->ch[ci];
  Xfer& x = *out;
  x.op_seq = op_seq;
  x.pair_seq = k;
  x.src_rank = src;
  x.dst_rank = dst;
  x.chan = ci;
  char* other = nullptr;
  iccl_result_t r = open_peer_buffer(c, chn, side[kind ^ 1], &other);
  if (r) return r;
  char* own = (char*)(uintptr_t)side[kind].direct_ptr;
  x.src = kind == 0 ? own : other;
  x.dst = kind == 0 ? other : own;
  x.bytes = snd.bytes;
  x.s_slot = snd.slot;
  x.s_gen = snd.gen;
  x.r_ready_slot = x.r_done_slot = rcv.slot;
  x.r_ready_gen = x.r_done_gen = rcv.gen;
  x.dst_buffer_id = rcv.buffer_id;
  x.dst_base_offset = rcv.base_offset;
  x.dst_handle = rcv.handle;
  x.chunk = (size_t)c->cfg.chunk_bytes;
  x.nchunks = (int)((x.bytes + x.chunk - 1) / x.chunk);
  x.rec.resize(x.nchunks);
  x.path = pair_of(c, src, dst).active_path.load();
  x.last_progress = now_ns();
  x.group_stream = group && peer != c->rank;
  {
    std::lock_guard<std::mutex> gl(c->fault_mu);
    x.fault_ops_index = (int)(k - chn.fault_seq_base);
  }
  ICCL_TRACE("issue %s pair %d->%d #%llu, %zu B, %d chunk(s), path %d", kind == 0 ? "push" : "pull", src, dst,
             (unsigned long long)k, x.bytes, x.nchunks, x.path);
  return ICCL_SUCCESS;
}

// Hand an issued transfer to the proxy (completions, six pointers, monitor,
// watchdog) — or, issued by the proxy itself, track it in place.
static void rzv_track(iccl_comm* c, Xfer&& x, bool on_proxy) {
  publish(c, x);
  c->pending_xfers.fetch_add(1);
  if (on_proxy) {
    c->ch[x.chan].xfers.push_back(std::move(x));
    return;
  }
  {
    std::lock_guard<std::mutex> gl(c->qmu);
    c->handoff.push_back(std::move(x));
  }
  c->qcv.notify_one();
}

// Enqueue every chunk of a built transfer on the side streams (each behind
// waits on both user streams' ready flags, the last one writing both done
// flags) and hand it to the proxy.
static iccl_result_t rzv_launch(iccl_comm* c, Xfer&& x, bool on_proxy) {
  Channel& chn = c->ch[x.chan];
  while (x.next_issue < x.nchunks) {
    iccl_result_t r = issue_chunk(c, chn, x, x.next_issue);
    if (r == ICCL_ERR_IN_PROGRESS) break;  // relay ring full: the proxy issues the rest
    if (r) return r;
    x.next_issue++;
  }
  rzv_track(c, std::move(x), on_proxy);
  return ICCL_SUCCESS;
}

static iccl_result_t rzv_issue(iccl_comm* c, int kind, int peer, uint64_t k, uint64_t op_seq, const RzvSide* side,
                               cudaStream_t user_s) {
  Xfer x;
  iccl_result_t r = rzv_build(c, kind, peer, k, op_seq, false, side, &x);
  if (r) return r;
  if (user_s && c->event_ready && peer != c->rank) {
    x.own_ready = get_event(c);
    x.own_side = kind;
    ICCL_CHECK_CUDA(cudaEventRecord(x.own_ready, user_s));
  }
  return rzv_launch(c, std::move(x), false);
}

// ---------------------------------------------------------------- in-stream issue
// May the issuing side put the copy on its own user stream?  Only for a
// healthy pair that no fault script names (a stalled in-stream copy could not
// be migrated: its successors are the caller's own work) on the copy-engine
// transport — and, for a self pair, only when the other half's done wait
// cannot sit in front of the copy on that same stream (it does when it was
// posted outside this group on this stream).
static bool instream_ok(iccl_comm* c, int kind, int peer, const RzvSide* side, bool other_in_group,
                        cudaStream_t user_s) {
  if (!c->instream_ce) return false;
  if (peer == c->rank && !other_in_group && side[kind ^ 1].stream == (uint64_t)(uintptr_t)user_s) return false;
  return true;
}

// Is the transfer's pair armed for failover (a fault script names it, it
// runs on its backup path, or one of its paths is Down right now)?
static bool xfer_armed(iccl_comm* c, int kind, int peer) {
  const int src = kind == 0 ? c->rank : peer, dst = kind == 0 ? peer : c->rank;
  if (pair_armed(pair_of(c, src, dst))) return true;
  std::lock_guard<std::mutex> g(c->fault_mu);
  const Channel& chn = c->ch[2 * peer + kind];
  return chn.fault[0].down || chn.fault[1].down;
}

// The issuing side's wait for the other side's ready flag (hostFunc #1).
static void instream_ready_param(iccl_comm* c, const Xfer& x, int kind, std::vector<CUstreamBatchMemOpParams>& p) {
  CUstreamBatchMemOpParams w;
  memset(&w, 0, sizeof(w));
  w.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
  w.waitValue.address = kind == 0 ? (CUdeviceptr)&flags_of(c, x.dst_rank)->ready[x.r_ready_slot]
                                  : (CUdeviceptr)&flags_of(c, x.src_rank)->ready[x.s_slot];
  w.waitValue.value = kind == 0 ? x.r_ready_gen : x.s_gen;
  w.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  p.push_back(w);
}

// Both done flags (hostFunc #2): the other side's user stream waits on its
// own; this side's is for iccl_req_test / slot reuse.
static void instream_done_params(iccl_comm* c, const Xfer& x, std::vector<CUstreamBatchMemOpParams>& p) {
  CUstreamBatchMemOpParams w;
  memset(&w, 0, sizeof(w));
  w.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
  w.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  w.writeValue.address = (CUdeviceptr)&flags_of(c, x.dst_rank)->done[x.r_done_slot];
  w.writeValue.value = x.r_done_gen;
  p.push_back(w);
  w.writeValue.address = (CUdeviceptr)&flags_of(c, x.src_rank)->done[x.s_slot];
  w.writeValue.value = x.s_gen;
  p.push_back(w);
}

static iccl_result_t batch_memops(cudaStream_t s, std::vector<CUstreamBatchMemOpParams>& p);

// The issuer's waits on the other sides' ready flags (params of
// instream_ready_param): stream-memory waits, or K7 with ICCL_K7_READY.
static iccl_result_t ready_wait_ops(iccl_comm* c, cudaStream_t s, std::vector<CUstreamBatchMemOpParams>& p) {
  if (!c->k7_ready || p.empty()) return batch_memops(s, p);
  WaitList wl;
  memset(&wl, 0, sizeof(wl));
  wl.error = c->ll_error;
  for (size_t i = 0; i < p.size(); i++) {
    wl.addr[wl.n] = (const uint32_t*)(uintptr_t)p[i].waitValue.address;
    wl.gen[wl.n] = p[i].waitValue.value;
    if (++wl.n == kWaitMax || i + 1 == p.size()) {
      ICCL_CHECK_CUDA(launch_wait(wl, s));
      c->kernels_launched += 1;
      c->ctas_launched += 1;
      wl.n = 0;
    }
  }
  p.clear();
  return ICCL_SUCCESS;
}

static iccl_result_t batch_memops(cudaStream_t s, std::vector<CUstreamBatchMemOpParams>& p) {
  for (size_t i = 0; i < p.size(); i += 128) {
    unsigned n = (unsigned)std::min<size_t>(128, p.size() - i);
    ICCL_CHECK_CU(driver()->cuStreamBatchMemOp((CUstream)s, n, p.data() + i, 0));
  }
  p.clear();
  return ICCL_SUCCESS;
}

// The chunk copies of an in-stream transfer on user stream s — copy-engine
// copies, or K1 launches for the SM transport / small messages — each
// followed by its WC: an event after a copy (with the monitor on, the
// direction's monitor stream records a timing event behind every WC and an
// anchor at the op's start, so chunk times come from the device with nothing
// timed between the copies), or K1's own %globaltimer stamp (K4).
static iccl_result_t instream_copies(iccl_comm* c, Xfer& x, cudaStream_t s) {
  Channel& chn = c->ch[x.chan];
  const bool mon = c->monitor_enabled.load(std::memory_order_relaxed);
  const int eng = path_engine(c, chn, 0, x.bytes);
  cudaStream_t ms = c->streams[chn.mon_stream].s;
  cudaEvent_t last = nullptr;
  if (mon && eng == ENG_CE) {
    last = get_tevent(c);
    x.anchors.push_back(last);
    ICCL_CHECK_CUDA(cudaEventRecord(chn.bridge, s));
    ICCL_CHECK_CUDA(cudaStreamWaitEvent(ms, chn.bridge, 0));
    ICCL_CHECK_CUDA(cudaEventRecord(last, ms));
  }
  for (int k = 0; k < x.nchunks; k++) {
    const size_t off = (size_t)k * x.chunk, n = std::min(x.chunk, x.bytes - off);
    ChunkRec& rc = x.rec[k];
    rc.t1 = now_ns();
    rc.path = 0;
    rc.stream = -1;
    rc.stamp = -1;
    rc.done = false;
    c->copies_issued += 1;
    c->bytes_issued += n;
    if (eng == ENG_SM) {
      KernelStamp* st = nullptr;
      if (mon) {
        rc.stamp = c->next_stamp.fetch_add(1) % kStampSlots;
        st = &c->stamps[rc.stamp];
        memset((void*)st, 0, sizeof(KernelStamp));
      }
      int grid = 0;
      ICCL_CHECK_CUDA(launch_copy(x.src + off, x.dst + off, n, c->cfg.sm_cap, st, s, &grid));
      c->kernels_launched += 1;
      c->ctas_launched += grid;
      if (st) continue;  // the stamp is the WC
    } else {
      ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)(x.dst + off), (CUdeviceptr)(x.src + off), n,
                                                (CUstream)s));
    }
    if (!rc.ev) rc.ev = get_event(c);
    ICCL_CHECK_CUDA(cudaEventRecord(rc.ev, s));
    if (mon && eng == ENG_CE) {
      rc.tev = get_tevent(c);
      ICCL_CHECK_CUDA(cudaStreamWaitEvent(ms, rc.ev, 0));
      ICCL_CHECK_CUDA(cudaEventRecord(rc.tev, ms));
      rc.t1ev = last;
      last = rc.tev;
    }
  }
  x.next_issue = x.nchunks;
  x.instream = true;
  x.ustream = s;
  x.done_enqueued = true;
  return ICCL_SUCCESS;
}

// One in-stream transfer outside a group: ready wait, copies, done writes.
static iccl_result_t issue_instream(iccl_comm* c, Xfer&& x, int kind, cudaStream_t s) {
  std::vector<CUstreamBatchMemOpParams> p;
  instream_ready_param(c, x, kind, p);
  iccl_result_t r = ready_wait_ops(c, s, p);
  if (r) return r;
  r = instream_copies(c, x, s);
  if (r) return r;
  instream_done_params(c, x, p);
  r = batch_memops(s, p);
  if (r) return r;
  rzv_track(c, std::move(x), false);
  return ICCL_SUCCESS;
}

// ---------------------------------------------------------------- armed transfers
// A transfer on a pair armed for failover (a fault script names it) carries
// both attempts on the device from the start, so the failover needs no CUDA
// call at run time: a user thread sitting in a synchronous CUDA call (a
// pageable copy, .item()) behind the failing op blocks every other CUDA call
// of its process, and a proxy that still had to enqueue the backup would
// deadlock with it (probes/p2p_probe6, tests/test_gpu_failover.py).
//
//   primary, on the issuer's user stream U (in-stream) or the channel's copy
//   stream (then behind waits on both ready flags):
//     wait the other side's ready flag; per chunk k: [fault gate, if Down]
//     copy k, prog := k + 1; then p_fin := 1, go := 1;
//     wait ns (no-switch gate, open); both done flags; fin := 1
//   backup, on the channel's backup stream B:
//     K9a (one warp: waits for go in-kernel, decides), K9b (the copy grid,
//     empty unless switched); b_fin := 1 — no stream-memory wait on B: a
//     stream parked on one cost the GPU's other streams ~50 us per op
//
// No fault: the primary releases both sides itself (one memop wait on an open
// gate more than a plain in-stream transfer) and opens go with p_fin set, so
// K9 decides "exit" at once — one near-empty launch.  A stall (both ready
// flags set, no progress for delta): the watchdog thread sets ctl := probe
// and opens go; K9 stores a 16-byte CTS over the primary path unless that
// path's gate is closed.  A probe that does not land within delta means the
// path is dead — the primary is then parked on the same
// gate, in front of ns — so, with host stores only: ns := 0, resume :=
// completed (the receiver's breakpoint), ctl := switch, and the
// stale gate opens: the primary's flushed copies rewrite bytes K9 delivers
// (SPEC.md:285).  K9 copies chunks [resume, N) with a K4 stamp per chunk (the
// WCs); once every one landed and p_fin is set, the watchdog writes both done
// flags and reopens ns.
static iccl_result_t backup_stream(iccl_comm* c, Channel& chn, cudaStream_t* out) {
  if (chn.b_si < 0) {
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    StreamCtx sc;
    ICCL_CHECK_CUDA(cudaStreamCreateWithPriority(&sc.s, cudaStreamNonBlocking, hi));
    ICCL_CHECK_CUDA(cudaEventCreateWithFlags(&sc.ev, cudaEventDisableTiming));
    sc.engine = ENG_SM;
    c->streams.push_back(sc);
    chn.b_si = (int)c->streams.size() - 1;
  }
  *out = c->streams[chn.b_si].s;
  return ICCL_SUCCESS;
}

// Progress words of an armed primary are written from this stream, behind
// an untimed event recorded after each chunk: a stream-memory write between
// two copies would drain the copy engine (+4.6 us per chunk at 8 MiB chunks,
// profiles/r02/README.md §4), an event does not.
static iccl_result_t prog_stream(iccl_comm* c, Channel& chn, cudaStream_t* out) {
  if (chn.p_si < 0) {
    StreamCtx sc;
    ICCL_CHECK_CUDA(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    ICCL_CHECK_CUDA(cudaEventCreateWithFlags(&sc.ev, cudaEventDisableTiming));
    sc.engine = ENG_CE;
    c->streams.push_back(sc);
    chn.p_si = (int)c->streams.size() - 1;
  }
  *out = c->streams[chn.p_si].s;
  return ICCL_SUCCESS;
}

// The device-driven failover covers a transfer that starts on the primary
// with the SM backup; the relay backup and transfers issued on the backup
// path run the proxy-driven chunk pipeline (rzv_launch).
static bool armed_eligible(iccl_comm* c, const Xfer& x) {
  return x.path == 0 && c->cfg.backup_kind == ICCL_BACKUP_SM;
}

static CUstreamBatchMemOpParams wparam(uint32_t* addr, uint32_t v) {
  CUstreamBatchMemOpParams q;
  memset(&q, 0, sizeof(q));
  q.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
  q.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  q.writeValue.address = (CUdeviceptr)addr;
  q.writeValue.value = v;
  return q;
}

// instream: the primary goes on the issuer's user stream `us` (waiting on
// the other side's ready flag only); else on the channel's copy stream behind
// waits on both ready flags (the issuer's own op then carries markers).
static iccl_result_t armed_launch(iccl_comm* c, Xfer&& x, int kind, cudaStream_t us, bool instream) {
  Channel& chn = c->ch[x.chan];
  uint64_t t0 = now_ns();
  int slot = -1;
  while (slot < 0) {
    for (int i = 0; i < kArmedSlots && slot < 0; i++) {
      const uint32_t j = (c->armed_next + i) % kArmedSlots;
      if (!__atomic_load_n(&c->armed_used[j], __ATOMIC_ACQUIRE)) slot = (int)j;
    }
    ICCL_RETURN_IF(slot < 0 && now_ns() - t0 > 60ull * 1000000000ull, ICCL_ERR_TIMEOUT,
                   "more than 1024 armed transfers in flight for 60 s");
    if (slot < 0) sched_yield();
  }
  c->armed_next = (uint32_t)(slot + 1) % kArmedSlots;
  __atomic_store_n(&c->armed_used[slot], (uint8_t)1, __ATOMIC_RELEASE);
  ArmedWords* w = &c->armed_words[slot];
  memset((void*)w, 0, sizeof(*w));
  w->resume = (uint32_t)x.nchunks;
  w->ns = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  x.armed = true;
  x.aw = slot;
  const int eng = path_engine(c, chn, 0, x.bytes);
  cudaStream_t ps = instream ? us : c->streams[stream_for(c, chn, 0, ENG_CE, 0)].s;
  {
    std::lock_guard<std::mutex> g(c->fault_mu);  // a path already Down: the probe / the backup wait on its gate
    w->pgate = chn.fault[0].down ? (uint32_t)chn.fault[0].gate + 1 : 0;
    w->bgate = chn.fault[1].down ? (uint32_t)chn.fault[1].gate + 1 : 0;
  }
  iccl_result_t r;
  // backup attempt first (its controller waits for `go` in-kernel), then the
  // transfer goes to the watchdog, then the primary is enqueued from local
  // state: an enqueue behind a closed gate can block once the stream's
  // command queue is full, and the watchdog must already be watching then
  // (it opens the gate when it switches)
  if (c->armed_backup) {
    ICCL_RETURN_IF((((uintptr_t)x.src ^ (uintptr_t)x.dst) & 15) != 0, ICCL_ERR_INVALID_ARGUMENT,
                   "armed transfer between tensors of different alignment mod 16");
    cudaStream_t bs = nullptr;
    r = backup_stream(c, chn, &bs);
    if (r) return r;
    BackupOp b{};
    b.src = x.src;
    b.dst = x.dst;
    b.bytes = x.bytes;
    b.chunk = x.chunk;
    b.nchunks = (uint32_t)x.nchunks;
    b.ring = c->stamps;
    b.ring_slots = kStampSlots;
    b.w = w;
    b.gates = (const uint32_t*)c->gate_words;
    // the CTS probe (16 B) crosses the primary path in its direction: into the
    // peer's scratch (push) or out of it (pull)
    b.probe_src = chn.dir == 0 ? c->scratch : chn.peer_scratch;
    b.probe_dst = chn.dir == 0 ? chn.peer_scratch : c->scratch + 2048 + 16 * chn.peer;
    b.error = c->ll_error;
    // K9a -> K9b decision word: one per armed slot in GPU memory (after the K6 go words)
    b.dec_dev = c->ll_counters + 2 * kLLCounters + slot;
    b.seq = (c->armed_seq++) & 0x3fffffffu;
    b.stamp_base = (uint32_t)(c->next_stamp.fetch_add(x.nchunks) % kStampSlots);
    x.bstamp.assign(x.nchunks, -1);
    for (int k = 0; k < x.nchunks; k++) {
      x.bstamp[k] = (int)((b.stamp_base + k) % kStampSlots);
      memset((void*)&c->stamps[x.bstamp[k]], 0, sizeof(KernelStamp));
    }
    int grid = 0;
    if (c->k9_mode == 0) ICCL_CHECK_CUDA(launch_backup(b, c->cfg.sm_cap, bs, &grid));
    if (c->k9_mode == 1) ICCL_CHECK_CUDA(launch_backup(b, 0, bs, &grid));  // K9a only
    if (c->k9_mode == 3) ICCL_CHECK_CUDA(launch_backup(b, -1, bs, &grid));  // K9b without shared memory
    if (c->k9_mode == 4) ICCL_CHECK_CUDA(launch_backup(b, -2, bs, &grid));  // one-CTA K9b
    c->kernels_launched += 1;
    c->ctas_launched += grid;
    r = memop_write(bs, &w->b_fin, 1);
    if (r) return r;
  } else {  // attribution runs only: no failover possible
    x.bstamp.assign(x.nchunks, -1);
    __atomic_store_n(&w->b_fin, 1u, __ATOMIC_SEQ_CST);
  }
  // everything the primary's enqueue needs, copied out of x before handing it over
  cudaStream_t pstr = nullptr;
  if (c->prog_events) {
    r = prog_stream(c, chn, &pstr);
    if (r) return r;
    for (int k = 0; k < x.nchunks; k++)
      if (!x.rec[k].ev) x.rec[k].ev = get_event(c);  // returned to the pool when the watchdog retires x
  }
  std::vector<cudaEvent_t> evs;
  for (const ChunkRec& rc : x.rec) evs.push_back(rc.ev);
  std::vector<CUstreamBatchMemOpParams> p, fin;
  if (instream) {
    // this side's ready flag too (the watchdog tells an upstream stall of
    // either side by the two flags), then the wait on the other side's
    p.push_back(kind == 0 ? wparam(&flags_of(c, x.src_rank)->ready[x.s_slot], x.s_gen)
                          : wparam(&flags_of(c, x.dst_rank)->ready[x.r_ready_slot], x.r_ready_gen));
    instream_ready_param(c, x, kind, p);
  }
  instream_done_params(c, x, fin);
  fin.push_back(wparam(&w->fin, 1));
  const int nchunks = x.nchunks, fault_ops_index = x.fault_ops_index;
  const size_t chunk = x.chunk, bytes = x.bytes;
  const char* src = x.src;
  char* dst = x.dst;
  Xfer ready_x;  // wait_both_ready reads the flag slots only
  ready_x.src_rank = x.src_rank;
  ready_x.dst_rank = x.dst_rank;
  ready_x.s_slot = x.s_slot;
  ready_x.s_gen = x.s_gen;
  ready_x.r_ready_slot = x.r_ready_slot;
  ready_x.r_ready_gen = x.r_ready_gen;
  ready_x.own_ready = x.own_ready;
  ready_x.own_side = x.own_side;
  x.next_issue = x.nchunks;
  x.instream = instream;
  x.ustream = instream ? us : nullptr;
  x.done_enqueued = true;
  x.t_obs = now_ns();
  publish(c, x);
  c->pending_xfers.fetch_add(1);
  {
    std::lock_guard<std::mutex> g(c->amu);
    c->ahandoff.push_back(std::move(x));
  }
  // primary attempt
  r = instream ? batch_memops(ps, p) : wait_both_ready(c, ps, ready_x);
  if (r) return r;
  // every chunk of this transfer behind a Down path waits on the gate of the
  // Down it first met — a switch opens exactly that one (and re-arms the path
  // with a fresh gate for later transfers), even while this loop still runs
  int my_gate = -1;
  for (int k = 0; k < nchunks; k++) {
    const size_t off = (size_t)k * chunk, n = std::min(chunk, bytes - off);
    {
      std::lock_guard<std::mutex> g(c->fault_mu);
      if (fault_ops_index >= 0) fire_chunk_faults(c, chn, fault_ops_index, k, 0);
      if (chn.fault[0].down && my_gate < 0) {
        my_gate = chn.fault[0].gate;
        __atomic_store_n(&w->pgate, (uint32_t)my_gate + 1, __ATOMIC_SEQ_CST);  // before the first wait on it
      }
      if (my_gate >= 0) {
        r = memop_wait(ps, &c->gate_words[my_gate], 1);
        if (r) return r;
      }
    }
    if (eng == ENG_SM) {
      int grid = 0;
      ICCL_CHECK_CUDA(launch_copy(src + off, dst + off, n, c->cfg.sm_cap, nullptr, ps, &grid));
      c->kernels_launched += 1;
      c->ctas_launched += grid;
    } else {
      ICCL_CHECK_CU(driver()->cuMemcpyDtoDAsync((CUdeviceptr)(dst + off), (CUdeviceptr)(src + off), n, (CUstream)ps));
    }
    c->copies_issued += 1;
    c->bytes_issued += n;
    if (c->prog_events) {
      ICCL_CHECK_CUDA(cudaEventRecord(evs[k], ps));
      ICCL_CHECK_CUDA(cudaStreamWaitEvent(pstr, evs[k], 0));
      r = memop_write(pstr, &w->prog, (uint32_t)(k + 1));
    } else {
      r = memop_write(ps, &w->prog, (uint32_t)(k + 1));
    }
    if (r) return r;
  }
  p.clear();
  p.push_back(wparam(&w->p_fin, 1));
  p.push_back(wparam(&w->go, 1));
  r = batch_memops(ps, p);
  if (r) return r;
  r = memop_wait(ps, &w->ns, 1);
  if (r) return r;
  return batch_memops(ps, fin);
}

// ---------------------------------------------------------------- watchdog thread
static void armed_record(iccl_comm* c, const Channel& chn, const Xfer& x, int k, uint64_t t1, uint64_t t2) {
  iccl_mon_rec_t m{};
  m.t1_ns = t1;
  m.t2_ns = t2;
  m.bytes = std::min(x.chunk, x.bytes - (size_t)k * x.chunk);
  m.peer = chn.peer;
  m.path = x.switched && k >= (int)c->armed_words[x.aw].resume ? ICCL_PATH_BACKUP : ICCL_PATH_PRIMARY;
  m.chunk = k;
  m.dir = chn.dir;
  m.op_seq = x.op_seq;
  std::lock_guard<std::mutex> g(c->mon_mu);
  c->mon.push_back(m);
  if (c->mon.size() > (1u << 20)) c->mon.pop_front();
}

// switch_qp of an armed transfer whose primary is parked on a dead path
// (SPEC.md:255-263): host stores only.
static void armed_switch(iccl_comm* c, Channel& chn, Xfer& x) {
  ArmedWords* w = &c->armed_words[x.aw];
  const uint64_t t = now_ns();
  uint64_t detect = 0;
  int stale = -1;
  {
    std::lock_guard<std::mutex> g(c->fault_mu);
    if (chn.fault[0].down) {
      detect = t - chn.fault[0].down_at;
      stale = chn.fault[0].gate;
      chn.fault[0].gate = alloc_gate(c);  // later work on the still-Down path waits on a fresh epoch
    }
  }
  __atomic_store_n(&w->ns, 0u, __ATOMIC_SEQ_CST);  // the primary (parked on the gate) must not release the op
  __atomic_store_n(&w->resume, (uint32_t)x.completed, __ATOMIC_SEQ_CST);  // breakpoint = receiver done
  __atomic_store_n(&w->ctl, (uint32_t)kCtlSwitch, __ATOMIC_SEQ_CST);      // before the stale gate opens
  __atomic_store_n(&w->go, 1u, __ATOMIC_SEQ_CST);
  if (stale >= 0) release_gate(c, stale);  // the primary drains: its flushed copies rewrite delivered bytes
  x.switched = true;
  x.path = 1;
  x.switches++;
  x.last_progress = t;
  publish(c, x);
  PairState& ps = pair_of(c, chn.src, chn.dst);
  if (ps.active_path.exchange(1) != 1) {
    ps.switches.fetch_add(1);
    route_update(ps);
  }
  chn.armed_failed_over = true;
  chn.armed_last_probe = t;
  ICCL_TRACE("armed switch pair %d->%d to backup at chunk %d", chn.src, chn.dst, x.completed);
  push_switch_event(c, chn.peer, 1, x.completed, 1, detect);
}

// One watchdog pass over a channel's armed transfers.
static bool armed_progress(iccl_comm* c, Channel& chn) {
  bool busy = false;
  const uint64_t tnow = now_ns();
  const bool mon = c->monitor_enabled.load(std::memory_order_relaxed);
  for (Xfer& x : chn.armed) {
    ArmedWords* w = &c->armed_words[x.aw];
    if (!x.switched) {
      // primary chunks: t2 = when this (spinning) thread saw the progress
      // word move; chunks seen landing in one pass share the interval evenly
      const int p = std::min((int)__atomic_load_n(&w->prog, __ATOMIC_ACQUIRE), x.nchunks);
      const int m = p - x.completed;
      for (int j = 0; j < m; j++) {
        const uint64_t a = x.t_obs + (tnow - x.t_obs) * j / m, b = x.t_obs + (tnow - x.t_obs) * (j + 1) / m;
        if (mon) armed_record(c, chn, x, x.completed, a, b);
        x.completed++;
      }
      if (m > 0) {
        ICCL_TRACE("armed pair %d->%d: primary chunks %d..%d landed (+%.1f us since the last observation)", chn.src,
                   chn.dst, x.completed - m, x.completed - 1, (tnow - x.t_obs) * 1e-3);
        x.t_obs = tnow;
        x.last_progress = tnow;
        busy = true;
      }
    } else if (__atomic_load_n(&w->dec, __ATOMIC_ACQUIRE) == kDecExit) {
      // K9 saw the primary finish before the switch reached it: the primary
      // delivered every chunk (its flushed copies included) — complete the op
      if (__atomic_load_n(&w->p_fin, __ATOMIC_ACQUIRE) && __atomic_load_n(&w->ns, __ATOMIC_ACQUIRE) == 0) {
        x.completed = x.nchunks;
        __atomic_store_n(&flags_of(c, x.dst_rank)->done[x.r_done_slot], x.r_done_gen, __ATOMIC_SEQ_CST);
        __atomic_store_n(&flags_of(c, x.src_rank)->done[x.s_slot], x.s_gen, __ATOMIC_SEQ_CST);
        __atomic_store_n(&w->ns, 1u, __ATOMIC_SEQ_CST);
        busy = true;
      }
    } else {
      while (x.completed < x.nchunks) {
        KernelStamp* st = &c->stamps[x.bstamp[x.completed]];
        const unsigned long long t2 = __atomic_load_n(&st->t2, __ATOMIC_ACQUIRE);
        if (!t2) break;
        if (mon) {
          const unsigned long long t1 = __atomic_load_n(&st->t1, __ATOMIC_ACQUIRE);
          armed_record(c, chn, x, x.completed, (uint64_t)((int64_t)(t1 ? t1 : t2) + c->gtimer_offset),
                       (uint64_t)((int64_t)t2 + c->gtimer_offset));
        }
        x.completed++;
        x.last_progress = tnow;
        busy = true;
      }
      if (x.completed == x.nchunks && __atomic_load_n(&w->ns, __ATOMIC_ACQUIRE) == 0 &&
          __atomic_load_n(&w->p_fin, __ATOMIC_ACQUIRE)) {
        // every backup chunk landed and the primary drained: complete the op
        __atomic_store_n(&flags_of(c, x.dst_rank)->done[x.r_done_slot], x.r_done_gen, __ATOMIC_SEQ_CST);
        __atomic_store_n(&flags_of(c, x.src_rank)->done[x.s_slot], x.s_gen, __ATOMIC_SEQ_CST);
        __atomic_store_n(&w->ns, 1u, __ATOMIC_SEQ_CST);  // lets the parked primary pass (its done writes repeat)
        busy = true;
      }
    }
    publish(c, x);
  }
  // retire: the primary passed its done writes and the backup drained
  while (!chn.armed.empty()) {
    Xfer& x = chn.armed.front();
    ArmedWords* w = &c->armed_words[x.aw];
    if (!__atomic_load_n(&w->fin, __ATOMIC_ACQUIRE) || !__atomic_load_n(&w->b_fin, __ATOMIC_ACQUIRE)) break;
    if (!x.switched) {  // the last primary chunks may land between two passes
      const int m = x.nchunks - x.completed;
      for (int j = 0; j < m; j++) {
        const uint64_t a = x.t_obs + (tnow - x.t_obs) * j / m, b = x.t_obs + (tnow - x.t_obs) * (j + 1) / m;
        if (mon) armed_record(c, chn, x, x.completed, a, b);
        x.completed++;
      }
    }
    x.completed = x.nchunks;
    publish(c, x);
    put_events(c, x);  // the progress events (pool bookkeeping only, no CUDA call)
    __atomic_store_n(&c->armed_used[x.aw], (uint8_t)0, __ATOMIC_RELEASE);
    chn.armed.pop_front();
    c->pending_xfers.fetch_sub(1);
    busy = true;
  }
  // watchdog + CTS probe (check_receiver_timeout) on the front
  if (!chn.armed.empty()) {
    Xfer& x = chn.armed.front();
    ArmedWords* w = &c->armed_words[x.aw];
    const bool elig = cyc_geq(flags_of(c, x.src_rank)->ready[x.s_slot], x.s_gen) &&
                      cyc_geq(flags_of(c, x.dst_rank)->ready[x.r_ready_slot], x.r_ready_gen);
    if (!elig) {
      if (x.eligible) ICCL_TRACE("armed pair %d->%d: ready flags not both set", chn.src, chn.dst);
      x.last_progress = tnow;  // innocent stall upstream: a side's stream has not reached the op
      x.t_obs = tnow;
    } else if (!x.eligible) {
      ICCL_TRACE("armed pair %d->%d: both ready flags set", chn.src, chn.dst);
      x.eligible = true;
      x.last_progress = tnow;
      x.t_obs = tnow;
    }
    const uint64_t delta = c->cfg.delta_us * 1000ull;
    if (elig && x.completed < x.nchunks && tnow - x.last_progress > delta) {
      if (!x.switched) {
        if (!x.probing && !x.probe_ok) {
          __atomic_store_n(&w->ctl, (uint32_t)kCtlProbe, __ATOMIC_SEQ_CST);
          __atomic_store_n(&w->go, 1u, __ATOMIC_SEQ_CST);
          x.probing = true;
          x.probe_t = tnow;
        } else if (x.probing && __atomic_load_n(&w->probe_done, __ATOMIC_ACQUIRE)) {
          x.probing = false;  // CTS ok: an innocent stall
          x.probe_ok = true;
          x.last_progress = tnow;
        } else if (x.probing && tnow - x.probe_t > delta) {
          x.probing = false;
          armed_switch(c, chn, x);  // CTS lost: the path is dead
          busy = true;
        }
      } else {
        bool backup_down;
        {
          std::lock_guard<std::mutex> g(c->fault_mu);
          backup_down = chn.fault[1].down;
        }
        if (backup_down)  // both paths dead
          set_async(c, ICCL_ERR_CONNECTION_FAILED, "both paths of pair " + std::to_string(chn.src) + "->" +
                                                       std::to_string(chn.dst) + " are down");
      }
    }
  }
  // monitor_failed_link: once the primary is healthy again,
  // later transfers use it (in-flight ones finish on the backup)
  if (chn.armed_failed_over && tnow - chn.armed_last_probe >= c->cfg.probe_period_us * 1000ull) {
    chn.armed_last_probe = tnow;
    bool up;
    {
      std::lock_guard<std::mutex> g(c->fault_mu);
      up = !chn.fault[0].down;
    }
    PairState& ps = pair_of(c, chn.src, chn.dst);
    if (up) {
      chn.armed_failed_over = false;
      if (ps.active_path.exchange(0) != 0) {
        ps.switches.fetch_add(1);
        route_update(ps);
      }
      push_switch_event(c, chn.peer, 0, -1, 2, 0);
    }
  }
  return busy;
}

static void watch_loop(iccl_comm* c) {
  std::vector<Xfer> batch;
  while (!c->stop.load(std::memory_order_relaxed)) {
    {
      std::lock_guard<std::mutex> g(c->amu);
      batch.swap(c->ahandoff);
    }
    for (Xfer& x : batch) c->ch[x.chan].armed.push_back(std::move(x));
    batch.clear();
    // time-triggered faults fire here too: the proxy thread may sit in a CUDA
    // call that a user thread's synchronous call behind the faulted op blocks
    // (host stores only; fire_time_faults is idempotent under fault_mu);
    fire_time_faults(c);
    bool any = false, busy = false;
    for (Channel& chn : c->ch) {
      if (chn.armed.empty() && !chn.armed_failed_over) continue;
      any = true;
      busy |= armed_progress(c, chn);
    }
    // spin while armed transfers are in flight (the monitor's host-observed
    // t2 for primary chunks is as fine as this loop), nap otherwise
    if (!any) std::this_thread::sleep_for(std::chrono::microseconds(50));
    else if (!busy) sched_yield();
  }
}

static size_t ll_slot_offset(int src, uint32_t seq) {
  return ((size_t)src * kLLSlots + (seq - 1) % kLLSlots) * kLLLines * 8;
}
static size_t ll_credit_offset(int nranks, int peer) {
  return (size_t)nranks * kLLSlots * kLLLines * 8 + (size_t)peer * 64;
}
// Device flags of direct-class (K6) ops, after the credits in the LL region:
// ready[kSlots] then done[kSlots], gen-tagged like the host-mapped flags.  The
// owner's user stream writes its ready word locally and K6 on the peer polls
// it over NVLink; K6 stores the done word into the waiting side's GPU memory
// and K7 there polls local memory instead of the host-mapped flag.
static size_t dflag_ready_offset(int nranks, uint32_t slot) {
  return ll_credit_offset(nranks, nranks) + (size_t)slot * 4;
}
static size_t dflag_done_offset(int nranks, uint32_t slot) {
  return ll_credit_offset(nranks, nranks) + ((size_t)kSlots + slot) * 4;
}

// Monitor on: a K4 stamp slot for a K5 send / K6 op, whose record the proxy
// emits once the kernel's t2 lands (drain_kstamps).
static KernelStamp* alloc_kstamp(iccl_comm* c, OpDesc& op) {
  if (!c->monitor_enabled.load(std::memory_order_relaxed)) return nullptr;
  op.kstamp = c->next_stamp.fetch_add(1) % kStampSlots;
  KernelStamp* st = &c->stamps[op.kstamp];
  memset((void*)st, 0, sizeof(KernelStamp));
  return st;
}

static void push_krec(iccl_comm* c, const OpDesc& op, int dir) {
  if (op.kstamp < 0) return;
  std::lock_guard<std::mutex> g(c->mon_mu);
  c->krecs.push_back(iccl_comm::KRec{op.kstamp, op.bytes, op.op_seq, op.peer, dir});
  c->krecs_pending.fetch_add(1);
}

// Rendezvous of the k-th op of an ordered pair (SPEC.md:194's RTS / CTS): post
// my half (IPC handle, offset, op slot); the side that arrives second has
// both halves and issues the transfer right here, from its own API call — a
// push by the sender or a pull by the receiver.
//
// Why the API call and not the proxy: while any thread of a process sits in a
// synchronous CUDA call on a stream parked behind one of our ops (a pageable
// cudaMemcpy, .cpu()), every other CUDA call of that process blocks — memcpy,
// kernel launch, stream memop, event record alike (probes/p2p_probe6.cu).  A
// proxy that still had to enqueue the copy deadlocks with such a user; with
// all device work enqueued before the API returns nothing can.
//
// What the issuer enqueues: on a healthy pair no fault script names, the
// copy-engine copies go on its own user stream (in-stream: one wait on the
// other side's ready flag, the copies, one write of both done flags — the
// stream orders the rest); otherwise on the channel's side streams behind
// waits on both ready flags, where gates, the watchdog, switch_qp and the
// monitor's re-issue apply.  Mid-size ops take K6 on the user stream unless
// the pair is armed.
//
// Why senders try to come second: a copy-engine pull runs ~5% slower than a
// push (probes/p2p_probe6.cu), and the paper's transfers are sender-driven.
// A send therefore first waits up to `wait_us` for the receiver's half to be
// posted (receivers usually post early; inside a group every recv is posted
// before any send), and only then posts its own.
//
// The remote pushes of a group go to one stream, in call order: a GPU's copy
// engine runs its peer copies one after another whatever stream they are on,
// but in an order of its own — with one stream per peer, three senders of a
// 4-rank alltoallv ended up pushing into the same receiver at once (incast,
// each at half rate: MoE records, profiles/r01/README.md).  On one stream the
// rotated order of iccl_alltoallv (step k: rank i -> i + k) holds, so at each
// step every receiver has one sender.
static iccl_result_t rzv_post(iccl_comm* c, OpDesc& op, uint64_t wait_us, bool group, cudaStream_t user_s) {
  const int peer = op.peer, kind = op.kind;
  const uint64_t k = kind == 0 ? c->pair_sends[peer]++ : c->pair_recvs[peer]++;
  RzvEntry& e = rzv_entry(c, kind, peer, k);
  const uint64_t g = k / kRzvDepth;
  uint64_t t0 = now_ns();
  while (!rzv_free(e, k)) {
    if (c->async_err.load() != ICCL_SUCCESS) return (iccl_result_t)c->async_err.load();
    if (c->hdr->abort.load()) return ICCL_ERR_ABORTED;
    if (now_ns() - t0 > 60ull * 1000000000ull) {
      set_last_error("more than 1024 unmatched ops on a pair for 60 s");
      return ICCL_ERR_TIMEOUT;
    }
    sched_yield();
  }
  if (kind == 0 && peer != c->rank && wait_us > 0) {
    const uint64_t t_wait = now_ns(), deadline = t_wait + wait_us * 1000ull;
    while (e.arrivals.load(std::memory_order_acquire) < 2 * g + 1 && now_ns() < deadline) sched_yield();
    const bool timed_out = e.arrivals.load(std::memory_order_acquire) < 2 * g + 1;
    if (timed_out) c->cts_timeouts += 1;
    ICCL_TRACE("send %d->%d #%llu waited %.1f us for the CTS%s", c->rank, peer, (unsigned long long)k,
               (now_ns() - t_wait) * 1e-3, timed_out ? " (timed out)" : "");
  }
  RzvSide& mine = e.side[kind];
  mine.bytes = op.bytes;
  mine.slot = op.slot;
  mine.gen = op.gen;
  mine.direct_ptr = (uint64_t)(uintptr_t)op.src;
  mine.stream = (uint64_t)(uintptr_t)user_s;
  mine.buffer_id = 0;
  mine.base_offset = 0;
  if (peer != c->rank) {
    iccl_result_t r = export_buffer(c, op.src, &mine);
    if (r) return r;
    announce_buffer(c, peer, mine);
  }
  RzvSide side[2];
  if (!rzv_arrive(e, k, side)) {
    ICCL_TRACE("%s %d->%d #%llu posted first", kind == 0 ? "send" : "recv", kind == 0 ? c->rank : peer,
               kind == 0 ? peer : c->rank, (unsigned long long)k);
    return ICCL_SUCCESS;  // first: the peer issues
  }
  if (kind == 1 && peer != c->rank) c->pulls_issued += 1;
  const int src = kind == 0 ? c->rank : peer, dst = kind == 0 ? peer : c->rank;
  if (op.direct && !pair_armed(pair_of(c, src, dst))) {
    const RzvSide& other = side[kind ^ 1];
    // K6's TMA ring needs both tensors at the same alignment mod 16 (an IPC
    // mapping is page-aligned, so the peer's offset decides); else the copy
    // engine path below takes it
    if (((uintptr_t)op.src & 15) == (other.base_offset & 15) && side[0].bytes == side[1].bytes) {
      char* mapped = nullptr;
      Channel& chn = c->ch[2 * peer + kind];
      iccl_result_t r = open_peer_buffer(c, chn, other, &mapped);
      if (r) return r;
      DirectOp& d = op.dop;
      d.src = kind == 0 ? op.src : mapped;
      d.dst = kind == 0 ? mapped : (char*)op.src;
      d.peer_ready = &flags_of(c, peer)->ready[other.slot];
      d.peer_ready_gen = other.gen;
      d.peer_done = &flags_of(c, peer)->done[other.slot];
      d.peer_done_gen = other.gen;
      d.my_done = &flags_of(c, c->rank)->done[op.slot];
      d.my_done_gen = op.gen;
      d.peer_done_dev = nullptr;
      d.vec = op.bytes <= c->k6_vec_bytes;
      if (c->device_flags) {
        d.peer_ready = (const uint32_t*)(c->peer_ll[peer] + dflag_ready_offset(c->nranks, other.slot));
        d.peer_done_dev = (uint32_t*)(c->peer_ll[peer] + dflag_done_offset(c->nranks, other.slot));
      }
      d.counter = c->ll_counters + (c->ll_ctr_next++ % kLLCounters);
      d.go = c->ll_counters + kLLCounters + (op.slot % kLLCounters);
      d.error = c->ll_error;
      d.stamp = alloc_kstamp(c, op);
      op.issued_direct = true;
      ICCL_TRACE("direct %s pair %d->%d #%llu, %zu B", kind == 0 ? "push" : "pull", src, dst,
                 (unsigned long long)k, op.bytes);
      return ICCL_SUCCESS;
    }
  }
  if (group) {
    // a group's transfers are launched together once the whole group has met
    // its peers (iccl_group_end): all ready waits first, then the copies
    iccl_comm::GroupJob j{kind, peer, k, op.op_seq, {side[0], side[1]}, user_s};
    c->group_jobs.push_back(j);
    return ICCL_SUCCESS;
  }
  // the issue decision: armed pairs take the device-driven failover pipeline,
  // healthy ones the plain in-stream copy; the side-stream pipeline covers the
  // rest (a self pair whose other half waits on this very stream, the relay
  // backup, transfers issued on the backup path)
  const bool stream_ok = instream_ok(c, kind, peer, side, false, user_s);
  if (xfer_armed(c, kind, peer)) {
    Xfer x;
    iccl_result_t r = rzv_build(c, kind, peer, k, op.op_seq, false, side, &x);
    if (r) return r;
    if (armed_eligible(c, x)) {
      op.issued_instream = stream_ok;
      return armed_launch(c, std::move(x), kind, user_s, stream_ok);
    }
    return rzv_launch(c, std::move(x), false);
  }
  if (stream_ok) {
    Xfer x;
    iccl_result_t r = rzv_build(c, kind, peer, k, op.op_seq, false, side, &x);
    if (r) return r;
    op.issued_instream = true;
    return issue_instream(c, std::move(x), kind, user_s);
  }
  return rzv_issue(c, kind, peer, k, op.op_seq, side, user_s);
}

// ---------------------------------------------------------------- fused dispatch (K8)
// A send of a fused dispatch: its rows do not exist in any tensor yet (K8
// produces them straight into the receiver's buffer), so it waits for the
// receiver's half (CTS) unconditionally and always arrives second — the
// receiver never issues.  The mapped receive segment and the two flags go
// into the pending DispatchOp.  Every rank posts its dispatch receives
// before any dispatch send waits (group order), so the wait cannot deadlock.
static iccl_result_t fused_rendezvous(iccl_comm* c, OpDesc& op) {
  const int peer = op.peer;
  const uint64_t k = c->pair_sends[peer]++;
  RzvEntry& e = rzv_entry(c, 0, peer, k);
  const uint64_t g = k / kRzvDepth;
  const uint64_t t0 = now_ns();
  while (!rzv_free(e, k) || e.arrivals.load(std::memory_order_acquire) < 2 * g + 1) {
    if (c->async_err.load() != ICCL_SUCCESS) return (iccl_result_t)c->async_err.load();
    if (c->hdr->abort.load()) return ICCL_ERR_ABORTED;
    if (now_ns() - t0 > 60ull * 1000000000ull) {
      set_last_error("fused dispatch: rank " + std::to_string(peer) + " posted no matching receive within 60 s");
      return ICCL_ERR_TIMEOUT;
    }
    sched_yield();
  }
  RzvSide& mine = e.side[0];
  mine.bytes = op.bytes;
  mine.slot = op.slot;
  mine.gen = op.gen;
  mine.direct_ptr = 0;
  mine.stream = (uint64_t)(uintptr_t)c->dispatch_stream;
  mine.buffer_id = 0;
  mine.base_offset = 0;
  RzvSide side[2];
  ICCL_RETURN_IF(!rzv_arrive(e, k, side), ICCL_ERR_SYSTEM, "fused dispatch send arrived first");
  const RzvSide& rcv = side[1];
  if (rcv.bytes != op.bytes) {
    __atomic_store_n(&flags_of(c, c->rank)->done[op.slot], op.gen, __ATOMIC_SEQ_CST);
    __atomic_store_n(&flags_of(c, peer)->done[rcv.slot], rcv.gen, __ATOMIC_SEQ_CST);
    std::string msg = "dispatch of " + std::to_string(op.bytes) + " B from rank " + std::to_string(c->rank) +
                      " matched a receive of " + std::to_string(rcv.bytes) + " B on rank " + std::to_string(peer);
    set_async(c, ICCL_ERR_SIZE_MISMATCH, msg);
    set_last_error(msg);
    return ICCL_ERR_SIZE_MISMATCH;
  }
  char* mapped = nullptr;
  iccl_result_t r = open_peer_buffer(c, c->ch[2 * peer], rcv, &mapped);
  if (r) return r;
  FusedDest& d = c->dispatch_op.d[peer];
  d.seg = mapped;
  d.ready = &flags_of(c, peer)->ready[rcv.slot];
  d.ready_gen = rcv.gen;
  d.done = &flags_of(c, peer)->done[rcv.slot];
  d.done_gen = rcv.gen;
  d.my_done = &flags_of(c, c->rank)->done[op.slot];
  d.my_done_gen = op.gen;
  ICCL_TRACE("fused dispatch push %d->%d #%llu, %zu B", c->rank, peer, (unsigned long long)k, op.bytes);
  return ICCL_SUCCESS;
}

// K8 for the pending dispatch on stream s (its remote sends: `sends`).
static iccl_result_t launch_fused_dispatch(iccl_comm* c, cudaStream_t s, const std::vector<OpDesc>& sends) {
  DispatchOp& op = c->dispatch_op;
  OpDesc rec{};
  op.stamp = alloc_kstamp(c, rec);
  int grid = 0;
  ICCL_CHECK_CUDA(launch_dispatch(op, c->dispatch_ctas, s, &grid));
  c->kernels_launched += 1;
  c->ctas_launched += grid;
  c->dispatch_fused = false;  // launched
  for (const OpDesc& o : sends) {
    if (!o.fused) continue;
    c->copies_issued += 1;
    c->bytes_issued += o.bytes;
    OpDesc m = o;
    m.kstamp = rec.kstamp;
    push_krec(c, m, 0);
  }
  return ICCL_SUCCESS;
}

// A recv of a fused combine: it waits for the sender's half (RTS: the
// expert rank's tensor segment) unconditionally, so it always arrives second
// and claims the transfer — K10 pulls the rows; the sender never issues.
static iccl_result_t pull_rendezvous(iccl_comm* c, OpDesc& op) {
  const int peer = op.peer;
  const uint64_t k = c->pair_recvs[peer]++;
  RzvEntry& e = rzv_entry(c, 1, peer, k);
  const uint64_t g = k / kRzvDepth;
  const uint64_t t0 = now_ns();
  while (!rzv_free(e, k) || e.arrivals.load(std::memory_order_acquire) < 2 * g + 1) {
    if (c->async_err.load() != ICCL_SUCCESS) return (iccl_result_t)c->async_err.load();
    if (c->hdr->abort.load()) return ICCL_ERR_ABORTED;
    if (now_ns() - t0 > 60ull * 1000000000ull) {
      set_last_error("fused combine: rank " + std::to_string(peer) + " posted no matching send within 60 s");
      return ICCL_ERR_TIMEOUT;
    }
    sched_yield();
  }
  RzvSide& mine = e.side[1];
  mine.bytes = op.bytes;
  mine.slot = op.slot;
  mine.gen = op.gen;
  mine.direct_ptr = (uint64_t)(uintptr_t)op.src;
  mine.stream = (uint64_t)(uintptr_t)c->combine_stream;
  mine.buffer_id = 0;
  mine.base_offset = 0;
  RzvSide side[2];
  ICCL_RETURN_IF(!rzv_arrive(e, k, side), ICCL_ERR_SYSTEM, "fused combine recv arrived first");
  const RzvSide& snd = side[0];
  if (snd.bytes != op.bytes) {
    __atomic_store_n(&flags_of(c, c->rank)->done[op.slot], op.gen, __ATOMIC_SEQ_CST);
    __atomic_store_n(&flags_of(c, peer)->done[snd.slot], snd.gen, __ATOMIC_SEQ_CST);
    std::string msg = "combine of " + std::to_string(snd.bytes) + " B from rank " + std::to_string(peer) +
                      " matched a receive of " + std::to_string(op.bytes) + " B on rank " + std::to_string(c->rank);
    set_async(c, ICCL_ERR_SIZE_MISMATCH, msg);
    set_last_error(msg);
    return ICCL_ERR_SIZE_MISMATCH;
  }
  char* mapped = nullptr;
  iccl_result_t r = open_peer_buffer(c, c->ch[2 * peer + 1], snd, &mapped);
  if (r) return r;
  FusedSrc& d = c->combine_op.d[peer];
  d.seg = mapped;
  d.ready = &flags_of(c, peer)->ready[snd.slot];
  d.ready_gen = snd.gen;
  d.done = &flags_of(c, peer)->done[snd.slot];
  d.done_gen = snd.gen;
  d.my_done = &flags_of(c, c->rank)->done[op.slot];
  d.my_done_gen = op.gen;
  c->pulls_issued += 1;
  ICCL_TRACE("fused combine pull %d->%d #%llu, %zu B", peer, c->rank, (unsigned long long)k, op.bytes);
  return ICCL_SUCCESS;
}

// K10 for the pending combine on stream s (its pulling recvs: `recvs`).
static iccl_result_t launch_fused_combine(iccl_comm* c, cudaStream_t s, const std::vector<OpDesc>& recvs) {
  CombineOp& op = c->combine_op;
  OpDesc rec{};
  op.stamp = alloc_kstamp(c, rec);
  int grid = 0;
  ICCL_CHECK_CUDA(launch_combine(op, c->dispatch_ctas, s, &grid));
  c->kernels_launched += 1;
  c->ctas_launched += grid;
  c->combine_fused = false;  // launched
  for (const OpDesc& o : recvs) {
    if (!o.pull) continue;
    c->copies_issued += 1;
    c->bytes_issued += o.bytes;
    OpDesc m = o;
    m.kstamp = rec.kstamp;
    push_krec(c, m, 1);
  }
  return ICCL_SUCCESS;
}

// K6 for every op of `ops` this side issues directly, on stream s.
static iccl_result_t launch_direct_ops(iccl_comm* c, cudaStream_t s, const std::vector<OpDesc>& ops) {
  for (const OpDesc& op : ops) {
    if (!op.issued_direct) continue;
    int grid = 0;
    ICCL_CHECK_CUDA(launch_direct(op.dop, op.bytes, c->direct_ctas, s, &grid));
    c->kernels_launched += 1;
    c->ctas_launched += grid;
    c->copies_issued += 1;
    c->bytes_issued += op.bytes;
    push_krec(c, op, op.kind);  // dir: 0 pushed by this rank, 1 pulled
  }
  return ICCL_SUCCESS;
}

// Stream markers of copy-engine ops: phase 0 = WriteValue(ready) for every
// op, phase 1 = WaitValue(done) for every op; LL kernels of the same group go
// between the two phases (ready first, so no peer ever waits on our LL kernel
// through our stream order).
static iccl_result_t stream_markers(iccl_comm* c, cudaStream_t s, const std::vector<OpDesc>& ops, int phases = 3) {
  RankFlags* mine = flags_of(c, c->rank);
  std::vector<CUstreamBatchMemOpParams> p;
  p.reserve(2 * ops.size());
  for (const OpDesc& op : ops) {
    if (!(phases & 1)) break;
    CUstreamBatchMemOpParams w;
    memset(&w, 0, sizeof(w));
    w.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    w.writeValue.address = (CUdeviceptr)&mine->ready[op.slot];
    w.writeValue.value = op.gen;
    w.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    p.push_back(w);
    if (op.direct && c->device_flags) {  // the word K6 on the peer polls
      w.writeValue.address = (CUdeviceptr)(c->ll_region + dflag_ready_offset(c->nranks, op.slot));
      p.push_back(w);
    }
  }
  // done waits: a stream memop wait per op — except for direct-class ops
  // (K6 sizes), whose wait is K7: a memop wait on the host-mapped flag cost
  // ~6 us more per op in the mid-size sweep than a kernel polling it
  WaitList wl;
  memset(&wl, 0, sizeof(wl));
  wl.error = c->ll_error;
  std::vector<WaitList> kwaits;
  for (const OpDesc& op : ops) {
    if (!(phases & 2)) break;
    if ((op.direct || c->k7_ce) && c->kernel_waits) {
      wl.addr[wl.n] = &mine->done[op.slot];
      wl.alt[wl.n] = nullptr;
      if (c->device_flags) {  // K6 stores the local word; CE fallbacks only the host flag
        wl.addr[wl.n] = (const uint32_t*)(c->ll_region + dflag_done_offset(c->nranks, op.slot));
        wl.alt[wl.n] = &mine->done[op.slot];
      }
      wl.gen[wl.n] = op.gen;
      if (++wl.n == kWaitMax) {
        kwaits.push_back(wl);
        wl.n = 0;
      }
      continue;
    }
    CUstreamBatchMemOpParams w;
    memset(&w, 0, sizeof(w));
    w.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    w.waitValue.address = (CUdeviceptr)&mine->done[op.slot];
    w.waitValue.value = op.gen;
    w.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
    p.push_back(w);
  }
  iccl_result_t r = batch_memops(s, p);
  if (r) return r;
  if (wl.n > 0) kwaits.push_back(wl);
  for (const WaitList& w : kwaits) {
    ICCL_CHECK_CUDA(launch_wait(w, s));
    c->kernels_launched += 1;
    c->ctas_launched += 1;
  }
  return ICCL_SUCCESS;
}

// One fused K5 launch per (stream, group): every LL op of the group gets its
// own CTAs (1..kLLMaxBlk by size), so sends and recvs progress concurrently.
static iccl_result_t launch_ll_ops(iccl_comm* c, cudaStream_t s, std::vector<OpDesc>& ops) {
  RankFlags* mine = flags_of(c, c->rank);
  size_t i = 0;
  while (i < ops.size()) {
    LLBatch b;
    memset(&b, 0, sizeof(b));
    b.error = c->ll_error;
    uint32_t blocks = 0;
    const size_t first = i;
    for (; i < ops.size() && b.n < kLLMaxOps; i++) {
      OpDesc& op = ops[i];
      const size_t lines = (op.bytes + 3) / 4;
      const uint32_t nblk = (uint32_t)std::min<size_t>(c->ll_max_blk, std::max<size_t>(1, (lines + c->ll_lines_per_blk - 1) /
                                                                                            c->ll_lines_per_blk));
      if (b.n > 0 && blocks + nblk > (uint32_t)kLLMaxBlocksPerLaunch) break;
      LLDesc& d = b.d[b.n++];
      d.kind = op.kind;
      d.seq = op.ll_seq;
      d.bytes = op.bytes;
      d.buf = (char*)op.src;
      if (op.kind == 0) {
        d.slot = c->peer_ll[op.peer] + ll_slot_offset(c->rank, op.ll_seq);
        d.credit = (unsigned int*)(c->ll_region + ll_credit_offset(c->nranks, op.peer));
        d.stamp = alloc_kstamp(c, op);  // the sender's record: first line out -> last line out
      } else {
        d.slot = c->ll_region + ll_slot_offset(op.peer, op.ll_seq);
        d.credit = (unsigned int*)(c->peer_ll[op.peer] + ll_credit_offset(c->nranks, c->rank));
        d.stamp = nullptr;
      }
      d.done_flag = &mine->done[op.slot];
      d.done_gen = op.gen;
      d.first_blk = blocks;
      d.nblk = nblk;
      d.counter = c->ll_counters + (c->ll_ctr_next++ % kLLCounters);
      blocks += nblk;
    }
    ICCL_CHECK_CUDA(launch_ll(b, s));
    c->kernels_launched += 1;
    c->ctas_launched += blocks;
    for (size_t j = first; j < i; j++)
      if (ops[j].kind == 0) push_krec(c, ops[j], 0);
  }
  return ICCL_SUCCESS;
}

// Six-pointer record of an op nobody else publishes yet: one chunk, posted
// once its kernel or copy is queued (the issuer's proxy overwrites it with
// the real chunk pointers when the op runs on the chunked path).
static void publish_simple(iccl_comm* c, const OpDesc& op, int posted) {
  XferPub& p = flags_of(c, c->rank)->pub[op.slot];
  __atomic_store_n(&p.gen, 0u, __ATOMIC_RELEASE);
  p.kind = op.kind;
  p.total = 1;
  p.posted = posted;
  p.done = 0;
  p.path = 0;
  p.switches = 0;
  p.bytes = op.bytes;
  __atomic_store_n(&p.gen, op.gen, __ATOMIC_RELEASE);
}

static iccl_result_t enqueue_op(iccl_comm* c, int kind, const void* buf, size_t bytes, int peer, cudaStream_t s,
                                iccl_req_t* req) {
  ICCL_RETURN_IF(!c, ICCL_ERR_INVALID_ARGUMENT, "null communicator");
  ICCL_RETURN_IF(peer < 0 || peer >= c->nranks, ICCL_ERR_INVALID_ARGUMENT, "peer out of range");
  ICCL_RETURN_IF(bytes == 0, ICCL_ERR_ZERO_LENGTH_MESSAGE, "zero-length message (SPEC.md:236)");
  ICCL_RETURN_IF(!buf, ICCL_ERR_UNREGISTERED_REGION, "null buffer");
  int ae = c->async_err.load();
  if (ae != ICCL_SUCCESS) {
    set_last_error(c->async_msg);
    return (iccl_result_t)ae;
  }
  OpDesc op{};
  op.kind = kind;
  op.peer = peer;
  op.src = (const char*)buf;
  op.bytes = bytes;
  iccl_result_t r = next_slot(c, &op.slot, &op.gen, &op.op_seq);
  if (r) return r;
  publish_simple(c, op, 0);
  // Small messages between different GPUs take the LL kernel path (K5) unless
  // the copy-engine transport is forced or the pair is armed for failover
  // (route_small: both sides route the pair's q-th small op alike).
  // (a dispatch's segments never take LL: a fused sender has no source
  // tensor to stream, and both sides must classify alike)
  const bool small = !c->in_dispatch && !c->in_combine && peer != c->rank && c->cfg.transport != ICCL_TRANSPORT_CE &&
                     bytes <= c->cfg.sm_small_bytes && bytes <= kLLMaxBytes && c->ll_region != nullptr;
  op.ll = small && !route_small(pair_of(c, kind == 0 ? c->rank : peer, kind == 0 ? peer : c->rank), kind);
  op.direct = !small && peer != c->rank && c->cfg.transport == ICCL_TRANSPORT_AUTO &&
              bytes <= (size_t)c->cfg.direct_max_kib * 1024;
  if (c->in_dispatch && peer != c->rank) {
    if (kind == 1) op.direct = true;  // done wait in K7 (whoever fills the segment)
    op.fused = kind == 0 && c->dispatch_fused;
  }
  if (c->in_combine && peer != c->rank) {
    if (kind == 0) op.direct = true;  // done wait in K7 (whoever drains the segment)
    op.pull = kind == 1 && c->combine_fused;
  }
  if (op.ll) {
    op.ll_seq = kind == 0 ? ++c->ll_sent[peer] : ++c->ll_recvd[peer];
  } else if ((kind == 1 && !op.pull) || c->group_depth == 0) {
    r = rzv_post(c, op, kind == 0 ? kSendWaitUs : 0, c->group_depth > 0, s);
    if (r) return r;
  }  // a send inside a group posts at group_end, after every recv of the group (a
     // combine's pulling recv too, after its sender's half)
  c->ranks[c->rank].op_count.fetch_add(1, std::memory_order_relaxed);
  if (req) *req = ((uint64_t)op.slot << 32) | op.gen;
  if (c->group_depth > 0) {
    c->group_ops.emplace_back(op, s);
    return ICCL_SUCCESS;
  }
  if (op.ll || op.issued_direct) {
    std::vector<OpDesc> one{op};
    r = op.ll ? launch_ll_ops(c, s, one) : launch_direct_ops(c, s, one);
    if (!r) publish_simple(c, op, 1);
    return r;
  }
  if (op.issued_instream) return ICCL_SUCCESS;  // copies + done writes already on s
  return stream_markers(c, s, {op});
}

extern "C" {

iccl_result_t iccl_get_unique_id(iccl_unique_id_t* uid) {
  if (!uid) return ICCL_ERR_INVALID_ARGUMENT;
  memset(uid, 0, sizeof(*uid));
  UidBlob b{};
  b.magic = kMagic;
  std::random_device rd;
  snprintf(b.shm_name, sizeof(b.shm_name), "/iccl-b200-%d-%08x%08x", (int)getpid(), rd(), rd());
  memcpy(uid->internal, &b, sizeof(b));
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_init_rank(iccl_comm_t* out, int nranks, iccl_unique_id_t uid, int rank, int cuda_dev,
                                  const iccl_config_t* cfg) {
  ICCL_RETURN_IF(!out, ICCL_ERR_INVALID_ARGUMENT, "null comm out");
  ICCL_RETURN_IF(nranks < 1 || nranks > kMaxRanks, ICCL_ERR_INVALID_ARGUMENT, "nranks out of range");
  ICCL_RETURN_IF(rank < 0 || rank >= nranks, ICCL_ERR_INVALID_ARGUMENT, "rank out of range");
  UidBlob b;
  memcpy(&b, uid.internal, sizeof(b));
  ICCL_RETURN_IF(b.magic != kMagic, ICCL_ERR_INVALID_ARGUMENT, "bad unique id");
  iccl_config_t conf;
  if (cfg) conf = *cfg;
  else iccl_config_init(&conf);
  iccl_result_t r = iccl_config_validate(&conf);
  if (r) return r;

  ICCL_RETURN_IF(!driver(), ICCL_ERR_CUDA, last_error());
  ICCL_CHECK_CU(driver()->cuInit(0));
  ICCL_CHECK_CUDA(cudaSetDevice(cuda_dev));
  ICCL_CHECK_CUDA(cudaFree(0));  // make the primary context current
  ICCL_CHECK_CUDA(preload_kernels());
  CUdevice cd;
  ICCL_CHECK_CU(driver()->cuDeviceGet(&cd, cuda_dev));
  int memops = 0;
  driver()->cuDeviceGetAttribute(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, cd);

  auto* c = new iccl_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->dev = cuda_dev;
  c->cfg = conf;
  c->monitor_enabled.store(conf.monitor_enabled);
  c->shm_name = b.shm_name;
  for (int i = 0; i < 2 * kMaxRanks; i++) c->path_req[i].store(-1);
  c->pair_sends.assign(nranks, 0);
  c->announced.assign(nranks, {});
  c->pair_recvs.assign(nranks, 0);
  c->peer_ipc.resize(nranks);
  ShmLayout L(nranks);
  int fd = shm_open(b.shm_name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) {
    set_last_error(std::string("shm_open: ") + strerror(errno));
    delete c;
    return ICCL_ERR_SYSTEM;
  }
  if (ftruncate(fd, (off_t)L.total) != 0) {
    set_last_error(std::string("ftruncate: ") + strerror(errno));
    close(fd);
    delete c;
    return ICCL_ERR_SYSTEM;
  }
  void* m = mmap(nullptr, L.total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) {
    set_last_error(std::string("mmap: ") + strerror(errno));
    delete c;
    return ICCL_ERR_SYSTEM;
  }
  c->shm = m;
  c->shm_bytes = L.total;
  c->hdr = (ShmHeader*)m;
  c->ranks = (RankInfo*)((char*)m + L.off_ranks);
  c->flags = (RankFlags*)((char*)m + L.off_flags);
  c->rings = (RzvRing*)((char*)m + L.off_rings);
  // device-visible control block: every rank's copy streams write flags here
  ICCL_CHECK_CUDA(cudaHostRegister(m, L.total, cudaHostRegisterMapped | cudaHostRegisterPortable));
  c->pinned_bytes = 64 * 1024 + sizeof(KernelStamp) * kStampSlots + kGateWords * 4 + sizeof(ArmedWords) * kArmedSlots;
  ICCL_CHECK_CUDA(cudaHostAlloc((void**)&c->pinned, c->pinned_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(c->pinned, 0, c->pinned_bytes);
  c->gate_words = (volatile uint32_t*)((char*)c->pinned + 64 * 1024 + sizeof(KernelStamp) * kStampSlots);
  c->armed_words = (ArmedWords*)((char*)c->gate_words + kGateWords * 4);
  c->armed_used.assign(kArmedSlots, 0);
  c->gate_closed.assign(kGateWords, 0);
  c->stamps = (KernelStamp*)((char*)c->pinned + 64 * 1024);
  c->gtimer = (unsigned long long*)((char*)c->pinned + 48 * 1024);
  ICCL_CHECK_CUDA(cudaMalloc((void**)&c->scratch, kScratchBytes));
  ICCL_CHECK_CUDA(cudaMemset(c->scratch, 0, kScratchBytes));

  RankInfo& me = c->ranks[rank];
  me.pid = (int)getpid();
  me.dev = cuda_dev;
  cudaDeviceGetPCIBusId(me.bus_id, sizeof(me.bus_id), cuda_dev);
  ICCL_CHECK_CUDA(cudaIpcGetMemHandle(&me.scratch_handle, c->scratch));
  {
    size_t ll_bytes = dflag_done_offset(nranks, kSlots);
    ICCL_CHECK_CUDA(cudaMalloc((void**)&c->ll_region, ll_bytes));
    ICCL_CHECK_CUDA(cudaMemset(c->ll_region, 0, ll_bytes));
    ICCL_CHECK_CUDA(cudaIpcGetMemHandle(&me.ll_handle, c->ll_region));
    c->ll_error = (unsigned int*)((char*)c->pinned + 56 * 1024);
    c->kernel_waits = env_us("ICCL_KERNEL_WAITS", 1) != 0;
    c->device_flags = env_us("ICCL_DEVICE_FLAGS", 0) != 0;
    c->event_ready = env_us("ICCL_EVENT_READY", 0) != 0;
    c->k6_vec_bytes = (size_t)env_us("ICCL_K6_VEC_KIB", 0) * 1024;
    c->dispatch_ctas = (int)env_us("ICCL_DISPATCH_CTAS", 0);
    // kLLCounters arrival counters + kLLCounters K6 go words + kArmedSlots K9 decision words
    const size_t nctr = 2 * kLLCounters + kArmedSlots;
    ICCL_CHECK_CUDA(cudaMalloc((void**)&c->ll_counters, nctr * sizeof(unsigned int)));
    ICCL_CHECK_CUDA(cudaMemset(c->ll_counters, 0xff, nctr * sizeof(unsigned int)));
    ICCL_CHECK_CUDA(cudaMemset(c->ll_counters, 0, 2 * kLLCounters * sizeof(unsigned int)));
    c->ll_sent.assign(nranks, 0);
    c->ll_recvd.assign(nranks, 0);
    c->peer_ll.assign(nranks, nullptr);
    ICCL_CHECK_CUDA(cudaDeviceSynchronize());
  }
  c->relay_sent.assign(nranks, 0);
  c->relay_next.assign(nranks, 1);
  c->peer_relay.assign(nranks, nullptr);
  me.relay_slot_bytes = 0;
  if (conf.backup_kind == ICCL_BACKUP_RELAY && nranks >= 3) {
    c->relay_slot_bytes = (size_t)conf.relay_slot_mib << 20;
    const size_t bytes = (size_t)nranks * kRelaySlots * c->relay_slot_bytes;
    ICCL_CHECK_CUDA(cudaMalloc((void**)&c->relay_buf, bytes));
    ICCL_CHECK_CUDA(cudaIpcGetMemHandle(&me.relay_handle, c->relay_buf));
    me.relay_slot_bytes = c->relay_slot_bytes;
  }
  if (rank == 0) {
    c->hdr->nranks = nranks;
    c->hdr->magic = kMagic;
  }
  c->hdr->attached.fetch_add(1);
  // wait for everyone to attach (the first barrier also orders the RankInfo writes)
  uint64_t t0 = now_ns();
  while (c->hdr->attached.load() < nranks) {
    if ((now_ns() - t0) > 120ull * 1000000000ull) {
      set_last_error("timed out waiting for ranks to attach");
      return ICCL_ERR_TIMEOUT;
    }
    usleep(100);
  }
  r = shm_barrier(c);
  if (r) return r;
  if (rank == 0) shm_unlink(b.shm_name);

  // streams: per channel (peer x {push, pull}) S copy-engine streams; per
  // rank the group streams, one backup SM-kernel stream, one probe stream, a
  // monitor stream per direction and (relay backup) a hop-1 stream plus a
  // forwarding stream per source — 22 streams at N = 8 (29 with the relay),
  // within CUDA_DEVICE_MAX_CONNECTIONS = 32, so no stream shares a hardware
  // queue with a parked one
  int prio_lo, prio_hi;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  c->ch.resize(2 * nranks);
  uint32_t* prog = c->pinned;  // first 32 KB of pinned: progress words
  int next_prog = 0;
  // the proxy indexes c->streams while the API thread may still add a
  // channel's backup / progress stream: reserve so it never reallocates
  c->streams.reserve(64 + 40 * (size_t)nranks);
  auto mk_stream = [&](int engine) -> int {
    StreamCtx sc;
    cudaStreamCreateWithPriority(&sc.s, cudaStreamNonBlocking, prio_hi);
    cudaEventCreateWithFlags(&sc.ev, cudaEventDisableTiming);
    sc.prog = prog + 16 * (next_prog++);  // one 64-byte line each
    sc.engine = engine;
    c->streams.push_back(sc);
    return (int)c->streams.size() - 1;
  };
  // the group streams: remote pushes / remote pulls of a group (rzv_post)
  // ICCL_GROUP_LANES (1..4) streams per direction: consecutive transfers of a
  // group alternate between them
  const int lanes = (int)std::min<uint64_t>(4, std::max<uint64_t>(1, env_us("ICCL_GROUP_LANES", 1)));
  std::vector<int> group_si[2];
  for (int d = 0; d < 2; d++)
    for (int l = 0; l < lanes; l++) group_si[d].push_back(mk_stream(ENG_CE_GROUP));
  c->group_lanes = lanes;
  c->sm_si = mk_stream(ENG_SM);
  c->probe_si = mk_stream(ENG_CE);
  c->mon_si[0] = mk_stream(ENG_CE);
  c->mon_si[1] = mk_stream(ENG_CE);
  if (c->relay_buf) c->relay_si = mk_stream(ENG_RELAY);
  c->self_si = mk_stream(ENG_CE);
  ICCL_CHECK_CUDA(cudaEventCreateWithFlags(&c->self_fork, cudaEventDisableTiming));
  ICCL_CHECK_CUDA(cudaEventCreateWithFlags(&c->self_join, cudaEventDisableTiming));
  c->self_overlap = env_us("ICCL_SELF_OVERLAP", 1) != 0;
  c->k7_ce = env_us("ICCL_K7_CE", 0) != 0;
  c->k7_ready = env_us("ICCL_K7_READY", 0) != 0;
  c->a2a_pieces = (int)std::min<uint64_t>(16, std::max<uint64_t>(1, env_us("ICCL_A2A_PIECES", 1)));
  c->a2a_order = (int)env_us("ICCL_A2A_ORDER", 0);
  c->ll_lines_per_blk = (size_t)std::max<uint64_t>(256, env_us("ICCL_LL_LINES_PER_BLK", kLLLinesPerBlk));
  c->ll_max_blk = (int)std::min<uint64_t>(64, std::max<uint64_t>(1, env_us("ICCL_LL_MAX_BLK", kLLMaxBlk)));
  c->instream_ce = env_us("ICCL_INSTREAM", 1) != 0;
  c->armed_backup = env_us("ICCL_ARMED_BACKUP", 1) != 0;
  c->k9_mode = (int)env_us("ICCL_K9_MODE", 0);
  c->prog_events = env_us("ICCL_PROG_EVENTS", 1) != 0;
  std::vector<char*> peer_scratch(nranks, nullptr);
  for (int p = 0; p < nranks; p++) {
    if (p == rank) {
      peer_scratch[p] = c->scratch + 2048;
    } else {
      void* ps = nullptr;
      ICCL_CHECK_CUDA(cudaIpcOpenMemHandle(&ps, c->ranks[p].scratch_handle, cudaIpcMemLazyEnablePeerAccess));
      c->peer_scratch_base.push_back((char*)ps);
      peer_scratch[p] = (char*)ps + 16 * (1 + rank);
      void* pl = nullptr;
      ICCL_CHECK_CUDA(cudaIpcOpenMemHandle(&pl, c->ranks[p].ll_handle, cudaIpcMemLazyEnablePeerAccess));
      c->peer_ll[p] = (char*)pl;
    }
  }
  for (int ci = 0; ci < 2 * nranks; ci++) {
    const int p = ci / 2;
    Channel& chn = c->ch[ci];
    chn.peer = p;
    chn.dir = ci % 2;
    chn.src = chn.dir == 0 ? rank : p;
    chn.dst = chn.dir == 0 ? p : rank;
    chn.peer_scratch = peer_scratch[p];
    for (int s = 0; s < conf.streams_per_peer; s++) {
      int si = mk_stream(ENG_CE);
      chn.path_streams[0].push_back(si);
      chn.path_streams[1].push_back(si);
    }
    chn.path_streams[1].push_back(c->sm_si);
    if (c->relay_buf && p != rank && chn.dir == 0) {
      for (int q = 0; q < nranks; q++)
        if (q != rank && q != p) {
          chn.relay_rank = q;  // lowest-index GPU that is not an endpoint
          break;
        }
      chn.path_streams[1].push_back(c->relay_si);
    }
    if (p != rank) {
      for (int gs : group_si[chn.dir]) {
        chn.path_streams[0].push_back(gs);
        chn.path_streams[1].push_back(gs);
      }
    }
    chn.probe_stream = c->probe_si;
    chn.mon_stream = c->mon_si[chn.dir];
    ICCL_CHECK_CUDA(cudaEventCreateWithFlags(&chn.bridge, cudaEventDisableTiming));
    c->all_events.push_back(chn.bridge);
  }
  if (c->relay_buf) {
    c->relay_serve.assign(nranks, -1);
    for (int q = 0; q < nranks; q++)
      if (q != rank) c->relay_serve[q] = mk_stream(ENG_RELAY);
  }
  // %globaltimer -> CLOCK_MONOTONIC offset for SM-path monitor stamps
  {
    cudaStream_t s = c->streams[0].s;
    *c->gtimer = 0;
    uint64_t h0 = now_ns();
    ICCL_CHECK_CUDA(launch_read_globaltimer(c->gtimer, s));
    // time base of the monitor's timing events: recorded right behind the
    // %globaltimer read, so both stamp kinds share one clock (to ~1 us)
    ICCL_CHECK_CUDA(cudaEventCreate(&c->base_ev));
    c->all_events.push_back(c->base_ev);
    ICCL_CHECK_CUDA(cudaEventRecord(c->base_ev, s));
    ICCL_CHECK_CUDA(cudaStreamSynchronize(s));
    uint64_t h1 = now_ns();
    c->gtimer_offset = (int64_t)((h0 + h1) / 2) - (int64_t)(*c->gtimer);
    c->base_abs_ns = (int64_t)(*c->gtimer) + c->gtimer_offset;
  }
  r = shm_barrier(c);
  if (r) return r;
  c->proxy = std::thread(proxy_loop, c);
  c->watchdog = std::thread(watch_loop, c);
  *out = c;
  return ICCL_SUCCESS;
}

// sync = false (abort): the side streams may be parked for good on a wait
// for a peer that died (its ready flag, a relay counter), so they are
// destroyed without synchronising; CUDA releases them once they drain.
static void teardown(iccl_comm* c, bool sync = true) {
  if (c->proxy.joinable()) {
    c->stop.store(true);
    c->qcv.notify_one();
    c->proxy.join();
  }
  if (c->watchdog.joinable()) {
    c->stop.store(true);
    c->watchdog.join();
  }
  for (auto& sc : c->streams) {
    if (sc.s) {
      if (sync) cudaStreamSynchronize(sc.s);
      cudaStreamDestroy(sc.s);
    }
    if (sc.ev) cudaEventDestroy(sc.ev);
  }
  for (cudaEvent_t e : c->all_events) cudaEventDestroy(e);
  if (c->self_fork) cudaEventDestroy(c->self_fork);
  if (c->self_join) cudaEventDestroy(c->self_join);
  for (auto& cache : c->peer_ipc)
    for (auto& kv : cache) cudaIpcCloseMemHandle(kv.second);
  for (char* p : c->peer_scratch_base) cudaIpcCloseMemHandle(p);
  for (size_t p = 0; p < c->peer_ll.size(); p++)
    if (c->peer_ll[p] && (int)p != c->rank) cudaIpcCloseMemHandle(c->peer_ll[p]);
  for (char* p : c->peer_relay)
    if (p) cudaIpcCloseMemHandle(p);
  if (c->relay_buf) cudaFree(c->relay_buf);
  if (c->ll_region) cudaFree(c->ll_region);
  if (c->ll_counters) cudaFree(c->ll_counters);
  if (c->scratch) cudaFree(c->scratch);
  if (c->shm) {
    cudaHostUnregister(c->shm);
    munmap(c->shm, c->shm_bytes);
  }
  if (c->pinned) cudaFreeHost(c->pinned);
}

iccl_result_t iccl_comm_destroy(iccl_comm_t c) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  // drain: every send this rank owns must have been handed to the device
  uint64_t t0 = now_ns();
  while (c->pending_xfers.load() > 0 && c->async_err.load() == ICCL_SUCCESS && !c->hdr->abort.load()) {
    if (now_ns() - t0 > 120ull * 1000000000ull) break;
    usleep(50);
  }
  // every rank's sends retired (their relayed pieces included) before any
  // proxy stops: a relay GPU serves forwarding requests until here
  iccl_result_t r0 = c->hdr->abort.load() ? ICCL_SUCCESS : shm_barrier(c);
  if (c->proxy.joinable()) {
    c->stop.store(true);
    c->qcv.notify_one();
    c->proxy.join();
  }
  if (c->watchdog.joinable()) c->watchdog.join();
  // Injected faults may still hold probes behind a closed gate; no data copy
  // is gated any more (stale copies are flushed before their op completes),
  // so open every gate and let the side streams drain.
  for (int g = 0; g < kGateWords; g++) __atomic_store_n((uint32_t*)&c->gate_words[g], 1u, __ATOMIC_SEQ_CST);
  for (auto& sc : c->streams) cudaStreamSynchronize(sc.s);
  iccl_result_t r = c->hdr->abort.load() ? ICCL_SUCCESS : shm_barrier(c);
  if (r == ICCL_SUCCESS) r = r0;
  teardown(c);
  delete c;
  return r == ICCL_ERR_ABORTED ? ICCL_SUCCESS : r;
}

iccl_result_t iccl_comm_abort(iccl_comm_t c) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  c->hdr->abort.store(1);
  set_async(c, ICCL_ERR_ABORTED, "communicator aborted");
  // release every op slot of this rank so no user stream stays blocked
  RankFlags* mine = flags_of(c, c->rank);
  for (uint64_t s = c->op_seq > (uint64_t)kSlots ? c->op_seq - kSlots : 0; s < c->op_seq; s++)
    __atomic_store_n(&mine->done[s % kSlots], (uint32_t)(s + 1), __ATOMIC_SEQ_CST);
  for (int g = 0; g < kGateWords; g++) __atomic_store_n((uint32_t*)&c->gate_words[g], 1u, __ATOMIC_SEQ_CST);
  for (int i = 0; i < kArmedSlots; i++) {  // unpark every armed attempt (the backups copy nothing)
    ArmedWords* w = &c->armed_words[i];
    __atomic_store_n(&w->resume, 0xffffffffu, __ATOMIC_SEQ_CST);
    __atomic_store_n(&w->ctl, (uint32_t)kCtlAbort, __ATOMIC_SEQ_CST);
    __atomic_store_n(&w->go, 1u, __ATOMIC_SEQ_CST);
    __atomic_store_n(&w->ns, 1u, __ATOMIC_SEQ_CST);
  }
  // mapped peer memory and the control block stay mapped (leaked): a parked
  // stream may still touch them when it drains
  c->peer_ipc.clear();
  c->peer_scratch_base.clear();
  c->peer_ll.clear();
  c->peer_relay.clear();
  c->shm = nullptr;
  c->scratch = c->ll_region = c->relay_buf = nullptr;
  c->ll_counters = nullptr;
  c->pinned = nullptr;
  teardown(c, false);
  delete c;
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_count(iccl_comm_t c, int* n) {
  if (!c || !n) return ICCL_ERR_INVALID_ARGUMENT;
  *n = c->nranks;
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_user_rank(iccl_comm_t c, int* r) {
  if (!c || !r) return ICCL_ERR_INVALID_ARGUMENT;
  *r = c->rank;
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_get_async_error(iccl_comm_t c, iccl_result_t* err) {
  if (!c || !err) return ICCL_ERR_INVALID_ARGUMENT;
  *err = (iccl_result_t)c->async_err.load();
  if (*err != ICCL_SUCCESS) set_last_error(c->async_msg);
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_op_counts(iccl_comm_t c, uint64_t* counts, int n) {
  if (!c || !counts || n < c->nranks) return ICCL_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < c->nranks; i++) counts[i] = c->ranks[i].op_count.load();
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_stats(iccl_comm_t c, iccl_stats_t* s) {
  if (!c || !s) return ICCL_ERR_INVALID_ARGUMENT;
  memset(s, 0, sizeof(*s));
  s->kernels_launched = c->kernels_launched.load();
  s->ctas_launched = c->ctas_launched.load();
  s->copies_issued = c->copies_issued.load();
  s->bytes_issued = c->bytes_issued.load();
  s->pulls_issued = c->pulls_issued.load();
  s->cts_timeouts = c->cts_timeouts.load();
  s->pending_xfers = c->pending_xfers.load() + c->krecs_pending.load();  // K5 / K6 / K8 records not yet emitted count
  return ICCL_SUCCESS;
}

iccl_result_t iccl_register(iccl_comm_t c, void* ptr, size_t bytes, uint64_t* handle) {
  if (!c || !ptr || !handle) return ICCL_ERR_INVALID_ARGUMENT;
  CUdeviceptr base = 0;
  size_t asize = 0;
  ICCL_CHECK_CU(driver()->cuMemGetAddressRange(&base, &asize, (CUdeviceptr)ptr));
  ICCL_RETURN_IF((CUdeviceptr)ptr + bytes > base + asize, ICCL_ERR_UNREGISTERED_REGION,
                 "region exceeds its allocation");
  unsigned long long bid = 0;
  ICCL_CHECK_CU(driver()->cuPointerGetAttribute(&bid, CU_POINTER_ATTRIBUTE_BUFFER_ID, (CUdeviceptr)ptr));
  if (!c->export_cache.count(bid)) {
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
    ICCL_RETURN_IF(e != cudaSuccess, ICCL_ERR_UNREGISTERED_REGION, "allocation cannot be exported over IPC");
    c->export_cache.emplace(bid, h);
  }
  *handle = bid;
  return ICCL_SUCCESS;
}

// The caller promises no op in flight uses the buffer: drop the export and
// tell every peer that mapped it to close its mapping (their proxies do it).
iccl_result_t iccl_deregister(iccl_comm_t c, uint64_t handle) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  auto it = c->export_cache.find(handle);
  ICCL_RETURN_IF(it == c->export_cache.end(), ICCL_ERR_UNREGISTERED_REGION, "unknown registration handle");
  const cudaIpcMemHandle_t h = it->second;
  c->export_cache.erase(it);
  for (int p = 0; p < c->nranks; p++) {
    if (p == c->rank || !c->announced[p].count(handle)) continue;
    uint64_t t0 = now_ns();
    while (!announce_entry(c, p, AnnEntry{handle, 1, h})) {  // the ring drains in the peer's proxy
      ICCL_RETURN_IF(now_ns() - t0 > 10ull * 1000000000ull, ICCL_ERR_TIMEOUT, "peer did not drain its announcements");
      usleep(50);
    }
    c->announced[p].erase(handle);
  }
  return ICCL_SUCCESS;
}

iccl_result_t iccl_send(iccl_comm_t c, const void* buf, size_t bytes, int peer, cudaStream_t s, iccl_req_t* req) {
  return enqueue_op(c, 0, buf, bytes, peer, s, req);
}

iccl_result_t iccl_recv(iccl_comm_t c, void* buf, size_t bytes, int peer, cudaStream_t s, iccl_req_t* req) {
  return enqueue_op(c, 1, buf, bytes, peer, s, req);
}

iccl_result_t iccl_group_start(iccl_comm_t c) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  c->group_depth++;
  return ICCL_SUCCESS;
}

iccl_result_t iccl_group_end(iccl_comm_t c) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_RETURN_IF(c->group_depth <= 0, ICCL_ERR_INVALID_ARGUMENT, "group_end without group_start");
  if (--c->group_depth > 0) return ICCL_SUCCESS;
  std::vector<std::pair<OpDesc, cudaStream_t>> ops;
  ops.swap(c->group_ops);
  // the group's sends, in call order: each waits (within one shared budget)
  // for its receiver's half so that it arrives second and pushes
  const uint64_t deadline = now_ns() + kGroupSendWaitUs * 1000ull;
  for (auto& p : ops) {
    if (p.first.kind != 0 || p.first.ll) continue;
    if (p.first.fused) {
      iccl_result_t r = fused_rendezvous(c, p.first);
      if (r) return r;
      continue;
    }
    const uint64_t t = now_ns();
    // a combine's sends post at once: their receivers pull (K10) and wait for them
    const uint64_t budget = c->in_combine ? 0 : (t < deadline ? (deadline - t) / 1000 : 0);
    iccl_result_t r = rzv_post(c, p.first, budget, true, p.second);
    if (r) return r;
  }
  for (auto& p : ops) {
    if (!p.first.pull) continue;
    iccl_result_t r = pull_rendezvous(c, p.first);
    if (r) return r;
  }
  // every transfer this side issues for the group: in-stream on the op's own
  // stream where the pair allows it, else on the side streams
  std::vector<iccl_comm::GroupJob> jobs;
  jobs.swap(c->group_jobs);
  auto find_op = [&](int kind, int peer, const RzvSide& s) -> OpDesc* {
    for (auto& p : ops)
      if (p.first.kind == kind && p.first.peer == peer && p.first.slot == s.slot && p.first.gen == s.gen)
        return &p.first;
    return nullptr;
  };
  // mode per job: 1 plain in-stream, 2 armed in-stream, 3 armed on the side
  // streams, 0 the proxy-driven side-stream pipeline (see rzv_post)
  std::vector<Xfer> xs(jobs.size());
  std::vector<char> mode(jobs.size(), 0), elide(jobs.size(), 0);
  for (size_t i = 0; i < jobs.size(); i++) {
    const auto& j = jobs[i];
    iccl_result_t r = rzv_build(c, j.kind, j.peer, j.k, j.op_seq, true, j.side, &xs[i]);
    if (r) return r;
    const RzvSide& other = j.side[j.kind ^ 1];
    OpDesc* oth = j.peer == c->rank ? find_op(j.kind ^ 1, j.peer, other) : nullptr;
    const bool stream_ok = instream_ok(c, j.kind, j.peer, j.side, oth != nullptr, j.stream);
    if (xfer_armed(c, j.kind, j.peer))
      mode[i] = armed_eligible(c, xs[i]) ? (stream_ok ? 2 : 3) : 0;
    else
      mode[i] = stream_ok ? 1 : 0;
    if (mode[i] != 1 && mode[i] != 2) continue;
    if (OpDesc* me = find_op(j.kind, j.peer, j.side[j.kind])) me->issued_instream = true;
    if (mode[i] == 1 && oth && other.stream == (uint64_t)(uintptr_t)j.stream) {
      // self pair, both halves of one group on one stream: the stream already
      // orders the copy after both ops' positions — no markers, no waits
      oth->markers_elided = true;
      elide[i] = 1;
    }
  }
  {
    // Side-stream transfers: a group's pushes share one stream (rzv_post):
    // enqueue every ready wait first, then the copies back to back — a wait
    // placed between two copies would cost each a copy-engine drain (~15 us
    // per peer in the 4-rank alltoallv records).  Armed ones go to their
    // channel's own streams.
    int nth[2] = {0, 0};
    for (size_t i = 0; i < xs.size(); i++) {
      if (mode[i] == 3) xs[i].group_stream = false;
      if (mode[i] == 0 && xs[i].group_stream) xs[i].group_lane = nth[c->ch[xs[i].chan].dir]++ % c->group_lanes;
    }
    for (size_t i = 0; i < xs.size(); i++) {
      if (mode[i] != 0) continue;
      iccl_result_t r = ready_waits(c, c->ch[xs[i].chan], xs[i]);
      if (r) return r;
    }
    for (size_t i = 0; i < xs.size(); i++) {
      iccl_result_t r = ICCL_SUCCESS;
      if (mode[i] == 0) r = rzv_launch(c, std::move(xs[i]), false);
      if (mode[i] == 3) r = armed_launch(c, std::move(xs[i]), jobs[i].kind, jobs[i].stream, false);
      if (r) return r;
    }
  }
  // Per user stream: ready markers of the ops a peer (or a side stream)
  // issues, then the kernels (LL, K6 this side runs), then this side's
  // in-stream transfers (their ready waits hoisted in front of the copies, the
  // done writes batched behind them), then the done waits — no kernel or copy
  // of ours ever sits in front of a ready flag a peer needs.
  std::vector<cudaStream_t> order;
  for (auto& p : ops)
    if (std::find(order.begin(), order.end(), p.second) == order.end()) order.push_back(p.second);
  for (cudaStream_t s : order) {
    std::vector<OpDesc> ce, ll, direct, fused;
    for (auto& p : ops) {
      if (p.second != s || p.first.issued_instream || p.first.markers_elided) continue;
      (p.first.fused || p.first.pull ? fused : p.first.ll ? ll : p.first.issued_direct ? direct : ce).push_back(p.first);
    }
    iccl_result_t r = ICCL_SUCCESS;
    if (!ce.empty()) r = stream_markers(c, s, ce, 1);  // ready
    if (!r && !ll.empty()) r = launch_ll_ops(c, s, ll);
    if (!r && !direct.empty()) r = launch_direct_ops(c, s, direct);
    if (!r && c->dispatch_fused && c->dispatch_stream == s) r = launch_fused_dispatch(c, s, fused);
    if (!r && c->combine_fused && c->combine_stream == s) r = launch_fused_combine(c, s, fused);
    if (r) return r;
    std::vector<CUstreamBatchMemOpParams> p;
    std::vector<size_t> mine;
    for (size_t i = 0; i < jobs.size(); i++)
      if (mode[i] == 1 && jobs[i].stream == s) mine.push_back(i);
    if (!mine.empty()) {
      for (size_t i : mine)
        if (!elide[i]) instream_ready_param(c, xs[i], jobs[i].kind, p);
      r = ready_wait_ops(c, s, p);
      // the self copy (both halves on s, nothing to wait for) forks off to
      // self_si when NVLink copies follow it, and s joins it before the done
      // writes: a local copy and a peer copy run on different copy engines
      std::vector<size_t> self, remote;
      for (size_t i : mine) (elide[i] && c->self_overlap ? self : remote).push_back(i);
      bool armed_here = false;  // armed transfers of this stream (mode 2) go between the fork and the join
      for (size_t i = 0; i < jobs.size(); i++) armed_here |= mode[i] == 2 && jobs[i].stream == s;
      if (remote.empty() && !armed_here) {
        remote.swap(self);
      }
      cudaStream_t ss = c->streams[c->self_si].s;
      if (!r && !self.empty()) {
        ICCL_CHECK_CUDA(cudaEventRecord(c->self_fork, s));
        ICCL_CHECK_CUDA(cudaStreamWaitEvent(ss, c->self_fork, 0));
        for (size_t i : self)
          if (!r) r = instream_copies(c, xs[i], ss);
        if (!r) ICCL_CHECK_CUDA(cudaEventRecord(c->self_join, ss));
      }
      for (size_t i : remote)
        if (!r) r = instream_copies(c, xs[i], s);
      for (size_t i = 0; i < jobs.size() && !r; i++)
        if (mode[i] == 2 && jobs[i].stream == s) r = armed_launch(c, std::move(xs[i]), jobs[i].kind, s, true);
      if (!r && !self.empty()) ICCL_CHECK_CUDA(cudaStreamWaitEvent(s, c->self_join, 0));
      for (size_t i : mine) instream_done_params(c, xs[i], p);
      if (!r) r = batch_memops(s, p);
      if (r) return r;
      for (size_t i : mine) rzv_track(c, std::move(xs[i]), false);
    } else {
      for (size_t i = 0; i < jobs.size() && !r; i++)
        if (mode[i] == 2 && jobs[i].stream == s) r = armed_launch(c, std::move(xs[i]), jobs[i].kind, s, true);
    }
    if (r) return r;
    if (!ce.empty()) r = stream_markers(c, s, ce, 2);  // done waits
    if (r) return r;
    for (const OpDesc& o : ll) publish_simple(c, o, 1);
    for (const OpDesc& o : direct) publish_simple(c, o, 1);
    for (const OpDesc& o : fused) publish_simple(c, o, 1);
  }
  return ICCL_SUCCESS;
}

iccl_result_t iccl_alltoallv(iccl_comm_t c, const void* sbuf, const size_t* scounts, const size_t* sdispls,
                             void* rbuf, const size_t* rcounts, const size_t* rdispls, size_t elem_bytes,
                             cudaStream_t s) {
  if (!c || !scounts || !sdispls || !rcounts || !rdispls || elem_bytes == 0) return ICCL_ERR_INVALID_ARGUMENT;
  iccl_result_t r = iccl_group_start(c);
  if (r) return r;
  const int n = c->nranks;
  // rotated schedule: step k pairs rank i with i+k (send) and i-k (recv) so
  // the NVSwitch sees no incast; k = 0 is the self copy.
  // ICCL_A2A_PIECES = P > 1 splits every remote segment into P pieces (both
  // sides split a pair's count the same way) and rotates piece-major, so a
  // rank that finishes a step early cannot run ahead by a whole segment.
  const int pieces = c->a2a_pieces;
  // ICCL_A2A_ORDER=1: the remote sends in decreasing size (largest segment
  // first) instead of the rotation; receives keep the rotated order
  std::vector<int> send_to(n);
  for (int k = 0; k < n; k++) send_to[k] = (c->rank + k) % n;
  if (c->a2a_order == 1)
    std::stable_sort(send_to.begin() + 1, send_to.end(), [&](int a, int b) { return scounts[a] > scounts[b]; });
  for (int pc = 0; pc < pieces && r == ICCL_SUCCESS; pc++) {
    for (int k = pc == 0 ? 0 : 1; k < n && r == ICCL_SUCCESS; k++) {
      int to = send_to[k], from = (c->rank - k + n) % n;
      const int np = k == 0 ? 1 : pieces;
      if (k == 0 && pc > 0) continue;
      auto piece = [&](size_t cnt, size_t* lo, size_t* len) {  // piece pc of cnt elements
        *lo = cnt * (size_t)pc / np;
        *len = cnt * (size_t)(pc + 1) / np - *lo;
      };
      size_t lo, len;
      piece(rcounts[from], &lo, &len);
      if (len) r = iccl_recv(c, (char*)rbuf + (rdispls[from] + lo) * elem_bytes, len * elem_bytes, from, s, nullptr);
      piece(scounts[to], &lo, &len);
      if (!r && len)
        r = iccl_send(c, (const char*)sbuf + (sdispls[to] + lo) * elem_bytes, len * elem_bytes, to, s, nullptr);
    }
  }
  iccl_result_t r2 = iccl_group_end(c);
  return r ? r : r2;
}

// Fused MoE dispatch (K8): see include/iccl_b200.h.  Equivalent to
// iccl_expand_rows into a packed buffer followed by iccl_alltoallv of it, in
// one kernel and without the packed buffer.  If a pair this rank sends to is
// armed for failover (a fault script names it, or it runs on its backup
// path), the call takes exactly that unfused form instead — K2 into a staging
// buffer, then the alltoallv, where the gates, the watchdog and the switch
// apply; receivers cannot tell the two forms apart.
iccl_result_t iccl_dispatch_rows(iccl_comm_t c, const void* tokens, int64_t n_tokens, int32_t k, const int64_t* pos,
                                 const size_t* scounts, void* rbuf, const size_t* rcounts, int64_t row_bytes,
                                 cudaStream_t s) {
  ICCL_RETURN_IF(!c || !scounts || !rcounts || n_tokens < 0 || k < 1 || k > 32 || row_bytes <= 0 || (row_bytes & 15),
                 ICCL_ERR_INVALID_ARGUMENT, "dispatch: bad arguments (1 <= k <= 32, row_bytes a multiple of 16)");
  ICCL_RETURN_IF(c->group_depth > 0, ICCL_ERR_INVALID_ARGUMENT, "dispatch inside a group");
  ICCL_RETURN_IF(c->nranks > kMaxFusedRanks, ICCL_ERR_INVALID_ARGUMENT, "dispatch: more than 64 ranks");
  ICCL_RETURN_IF(((uintptr_t)tokens & 15) || ((uintptr_t)rbuf & 15), ICCL_ERR_INVALID_ARGUMENT,
                 "dispatch: tokens and the receive buffer must be 16-byte aligned");
  int ae = c->async_err.load();
  if (ae != ICCL_SUCCESS) {
    set_last_error(c->async_msg);
    return (iccl_result_t)ae;
  }
  const int n = c->nranks, me = c->rank;
  std::vector<size_t> sd(n), rd(n);
  size_t stot = 0, rtot = 0;
  for (int d = 0; d < n; d++) {
    sd[d] = stot;
    rd[d] = rtot;
    stot += scounts[d];
    rtot += rcounts[d];
  }
  ICCL_RETURN_IF(stot != (size_t)n_tokens * (size_t)k, ICCL_ERR_INVALID_ARGUMENT,
                 "dispatch: send counts must add up to n_tokens * k");
  ICCL_RETURN_IF(scounts[me] != rcounts[me], ICCL_ERR_SIZE_MISMATCH, "dispatch: self send and receive counts differ");
  ICCL_RETURN_IF(stot > 0 && (!tokens || !pos), ICCL_ERR_INVALID_ARGUMENT, "dispatch: null tokens / pos");
  ICCL_RETURN_IF(rtot > 0 && !rbuf, ICCL_ERR_INVALID_ARGUMENT, "dispatch: null receive buffer");
  bool fused = true;
  for (int d = 0; d < n && fused; d++)
    if (d != me && scounts[d] && xfer_armed(c, 0, d)) fused = false;
  iccl_result_t r = ICCL_SUCCESS;
  if (!fused) {
    const size_t need = stot * (size_t)row_bytes;
    if (need > c->dispatch_stage_bytes) {
      if (c->dispatch_stage) {
        ICCL_CHECK_CUDA(cudaStreamSynchronize(s));  // the previous fallback's copies may still read it
        ICCL_CHECK_CUDA(cudaFree(c->dispatch_stage));
        c->dispatch_stage = nullptr;
      }
      ICCL_CHECK_CUDA(cudaMalloc((void**)&c->dispatch_stage, need));
      c->dispatch_stage_bytes = need;
    }
    if (stot) ICCL_CHECK_CUDA(launch_expand_rows(tokens, c->dispatch_stage, pos, n_tokens, k, row_bytes, 0, s));
    c->in_dispatch = true;
    r = iccl_alltoallv(c, c->dispatch_stage, scounts, sd.data(), rbuf, rcounts, rd.data(), (size_t)row_bytes, s);
    c->in_dispatch = false;
    return r;
  }
  // the dispatch's own op slot: its done flag (written by K8's last CTA)
  // retires it, and it keys K8's go word
  OpDesc dop{};
  r = next_slot(c, &dop.slot, &dop.gen, &dop.op_seq);
  if (r) return r;
  DispatchOp& op = c->dispatch_op;
  memset(&op, 0, sizeof(op));
  op.tokens = (const int4*)tokens;
  op.pos = pos;
  op.n_tokens = n_tokens;
  op.k = k;
  op.n = n;
  op.row16 = row_bytes / 16;
  op.parts = (int)std::max<int64_t>(1, std::min<int64_t>(8, op.row16 / 128));
  op.ticket = c->ll_counters + (c->ll_ctr_next++ % kLLCounters);
  op.counter = c->ll_counters + (c->ll_ctr_next++ % kLLCounters);
  op.go = c->ll_counters + kLLCounters + (dop.slot % kLLCounters);
  op.go_gen = dop.gen;
  op.error = c->ll_error;
  for (int d = 0; d < n; d++) {
    op.d[d].lo = (int64_t)sd[d];
    op.d[d].hi = (int64_t)(sd[d] + scounts[d]);
  }
  op.d[me].seg = (char*)rbuf + rd[me] * (size_t)row_bytes;
  op.d[me].my_done = &flags_of(c, me)->done[dop.slot];
  op.d[me].my_done_gen = dop.gen;
  c->dispatch_stream = s;
  c->dispatch_fused = true;
  c->in_dispatch = true;
  r = iccl_group_start(c);
  // rotated like iccl_alltoallv; the self segment is K8's local store
  for (int kk = 1; kk < n && r == ICCL_SUCCESS; kk++) {
    const int to = (me + kk) % n, from = (me - kk + n) % n;
    if (rcounts[from]) r = iccl_recv(c, (char*)rbuf + rd[from] * (size_t)row_bytes, rcounts[from] * (size_t)row_bytes,
                                     from, s, nullptr);
    if (!r && scounts[to]) r = iccl_send(c, tokens, scounts[to] * (size_t)row_bytes, to, s, nullptr);
  }
  iccl_result_t r2 = iccl_group_end(c);
  if (!r) r = r2;
  // no remote send on s (a single rank, or every row stays here): K8 still
  // stores the self segment
  if (!r && c->dispatch_fused) r = launch_fused_dispatch(c, s, {});
  c->dispatch_fused = false;
  c->in_dispatch = false;
  return r;
}

// Fused MoE combine (K10): see include/iccl_b200.h.  Equivalent to
// iccl_alltoallv of the expert rows back to their token ranks into a packed
// buffer followed by iccl_scatter_rows(packed -> out, order), in one kernel
// on the receiving side and without the packed buffer.  If a pair this rank
// receives from is armed for failover, the call takes exactly that unfused
// form (staging + alltoallv + K3); senders cannot tell the two forms apart.
iccl_result_t iccl_combine_rows(iccl_comm_t c, const void* expert_rows, const size_t* scounts, void* out,
                                const int64_t* order, const size_t* rcounts, int64_t row_bytes, cudaStream_t s) {
  ICCL_RETURN_IF(!c || !scounts || !rcounts || row_bytes <= 0 || (row_bytes & 15), ICCL_ERR_INVALID_ARGUMENT,
                 "combine: bad arguments (row_bytes a multiple of 16)");
  ICCL_RETURN_IF(c->group_depth > 0, ICCL_ERR_INVALID_ARGUMENT, "combine inside a group");
  ICCL_RETURN_IF(c->nranks > kMaxFusedRanks, ICCL_ERR_INVALID_ARGUMENT, "combine: more than 64 ranks");
  ICCL_RETURN_IF(((uintptr_t)expert_rows & 15) || ((uintptr_t)out & 15), ICCL_ERR_INVALID_ARGUMENT,
                 "combine: the expert rows and the output must be 16-byte aligned");
  int ae = c->async_err.load();
  if (ae != ICCL_SUCCESS) {
    set_last_error(c->async_msg);
    return (iccl_result_t)ae;
  }
  const int n = c->nranks, me = c->rank;
  std::vector<size_t> sd(n), rd(n);
  size_t stot = 0, rtot = 0;
  for (int d = 0; d < n; d++) {
    sd[d] = stot;
    rd[d] = rtot;
    stot += scounts[d];
    rtot += rcounts[d];
  }
  ICCL_RETURN_IF(scounts[me] != rcounts[me], ICCL_ERR_SIZE_MISMATCH, "combine: self send and receive counts differ");
  ICCL_RETURN_IF(stot > 0 && !expert_rows, ICCL_ERR_INVALID_ARGUMENT, "combine: null expert rows");
  ICCL_RETURN_IF(rtot > 0 && (!out || !order), ICCL_ERR_INVALID_ARGUMENT, "combine: null output / order");
  bool fused = true;
  for (int d = 0; d < n && fused; d++)
    if (d != me && rcounts[d] && xfer_armed(c, 1, d)) fused = false;
  iccl_result_t r = ICCL_SUCCESS;
  if (!fused) {
    const size_t need = rtot * (size_t)row_bytes;
    if (need > c->dispatch_stage_bytes) {
      if (c->dispatch_stage) {
        ICCL_CHECK_CUDA(cudaStreamSynchronize(s));
        ICCL_CHECK_CUDA(cudaFree(c->dispatch_stage));
        c->dispatch_stage = nullptr;
      }
      ICCL_CHECK_CUDA(cudaMalloc((void**)&c->dispatch_stage, need));
      c->dispatch_stage_bytes = need;
    }
    c->in_combine = true;
    r = iccl_alltoallv(c, expert_rows, scounts, sd.data(), c->dispatch_stage, rcounts, rd.data(), (size_t)row_bytes, s);
    c->in_combine = false;
    if (!r && rtot) ICCL_CHECK_CUDA(launch_scatter_rows(c->dispatch_stage, out, order, (int64_t)rtot, row_bytes, 148 * 8, s));
    return r;
  }
  OpDesc cop{};
  r = next_slot(c, &cop.slot, &cop.gen, &cop.op_seq);
  if (r) return r;
  CombineOp& op = c->combine_op;
  memset(&op, 0, sizeof(op));
  op.out = (int4*)out;
  op.order = order;
  op.n_rows = (int64_t)rtot;
  {  // a stride near n_rows / golden ratio, coprime to n_rows (a bijection of the rows)
    auto gcd = [](uint64_t a, uint64_t b) { while (b) { uint64_t t = a % b; a = b; b = t; } return a; };
    uint64_t st = rtot > 2 ? (uint64_t)(rtot * 0.6180339887) | 1 : 1;
    while (rtot > 1 && gcd(st, rtot) != 1) st += 2;
    op.stride = (int64_t)st;
  }
  op.n = n;
  op.row16 = row_bytes / 16;
  op.parts = (int)std::max<int64_t>(1, std::min<int64_t>(8, op.row16 / 128));
  op.ticket = c->ll_counters + (c->ll_ctr_next++ % kLLCounters);
  op.counter = c->ll_counters + (c->ll_ctr_next++ % kLLCounters);
  op.go = c->ll_counters + kLLCounters + (cop.slot % kLLCounters);
  op.go_gen = cop.gen;
  op.error = c->ll_error;
  for (int d = 0; d < n; d++) {
    op.d[d].lo = (int64_t)rd[d];
    op.d[d].hi = (int64_t)(rd[d] + rcounts[d]);
  }
  op.d[me].seg = (const char*)expert_rows + sd[me] * (size_t)row_bytes;
  op.d[me].my_done = &flags_of(c, me)->done[cop.slot];
  op.d[me].my_done_gen = cop.gen;
  c->combine_stream = s;
  c->combine_fused = true;
  c->in_combine = true;
  r = iccl_group_start(c);
  for (int kk = 1; kk < n && r == ICCL_SUCCESS; kk++) {
    const int to = (me + kk) % n, from = (me - kk + n) % n;
    if (rcounts[from]) r = iccl_recv(c, out, rcounts[from] * (size_t)row_bytes, from, s, nullptr);
    if (!r && scounts[to])
      r = iccl_send(c, (const char*)expert_rows + sd[to] * (size_t)row_bytes, scounts[to] * (size_t)row_bytes, to, s,
                    nullptr);
  }
  iccl_result_t r2 = iccl_group_end(c);
  if (!r) r = r2;
  if (!r && c->combine_fused) r = launch_fused_combine(c, s, {});  // no remote recv on s: the self segment
  c->combine_fused = false;
  c->in_combine = false;
  return r;
}

iccl_result_t iccl_alltoall(iccl_comm_t c, const void* sbuf, void* rbuf, size_t bytes_per_pair, cudaStream_t s) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_RETURN_IF(c->nranks < 2, ICCL_ERR_GROUP_TOO_SMALL, "alltoall needs >= 2 ranks (SPEC.md:429)");
  if (bytes_per_pair == 0) return ICCL_SUCCESS;  // immediate completion
  std::vector<size_t> cnt(c->nranks, bytes_per_pair), disp(c->nranks);
  for (int i = 0; i < c->nranks; i++) disp[i] = i * bytes_per_pair;
  return iccl_alltoallv(c, sbuf, cnt.data(), disp.data(), rbuf, cnt.data(), disp.data(), 1, s);
}

iccl_result_t iccl_req_test(iccl_comm_t c, iccl_req_t req, int* done) {
  if (!c || !done) return ICCL_ERR_INVALID_ARGUMENT;
  uint32_t slot = (uint32_t)(req >> 32), gen = (uint32_t)req;
  ICCL_RETURN_IF(slot >= (uint32_t)kSlots, ICCL_ERR_UNKNOWN_WR, "bad request handle");
  *done = cyc_geq(__atomic_load_n(&flags_of(c, c->rank)->done[slot], __ATOMIC_ACQUIRE), gen) ? 1 : 0;
  int ae = c->async_err.load();
  if (!*done && ae != ICCL_SUCCESS) {
    set_last_error(c->async_msg);
    return (iccl_result_t)ae;
  }
  return ICCL_SUCCESS;
}

iccl_result_t iccl_req_wait(iccl_comm_t c, iccl_req_t req, int64_t timeout_us) {
  uint64_t t0 = now_ns();
  for (;;) {
    int done = 0;
    iccl_result_t r = iccl_req_test(c, req, &done);
    if (r) return r;
    if (done) return ICCL_SUCCESS;
    if (timeout_us >= 0 && (now_ns() - t0) > (uint64_t)timeout_us * 1000ull) {
      set_last_error("request wait timed out");
      return ICCL_ERR_TIMEOUT;
    }
    sched_yield();
  }
}

iccl_result_t iccl_req_state(iccl_comm_t c, iccl_req_t req, iccl_xfer_state_t* st) {
  if (!c || !st) return ICCL_ERR_INVALID_ARGUMENT;
  int done = 0;
  iccl_result_t r = iccl_req_test(c, req, &done);
  if (r) return r;
  // Six pointers from the record the sender's proxy
  // publishes.  Zero-copy: posted == transmitted on the sender, and the
  // receiver's received == done (bytes land in the user buffer directly), so
  // the six collapse to posted / done, with acked == done.
  memset(st, 0, sizeof(*st));
  uint32_t slot = (uint32_t)(req >> 32), gen = (uint32_t)req;
  const XferPub& p = flags_of(c, c->rank)->pub[slot];
  bool have = __atomic_load_n(&p.gen, __ATOMIC_ACQUIRE) == gen;
  st->role = p.kind;
  st->total_chunks = have ? p.total : -1;
  st->bytes = have ? p.bytes : 0;
  int posted = have ? p.posted : 0, dn = have ? p.done : 0;
  if (done && have) posted = dn = p.total;
  st->posted = st->transmitted = posted;
  st->acked = dn;
  st->r_posted = have ? p.total : 0;
  st->received = st->done = dn;
  st->active_path = have ? p.path : 0;
  st->switches = have ? p.switches : 0;
  return ICCL_SUCCESS;
}

// The directed path rank -> peer is switched for whichever side issues its
// next transfer (the pair's shared state); transfers this rank has in flight
// on the pair move at the receiver's breakpoint (switch_qp).
iccl_result_t iccl_path_switch(iccl_comm_t c, int peer, int to) {
  if (!c || peer < 0 || peer >= c->nranks || (to != 0 && to != 1)) return ICCL_ERR_INVALID_ARGUMENT;
  pair_of(c, c->rank, peer).active_path.store(to);
  route_update(pair_of(c, c->rank, peer));
  c->path_req[2 * peer + 0].store(to);
  if (peer == c->rank) c->path_req[2 * peer + 1].store(to);  // a self pair is also issued by its pull side
  c->qcv.notify_one();
  return ICCL_SUCCESS;
}

iccl_result_t iccl_path_active(iccl_comm_t c, int peer, int* path) {
  if (!c || !path || peer < 0 || peer >= c->nranks) return ICCL_ERR_INVALID_ARGUMENT;
  *path = pair_of(c, c->rank, peer).active_path.load();
  return ICCL_SUCCESS;
}

iccl_result_t iccl_fault_set(iccl_comm_t c, const iccl_fault_t* f, int n) {
  if (!c || (n > 0 && !f) || n < 0) return ICCL_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; i++)
    ICCL_RETURN_IF(f[i].src < 0 || f[i].src >= c->nranks || f[i].dst < 0 || f[i].dst >= c->nranks,
                   ICCL_ERR_INVALID_ARGUMENT, "fault names an unknown path (UnknownPort)");
  std::vector<std::pair<int, int>> touched;
  {
    std::lock_guard<std::mutex> g(c->fault_mu);
    // the pairs a script names are armed for failover on both endpoints: their
    // ops (every size class) take the chunked path where the gates apply
    for (const Fault& old : c->faults) {
      pair_of(c, old.f.src, old.f.dst).faults_armed.fetch_sub(1);
      touched.emplace_back(old.f.src, old.f.dst);
    }
    c->faults.clear();
    int timed = 0;
    for (int i = 0; i < n; i++) {
      c->faults.push_back(Fault{f[i], false});
      timed += f[i].trigger_kind == 0 && (f[i].src == c->rank || f[i].dst == c->rank);
      pair_of(c, f[i].src, f[i].dst).faults_armed.fetch_add(1);
      touched.emplace_back(f[i].src, f[i].dst);
    }
    c->faults_t0 = now_ns();
    c->time_faults_pending.store(timed, std::memory_order_release);
    for (auto& chn : c->ch) chn.fault_seq_base = chn.dir == 0 ? c->pair_sends[chn.peer] : c->pair_recvs[chn.peer];
  }
  for (auto& t : touched) route_update(pair_of(c, t.first, t.second));
  // the streams an armed transfer of these pairs uses, created now: creating
  // a stream while the device is busy took up to 72 ms (profiles/r02/raw/
  // x_ac5_debug_n2.log), which would land inside the first armed issue
  for (int i = 0; i < n; i++)
    for (Channel& chn : c->ch)
      if (chn.src == f[i].src && chn.dst == f[i].dst) {
        cudaStream_t s = nullptr;
        iccl_result_t r = backup_stream(c, chn, &s);
        if (!r) r = prog_stream(c, chn, &s);
        if (r) return r;
      }
  return ICCL_SUCCESS;
}

iccl_result_t iccl_switch_events(iccl_comm_t c, iccl_switch_event_t* ev, int max, int* n) {
  if (!c || !n || max < 0) return ICCL_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> g(c->mon_mu);
  int k = 0;
  while (k < max && !c->sw_events.empty()) {
    ev[k++] = c->sw_events.front();
    c->sw_events.pop_front();
  }
  *n = k;
  return ICCL_SUCCESS;
}

iccl_result_t iccl_gather_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                               int ctas, cudaStream_t s) {
  if ((n_rows > 0 && (!src || !dst || !idx)) || n_rows < 0 || row_bytes <= 0) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_CHECK_CUDA(launch_gather_rows(src, dst, idx, n_rows, row_bytes, ctas > 0 ? ctas : 148 * 8, s));
  return ICCL_SUCCESS;
}

iccl_result_t iccl_scatter_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                                int ctas, cudaStream_t s) {
  if ((n_rows > 0 && (!src || !dst || !idx)) || n_rows < 0 || row_bytes <= 0) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_CHECK_CUDA(launch_scatter_rows(src, dst, idx, n_rows, row_bytes, ctas > 0 ? ctas : 148 * 8, s));
  return ICCL_SUCCESS;
}

iccl_result_t iccl_expand_rows(const void* src, void* dst, const int64_t* pos, int64_t n_src, int32_t k,
                               int64_t row_bytes, int ctas, cudaStream_t s) {
  if ((n_src > 0 && k > 0 && (!src || !dst || !pos)) || n_src < 0 || k < 0 || row_bytes <= 0)
    return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_CHECK_CUDA(launch_expand_rows(src, dst, pos, n_src, k, row_bytes, ctas, s));
  return ICCL_SUCCESS;
}

iccl_result_t iccl_copy_sm(const void* src, void* dst, size_t bytes, int ctas, cudaStream_t s) {
  if (bytes > 0 && (!src || !dst)) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_CHECK_CUDA(launch_copy(src, dst, bytes, ctas > 0 ? ctas : 16, nullptr, s));
  return ICCL_SUCCESS;
}

iccl_result_t iccl_comm_set_chunk_bytes(iccl_comm_t c, uint64_t chunk_bytes) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_RETURN_IF(chunk_bytes < 4096 || (chunk_bytes & 15), ICCL_ERR_INVALID_CONFIG,
                 "chunk_bytes must be >= 4096 and a multiple of 16");
  c->cfg.chunk_bytes = chunk_bytes;  // read by the API thread only (rzv_build)
  return ICCL_SUCCESS;
}

iccl_result_t iccl_monitor_config(iccl_comm_t c, int enabled, int window) {
  if (!c || window < 1) return ICCL_ERR_INVALID_ARGUMENT;
  c->monitor_enabled.store(enabled ? 1 : 0);
  c->cfg.monitor_window = window;
  return ICCL_SUCCESS;
}

// ---- self-test hooks: the shared-memory protocols on plain host memory ----
size_t iccl_selftest_pair_bytes(void) { return sizeof(PairState); }
size_t iccl_selftest_rzv_bytes(void) { return sizeof(RzvEntry); }

int iccl_selftest_route_small(void* pair, int side) { return route_small(*(PairState*)pair, side & 1) ? 1 : 0; }

void iccl_selftest_route_arm(void* pair, int faults_delta, int active_path) {
  PairState& ps = *(PairState*)pair;
  ps.faults_armed.fetch_add(faults_delta);
  if (active_path >= 0) ps.active_path.store(active_path);
  route_update(ps);
}

int iccl_selftest_rzv_post(void* entry, int kind, uint64_t k, uint64_t bytes, uint64_t* other_bytes) {
  RzvEntry& e = *(RzvEntry*)entry;
  while (!rzv_free(e, k)) sched_yield();
  e.side[kind & 1].bytes = bytes;
  e.side[kind & 1].slot = (uint32_t)(k % kSlots);
  e.side[kind & 1].gen = (uint32_t)(k + 1);
  RzvSide snap[2];
  if (!rzv_arrive(e, k, snap)) return 0;
  if (other_bytes) *other_bytes = snap[(kind & 1) ^ 1].bytes;
  return snap[0].gen == snap[1].gen ? 1 : -1;  // both halves belong to op k
}

// CPU self-test of the armed-transfer failover protocol (see the header):
// the watchdog's own pass (armed_progress) drives one transfer of a
// communicator whose control block lives in plain host memory, while a host
// thread plays the device — the primary attempt's stream (gate waits,
// chunk copies, prog / p_fin / go / ns / done / fin words) and K9's
// controller (decision, CTS probe, suffix copy with one K4 stamp per chunk).
int iccl_selftest_failover(int scenario, int nchunks, int fault_chunk, uint64_t delta_us, int64_t* out) {
  if (nchunks < 1 || nchunks > 256 || !out) return -1;
  iccl_comm* c = new iccl_comm();
  c->rank = 0;
  c->nranks = 2;
  c->cfg.delta_us = delta_us;
  c->cfg.probe_period_us = std::max<uint64_t>(1, delta_us / 2);
  c->cfg.chunk_bytes = 1 << 20;
  c->monitor_enabled = 1;
  c->flags = (RankFlags*)calloc(2, sizeof(RankFlags));
  c->rings = (RzvRing*)calloc(4, sizeof(RzvRing));
  c->armed_words = (ArmedWords*)calloc(kArmedSlots, sizeof(ArmedWords));
  c->stamps = (KernelStamp*)calloc(kStampSlots, sizeof(KernelStamp));
  c->gate_words = (volatile uint32_t*)calloc(kGateWords, 4);
  c->gate_closed.assign(kGateWords, 0);
  c->armed_used.assign(kArmedSlots, 0);
  c->ch.resize(4);
  for (int p = 0; p < 2; p++)
    for (int d = 0; d < 2; d++) {
      Channel& h = c->ch[2 * p + d];
      h.peer = p;
      h.dir = d;
      h.src = d == 0 ? 0 : p;
      h.dst = d == 0 ? p : 0;
    }
  Channel& chn = c->ch[2];  // pushes 0 -> 1
  ArmedWords* w = &c->armed_words[0];
  w->resume = (uint32_t)nchunks;
  w->ns = 1;
  const bool dead = scenario == 2 || scenario == 3;
  if (dead) {  // chunk-triggered Down of the primary (fired at issue, like fire_chunk_faults)
    chn.fault[0].down = true;
    chn.fault[0].gate = alloc_gate(c);
    chn.fault[0].down_at = now_ns();
  }
  if (scenario == 3) {  // the backup path is Down as well
    chn.fault[1].down = true;
    chn.fault[1].gate = alloc_gate(c);
    chn.fault[1].down_at = now_ns();
  }
  volatile uint32_t* pgate = dead ? &c->gate_words[chn.fault[0].gate] : nullptr;
  volatile uint32_t* bgate = scenario == 3 ? &c->gate_words[chn.fault[1].gate] : nullptr;
  w->pgate = dead ? (uint32_t)chn.fault[0].gate + 1 : 0;  // as armed_launch publishes them for K9a
  w->bgate = scenario == 3 ? (uint32_t)chn.fault[1].gate + 1 : 0;
  Xfer x;
  x.armed = true;
  x.aw = 0;
  x.src_rank = 0;
  x.dst_rank = 1;
  x.chan = 2;
  x.s_slot = x.r_ready_slot = x.r_done_slot = 0;
  x.s_gen = x.r_ready_gen = x.r_done_gen = 1;
  x.nchunks = nchunks;
  x.chunk = 1 << 20;
  x.bytes = (size_t)nchunks << 20;
  x.next_issue = nchunks;
  x.rec.resize(nchunks);
  x.bstamp.resize(nchunks);
  for (int k = 0; k < nchunks; k++) x.bstamp[k] = k;
  x.last_progress = x.t_obs = now_ns();
  c->armed_used[0] = 1;
  c->pending_xfers = 1;
  chn.armed.push_back(std::move(x));
  const uint64_t delta = delta_us * 1000ull;
  std::atomic<bool> quit{false};
  auto ld = [](volatile uint32_t* p) { return __atomic_load_n((uint32_t*)p, __ATOMIC_ACQUIRE); };
  auto st = [](volatile uint32_t* p, uint32_t v) { __atomic_store_n((uint32_t*)p, v, __ATOMIC_SEQ_CST); };
  auto nap = [] { std::this_thread::sleep_for(std::chrono::microseconds(20)); };
  // the primary attempt's stream
  std::thread primary([&] {
    if (scenario == 4) std::this_thread::sleep_for(std::chrono::nanoseconds(3 * delta));  // upstream stall
    st(&c->flags[0].ready[0], 1);
    st(&c->flags[1].ready[0], 1);
    for (int k = 0; k < nchunks && !quit; k++) {
      if (dead && k == fault_chunk)
        while (ld(pgate) == 0 && !quit) nap();
      if (scenario == 1 && k == fault_chunk) std::this_thread::sleep_for(std::chrono::nanoseconds(3 * delta));
      std::this_thread::sleep_for(std::chrono::microseconds(30));  // the chunk's copy
      st(&w->prog, (uint32_t)(k + 1));
    }
    st(&w->p_fin, 1);
    st(&w->go, 1);
    while (ld(&w->ns) == 0 && !quit) nap();
    st(&c->flags[1].done[0], 1);
    st(&c->flags[0].done[0], 1);
    st(&w->fin, 1);
  });
  // K9 on the backup stream
  std::thread backup([&] {
    while (ld(&w->go) == 0 && !quit) nap();
    uint32_t dec = kDecNone;
    bool probed = false;
    while (dec == kDecNone && !quit) {
      const uint32_t ctl = ld(&w->ctl);
      if (ctl == kCtlSwitch) dec = kDecCopy;
      else if (ctl == kCtlAbort) dec = kDecExit;
      else if (ld(&w->p_fin)) dec = ld(&w->ctl) == kCtlSwitch ? kDecCopy : kDecExit;
      else if (ctl == kCtlProbe && !probed &&
               (ld(&w->pgate) == 0 || ld(&c->gate_words[ld(&w->pgate) - 1]) != 0)) {
        st(&w->probe_done, 1);
        probed = true;
      } else {
        nap();
      }
    }
    st(&w->dec, dec);
    if (dec == kDecCopy) {
      while (bgate && ld(bgate) == 0 && ld(&w->ctl) != kCtlAbort && !quit) nap();
      if (!bgate || ld(bgate) != 0)
        for (uint32_t k = ld(&w->resume); k < (uint32_t)nchunks; k++) {
          const unsigned long long t1 = now_ns();
          std::this_thread::sleep_for(std::chrono::microseconds(40));
          __atomic_store_n(&c->stamps[k].t1, t1, __ATOMIC_RELEASE);
          __atomic_store_n(&c->stamps[k].t2, (unsigned long long)now_ns(), __ATOMIC_RELEASE);
        }
    }
    st(&w->b_fin, 1);
  });
  // the watchdog thread's pass, until the transfer retires (or fails)
  const uint64_t t0 = now_ns();
  int rc = 0;
  while (!chn.armed.empty()) {
    armed_progress(c, chn);
    if (c->async_err.load() != ICCL_SUCCESS) break;
    if (now_ns() - t0 > 20ull * 1000000000ull) {
      rc = 1;  // timed out
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(5));
  }
  int switched = 0;
  for (auto& e : c->sw_events) switched += e.to_path == 1 && e.trigger == 1;
  out[0] = switched;
  out[1] = switched ? (int64_t)ld(&w->resume) : -1;
  out[2] = c->flags[0].pub[0].done;
  out[3] = c->flags[0].pub[0].total;
  out[4] = ld(&c->flags[0].done[0]) == 1 && ld(&c->flags[1].done[0]) == 1;
  out[5] = (int64_t)c->mon.size();
  out[6] = ld(&w->probe_done);
  out[7] = c->async_err.load();
  // release whatever is still parked (both paths dead), then tear down
  quit = true;
  st(&w->ctl, kCtlAbort);
  st(&w->ns, 1);
  st(&w->go, 1);
  for (int g = 0; g < kGateWords; g++) st(&c->gate_words[g], 1);
  primary.join();
  backup.join();
  free(c->flags);
  free(c->rings);
  free(c->armed_words);
  free(c->stamps);
  free((void*)c->gate_words);
  c->flags = nullptr;
  delete c;
  return rc;
}

iccl_result_t iccl_monitor_read(iccl_comm_t c, iccl_mon_rec_t* recs, int max, int* n) {
  if (!c || !n || max < 0 || (max > 0 && !recs)) return ICCL_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> g(c->mon_mu);
  int k = 0;
  while (k < max && !c->mon.empty()) {
    recs[k++] = c->mon.front();
    c->mon.pop_front();
  }
  *n = k;
  return ICCL_SUCCESS;
}

}  // extern "C"
