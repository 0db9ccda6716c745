/*
 * iccl_b200.h — C ABI of the B200-native ICCL P2P hot path.
 *
 * This is the drop-in boundary.  The reference's own
 * boundary is a Python library API specified in SPEC.md (verbs / transport /
 * monitor / collectives, no code shipped) and, for the paper's real ICCL, the
 * NCCL C API of an NCCL 2.21.5 fork.  The entry points
 * below are NCCL-shaped (unique id, init-rank, stream-ordered send/recv,
 * group start/end) and carry the SPEC's extra surface (six-pointer transfer
 * state, path switch, fault script, window monitor).  Every function returns
 * an iccl_result_t; 0 is success and the other codes mirror the SPEC-named
 * exceptions.  No torch type appears here: buffers are device pointers and
 * byte counts, streams are cudaStream_t.  Each declaration cites the
 * reference interface it replaces.
 *
 * Threading: one API thread per communicator (as NCCL).  The library runs
 * one proxy thread per communicator that owns every copy-engine / kernel
 * submission; ordering with user work goes only through stream memory
 * operations on the caller's stream (no host callbacks).
 */
#ifndef ICCL_B200_H_
#define ICCL_B200_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICCL_B200_VERSION 100
#define ICCL_UNIQUE_ID_BYTES 128

/* Result codes.  Names after the SPEC exceptions they surface as. */
typedef enum {
  ICCL_SUCCESS = 0,
  ICCL_ERR_INVALID_ARGUMENT = 1,
  ICCL_ERR_CUDA = 2,
  ICCL_ERR_SYSTEM = 3,
  ICCL_ERR_QP_IN_ERROR_STATE = 4,    /* QpInErrorState      */
  ICCL_ERR_UNREGISTERED_REGION = 5,  /* UnregisteredRegion      */
  ICCL_ERR_ZERO_LENGTH_MESSAGE = 6,  /* ZeroLengthMessage  */
  ICCL_ERR_CONNECTION_FAILED = 7,    /* ConnectionFailed  */
  ICCL_ERR_UNKNOWN_WR = 8,           /* UnknownWr      */
  ICCL_ERR_TARGET_QP_DEAD = 9,       /* TargetQpDead      */
  ICCL_ERR_NON_POSITIVE_DURATION = 10, /* NonPositiveDuration SPEC.md:326    */
  ICCL_ERR_WINDOW_NOT_FULL = 11,     /* WindowNotFull      */
  ICCL_ERR_GROUP_TOO_SMALL = 12,     /* GroupTooSmall      */
  ICCL_ERR_NO_SM_AVAILABLE = 13,     /* NoSmAvailable      */
  ICCL_ERR_INVALID_CONFIG = 14,      /* InvalidConfig      */
  ICCL_ERR_CONFIG = 15,              /* ConfigError      */
  ICCL_ERR_SIZE_MISMATCH = 16,       /* send / recv byte counts differ        */
  ICCL_ERR_TIMEOUT = 17,             /* iccl_req_wait deadline                */
  ICCL_ERR_IN_PROGRESS = 18,         /* iccl_req_test: not complete yet       */
  ICCL_ERR_ABORTED = 19,             /* communicator aborted                  */
  ICCL_ERR_NUM_CODES
} iccl_result_t;

typedef struct iccl_comm* iccl_comm_t;

typedef struct {
  char internal[ICCL_UNIQUE_ID_BYTES];
} iccl_unique_id_t;

/* Transport and path ids. */
enum { ICCL_TRANSPORT_AUTO = 0, ICCL_TRANSPORT_CE = 1, ICCL_TRANSPORT_SM = 2 };
enum { ICCL_PATH_PRIMARY = 0, ICCL_PATH_BACKUP = 1 };
enum { ICCL_BACKUP_SM = 0, ICCL_BACKUP_RELAY = 1 };

/* Configuration (Table 5), every field
 * overridable by an ICCL_* environment variable in iccl_config_init. */
typedef struct {
  uint64_t chunk_bytes;       /* ICCL_CHUNK_BYTES     chunk size, SPEC.md:282 (4 MiB)            */
  int32_t streams_per_peer;   /* ICCL_QP_NUM          copy streams per peer: Table 5 "QP number" */
  int32_t sm_cap;             /* ICCL_SM_CAP          CTAs of the SM copy kernel: "channels"     */
  int32_t window;             /* ICCL_WINDOW_CHUNKS   chunks in flight per peer (posted-acked)   */
  int32_t monitor_window;     /* ICCL_MONITOR_WINDOW  W, Table 5 "window size 8"                 */
  int32_t monitor_enabled;    /* ICCL_MONITOR         1 = record chunk WR/WC stamps              */
  int32_t backup_kind;        /* ICCL_BACKUP          ICCL_BACKUP_SM | ICCL_BACKUP_RELAY         */
  int32_t transport;          /* ICCL_TRANSPORT       ICCL_TRANSPORT_*                           */
  int32_t timeout_exponent;   /* ICCL_IB_TIMEOUT      retry timeout exponent   */
  int32_t retry_count;        /* ICCL_IB_RETRY_CNT                                               */
  uint64_t delta_us;          /* ICCL_DELTA_US        watchdog delta; 0 = retry_timeout derived  */
  uint64_t probe_period_us;   /* ICCL_PROBE_PERIOD_US monitor_failed_link period */
  uint64_t sm_small_bytes;    /* ICCL_SM_SMALL_BYTES  AUTO: messages <= this use the SM path    */
  int32_t proxy_cpu;          /* ICCL_PROXY_CPU       core to pin the proxy to, -1 = none        */
  int32_t relay_slot_mib;     /* ICCL_RELAY_SLOT_MIB  relay backup: staging slot per source (x2)  */
  int32_t direct_max_kib;     /* ICCL_DIRECT_MAX_KIB  AUTO: larger-than-LL messages up to this go
                                                       the direct SM path (K6); 0 = off              */
  int32_t reserved[5];
} iccl_config_t;

/* Six progress pointers of one transfer (Fig. 6). */
typedef struct {
  int32_t role;             /* 0 sender, 1 receiver */
  int32_t total_chunks;
  int32_t posted, transmitted, acked; /* sender   */
  int32_t r_posted, received, done;   /* receiver */
  int32_t active_path;      /* ICCL_PATH_* */
  int32_t switches;
  uint64_t bytes;
} iccl_xfer_state_t;

/* Fault script entry: the directed copy path src->dst
 * goes Down or Up when the trigger fires.  trigger_kind 0: t_us after
 * iccl_fault_set; 1: when the sender issues chunk `chunk` of its
 * `op_index`-th send to dst (counted from iccl_fault_set). */
typedef struct {
  int32_t src, dst, path, up;
  int32_t trigger_kind;
  int32_t op_index;
  int64_t chunk;
  uint64_t t_us;
} iccl_fault_t;

/* Monitor record: one per chunk completion, the WR/WC pair of SPEC.md:304-307. */
typedef struct {
  uint64_t t1_ns;   /* WR post (CE path: proxy issue, CLOCK_MONOTONIC; SM path: %globaltimer mapped) */
  uint64_t t2_ns;   /* WC (CE path: proxy observes the device-written flag; SM path: kernel stamp)  */
  uint64_t bytes;
  int32_t peer;
  int32_t path;     /* ICCL_PATH_* */
  int32_t chunk;
  int32_t dir;      /* 0: pushed by this rank to peer, 1: pulled by this rank from peer */
  uint64_t op_seq;
} iccl_mon_rec_t;

/* Switch / failover event (transport event log). */
typedef struct {
  uint64_t t_ns;
  int32_t peer;
  int32_t to_path;
  int32_t resume_chunk;  /* breakpoint = receiver done */
  int32_t trigger;       /* 0 api, 1 watchdog+probe fail, 2 probe ok (switch back) */
  uint64_t detect_ns;    /* injection -> switch, when known */
} iccl_switch_event_t;

/* ---- library ------------------------------------------------------------ */
const char* iccl_get_error_string(iccl_result_t r);
/* Last detailed message of the calling thread (or the comm's async error). */
const char* iccl_get_last_error(void);
int iccl_get_version(void);

/* Defaults + ICCL_* env overrides.  Replaces RunConfig defaults. */
iccl_result_t iccl_config_init(iccl_config_t* cfg);
iccl_result_t iccl_config_validate(const iccl_config_t* cfg);

/* ---- communicator (CommGroup; ncclGetUniqueId/ncclCommInitRank) */
iccl_result_t iccl_get_unique_id(iccl_unique_id_t* uid);
iccl_result_t iccl_comm_init_rank(iccl_comm_t* comm, int nranks, iccl_unique_id_t uid, int rank, int cuda_dev,
                                  const iccl_config_t* cfg);
iccl_result_t iccl_comm_destroy(iccl_comm_t comm);
iccl_result_t iccl_comm_abort(iccl_comm_t comm);
iccl_result_t iccl_comm_count(iccl_comm_t comm, int* nranks);
iccl_result_t iccl_comm_user_rank(iccl_comm_t comm, int* rank);
iccl_result_t iccl_comm_get_async_error(iccl_comm_t comm, iccl_result_t* err);
/* opCount of every rank, read from the shared control block. */
iccl_result_t iccl_comm_op_counts(iccl_comm_t comm, uint64_t* counts, int n);

/* Counters of the work this rank issued (SURVEY.md §5 metrics): SM kernels
 * launched (K1 backup copies, K5 LL, K6 direct) and their CTAs, copy-engine
 * copies, payload bytes, and how the rendezvous went (pulls, CTS timeouts). */
typedef struct {
  uint64_t kernels_launched;
  uint64_t copies_issued;
  uint64_t bytes_issued;
  uint64_t ctas_launched;  /* CTAs of those kernels (the "SMs used" of the SM paths) */
  uint64_t pulls_issued;   /* transfers this rank issued as the receiver (it reached the rendezvous second) */
  uint64_t cts_timeouts;   /* sends that stopped waiting for the receiver's half and posted first */
  uint64_t pending_xfers;  /* transfers this rank issued that the proxy / watchdog has not retired yet
                              (kernel-path ops until their monitor record is emitted) */
  uint64_t reserved[1];
} iccl_stats_t;
iccl_result_t iccl_comm_stats(iccl_comm_t comm, iccl_stats_t* stats);

/* ---- memory registration (MemoryRegion; User Buffer Registration PAPER.md:410-412) */
iccl_result_t iccl_register(iccl_comm_t comm, void* ptr, size_t bytes, uint64_t* handle);
iccl_result_t iccl_deregister(iccl_comm_t comm, uint64_t handle);

/* ---- P2P (send_message / send_recv SPEC.md:228-236, 436-444; ncclSend/ncclRecv) */
typedef uint64_t iccl_req_t;
iccl_result_t iccl_send(iccl_comm_t comm, const void* buf, size_t bytes, int peer, cudaStream_t stream,
                        iccl_req_t* req);
iccl_result_t iccl_recv(iccl_comm_t comm, void* buf, size_t bytes, int peer, cudaStream_t stream,
                        iccl_req_t* req);
iccl_result_t iccl_group_start(iccl_comm_t comm);
iccl_result_t iccl_group_end(iccl_comm_t comm);

/* alltoall and the torch-shaped alltoallv.
 * Counts / displacements are in elements of elem_bytes. */
iccl_result_t iccl_alltoall(iccl_comm_t comm, const void* sbuf, void* rbuf, size_t bytes_per_pair,
                            cudaStream_t stream);
iccl_result_t iccl_alltoallv(iccl_comm_t comm, const void* sbuf, const size_t* scounts, const size_t* sdispls,
                             void* rbuf, const size_t* rcounts, const size_t* rdispls, size_t elem_bytes,
                             cudaStream_t stream);

/* ---- requests: host-side completion of an isend/irecv ------------------- */
iccl_result_t iccl_req_test(iccl_comm_t comm, iccl_req_t req, int* done);
iccl_result_t iccl_req_wait(iccl_comm_t comm, iccl_req_t req, int64_t timeout_us);
iccl_result_t iccl_req_state(iccl_comm_t comm, iccl_req_t req, iccl_xfer_state_t* state);

/* ---- primary-backup paths (switch_qp SPEC.md:255-263, monitor_failed_link 264-273) */
iccl_result_t iccl_path_switch(iccl_comm_t comm, int peer, int to_path);
iccl_result_t iccl_path_active(iccl_comm_t comm, int peer, int* path);
iccl_result_t iccl_fault_set(iccl_comm_t comm, const iccl_fault_t* faults, int n);
iccl_result_t iccl_switch_events(iccl_comm_t comm, iccl_switch_event_t* ev, int max, int* n);

/* Chunk size (SPEC.md:228-236's chunk_size, ICCL_CHUNK_BYTES) of the transfers
 * this rank issues from now on; same validation as iccl_config_t.chunk_bytes. */
iccl_result_t iccl_comm_set_chunk_bytes(iccl_comm_t comm, uint64_t chunk_bytes);

/* ---- window monitor ------------------------------------ */
iccl_result_t iccl_monitor_config(iccl_comm_t comm, int enabled, int window);
iccl_result_t iccl_monitor_read(iccl_comm_t comm, iccl_mon_rec_t* recs, int max, int* n);

/* ---- fused MoE dispatch (K8) ---------------------------------------------
 * Collective over the communicator, stream-ordered on s.  Result identical to
 *   iccl_expand_rows(tokens -> packed, pos, n_tokens, k)   (packed row pos[t*k+j] = token t)
 *   iccl_alltoallv(packed, scounts, sdispls = prefix(scounts),
 *                  rbuf, rcounts, rdispls = prefix(rcounts), row_bytes)
 * but in one kernel with no packed buffer: every routed row is stored
 * straight into the receive buffer of the rank owning its packed position
 * (NVLink stores into an IPC mapping; PAPER.md:214-217's zero staging).
 * Replaces the dispatch pack + alltoall of SPEC.md:427-444 / SURVEY.md §2.4.
 * Pairs armed for failover take the unfused form (same result).  k <= 32,
 * row_bytes a multiple of 16, tokens / rbuf 16-byte aligned. */
iccl_result_t iccl_dispatch_rows(iccl_comm_t comm, const void* tokens, int64_t n_tokens, int32_t k,
                                 const int64_t* pos, const size_t* scounts, void* rbuf, const size_t* rcounts,
                                 int64_t row_bytes, cudaStream_t s);

/* ---- fused MoE combine (K10) --------------------------------------------
 * Collective over the communicator, the reverse of iccl_dispatch_rows.
 * Result identical to
 *   iccl_alltoallv(expert_rows, scounts, prefix(scounts), packed, rcounts, prefix(rcounts), row_bytes)
 *   iccl_scatter_rows(packed -> out, idx = order)      (out row order[r] = packed row r)
 * but the receiving rank's kernel loads its rows straight from the senders'
 * expert_rows over NVLink and stores them at their out rows, with no packed
 * buffer.  scounts: rows this rank returns to each rank (grouped by rank in
 * expert_rows); rcounts: rows it gets back from each (the packed layout that
 * `order` indexes).  Pairs armed for failover take the unfused form. */
iccl_result_t iccl_combine_rows(iccl_comm_t comm, const void* expert_rows, const size_t* scounts, void* out,
                                const int64_t* order, const size_t* rcounts, int64_t row_bytes, cudaStream_t s);

/* ---- MoE pack / unpack permutation kernels (K2 / K3), stream-ordered ----
 * dst row i <- src row idx[i] (gather, dispatch pack); dst row idx[i] <- src
 * row i (scatter, combine unpack).  idx is a device int64 array; rows are
 * 16-byte multiples.  ctas <= 0 uses the full GPU. */
iccl_result_t iccl_gather_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                               int ctas, cudaStream_t stream);
iccl_result_t iccl_scatter_rows(const void* src, void* dst, const int64_t* idx, int64_t n_rows, int64_t row_bytes,
                                int ctas, cudaStream_t stream);
/* Dispatch pack in expand form: dst row pos[t*k + j] <- src row t for every
 * source row t < n_src_rows and j < k (each source row read once, written k
 * times; pos is the inverse of the gather index).  Same result as
 * iccl_gather_rows with idx[pos[t*k + j]] = t. */
iccl_result_t iccl_expand_rows(const void* src, void* dst, const int64_t* pos, int64_t n_src_rows, int32_t k,
                               int64_t row_bytes, int ctas, cudaStream_t stream);
/* SM copy kernel (K1) on its own, for measurement and for callers that want
 * the SM path explicitly: copies bytes src -> dst with <= ctas CTAs. */
iccl_result_t iccl_copy_sm(const void* src, void* dst, size_t bytes, int ctas, cudaStream_t stream);

/* ---- pure host arithmetic (no device needed; the product's own formulas) */
/* retry_timeout: 4.096 us * 2^exp * (retry + 1), in ns. */
uint64_t iccl_retry_timeout_ns(int timeout_exponent, int retry_count);
/* switch_qp pointer retreat: received := done; acked := done;
 * posted := transmitted := acked.  Returns the resume chunk. */
int iccl_switch_pointers(iccl_xfer_state_t* sender, iccl_xfer_state_t* receiver);
/* per-message and window throughput in bytes/s; records in completion order. */
iccl_result_t iccl_per_message_throughput(const iccl_mon_rec_t* rec, double* bytes_per_s);
iccl_result_t iccl_window_throughput(const iccl_mon_rec_t* recs, int n, int window, double* bytes_per_s);
/* sample_series: out[k] for k = 0 .. n-window; *n_out = max(0, n - window + 1). */
iccl_result_t iccl_sample_series(const iccl_mon_rec_t* recs, int n, int window, double* out_bps,
                                 uint64_t* out_t_ns, int* n_out);
/* detect_lagging_rank: *rank = -1 for None. */
iccl_result_t iccl_detect_lagging_rank(const uint64_t* op_counts, int n, uint64_t threshold, int* rank);

/* ---- self-test hooks (no device needed) ----------------------------------
 * The two shared-memory protocols of the control block, run on caller-owned
 * host memory so CPU tests can drive them from several processes:
 * - small-op routing (LL vs rendezvous) of one ordered pair: both sides must
 *   route the pair's q-th small op alike while the pair is armed / disarmed
 *   concurrently (fault scripts, switch_qp) — pair memory of
 *   iccl_selftest_pair_bytes(), zero-initialised;
 * - the rendezvous entry of one ordered pair (SPEC.md:194's RTS / CTS): the
 *   side arriving second claims op k and sees both halves, entries reused
 *   every 1024 ops — entry memory of iccl_selftest_rzv_bytes(), zeroed.
 * iccl_selftest_rzv_post returns 0 (posted first), 1 (second: claimed, the
 * other half's byte count in *other_bytes) or -1 (halves of different ops). */
size_t iccl_selftest_pair_bytes(void);
size_t iccl_selftest_rzv_bytes(void);
int iccl_selftest_route_small(void* pair, int side);
void iccl_selftest_route_arm(void* pair, int faults_delta, int active_path);
int iccl_selftest_rzv_post(void* entry, int kind, uint64_t k, uint64_t bytes, uint64_t* other_bytes);
/* The armed-transfer failover protocol on host memory:
 * the watchdog's own pass against a host thread playing the two device
 * attempts.  scenario 0 no fault; 1 a slow chunk (3 delta) on a live path:
 * the CTS probe lands, no switch; 2 the primary Down from
 * `fault_chunk`: probe lost, switch at the receiver's breakpoint, K9 copies
 * the suffix; 3 both paths Down: ConnectionFailed; 4 an
 * upstream stall (ready flags late by 3 delta): no probe at all.
 * out[8] = {watchdog switches, resume chunk or -1, published done, total,
 * both done flags written, monitor records, probe landed, async error};
 * returns 0, or 1 if the transfer did not retire within 20 s. */
int iccl_selftest_failover(int scenario, int nchunks, int fault_chunk, uint64_t delta_us, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* ICCL_B200_H_ */
