// Host-side arithmetic of the ICCL path: configuration (Table 5 defaults +
// ICCL_* env overrides), error strings, and the SPEC formulas the runtime
// and the Python layer use — retry_timeout, the switch_qp pointer retreat,
// the window throughput monitor and opCount lagging-rank detection.  These
// run without a GPU, so the CPU test suite checks them against the oracle.
#include <time.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "iccl_internal.h"

namespace iccl {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

static bool env_u64(const char* name, uint64_t* out) {
  const char* v = getenv(name);
  if (!v || !*v) return false;
  char* end = nullptr;
  unsigned long long x = strtoull(v, &end, 0);
  if (end == v) return false;
  // accept K/M/G suffixes for byte sizes
  if (*end == 'K' || *end == 'k') x <<= 10;
  else if (*end == 'M' || *end == 'm') x <<= 20;
  else if (*end == 'G' || *end == 'g') x <<= 30;
  *out = x;
  return true;
}

static bool env_i32(const char* name, int32_t* out) {
  const char* v = getenv(name);
  if (!v || !*v) return false;
  char* end = nullptr;
  long x = strtol(v, &end, 0);
  if (end == v) return false;
  *out = (int32_t)x;
  return true;
}

}  // namespace iccl

using namespace iccl;

extern "C" {

const char* iccl_get_error_string(iccl_result_t r) {
  switch (r) {
    case ICCL_SUCCESS: return "success";
    case ICCL_ERR_INVALID_ARGUMENT: return "invalid argument";
    case ICCL_ERR_CUDA: return "CUDA error";
    case ICCL_ERR_SYSTEM: return "system error";
    case ICCL_ERR_QP_IN_ERROR_STATE: return "QpInErrorState";
    case ICCL_ERR_UNREGISTERED_REGION: return "UnregisteredRegion";
    case ICCL_ERR_ZERO_LENGTH_MESSAGE: return "ZeroLengthMessage";
    case ICCL_ERR_CONNECTION_FAILED: return "ConnectionFailed";
    case ICCL_ERR_UNKNOWN_WR: return "UnknownWr";
    case ICCL_ERR_TARGET_QP_DEAD: return "TargetQpDead";
    case ICCL_ERR_NON_POSITIVE_DURATION: return "NonPositiveDuration";
    case ICCL_ERR_WINDOW_NOT_FULL: return "WindowNotFull";
    case ICCL_ERR_GROUP_TOO_SMALL: return "GroupTooSmall";
    case ICCL_ERR_NO_SM_AVAILABLE: return "NoSmAvailable";
    case ICCL_ERR_INVALID_CONFIG: return "InvalidConfig";
    case ICCL_ERR_CONFIG: return "ConfigError";
    case ICCL_ERR_SIZE_MISMATCH: return "send/recv size mismatch";
    case ICCL_ERR_TIMEOUT: return "timeout";
    case ICCL_ERR_IN_PROGRESS: return "in progress";
    case ICCL_ERR_ABORTED: return "communicator aborted";
    default: return "unknown error";
  }
}

const char* iccl_get_last_error(void) { return last_error(); }

int iccl_get_version(void) { return ICCL_B200_VERSION; }

// Table 5 / RunConfig defaults, mapped
// to the B200 path (SURVEY.md §5 "Config / flag system").
iccl_result_t iccl_config_init(iccl_config_t* c) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  memset(c, 0, sizeof(*c));
  // Every chunk boundary drains the copy engine (~4-5 us on B200, measured in
  // probes/p2p_probe3/4), so the default chunk is large; failover and the
  // monitor get finer breakpoints / records by lowering it.
  c->chunk_bytes = 256ull << 20;
  c->streams_per_peer = 1;       // Table 5 "QP number 2" -> copy streams; peer copies do not overlap across streams
  c->sm_cap = 16;                // Table 5 "channel number 32" maps to K1 CTAs
  c->window = 4;
  c->monitor_window = 8;         // Table 5 "window size 8"
  c->monitor_enabled = 0;
  c->backup_kind = ICCL_BACKUP_SM;
  c->transport = ICCL_TRANSPORT_AUTO;
  c->timeout_exponent = 18;      // ICCL_IB_TIMEOUT 18 (Table 5)
  c->retry_count = 7;            // ICCL_IB_RETRY_CNT 7 (Table 5)
  c->delta_us = 2000;            // NVLink-scale watchdog
  c->probe_period_us = 500;      // monitor_failed_link period
  c->sm_small_bytes = 1024 * 1024;  // AUTO: <= 1 MiB between GPUs takes the LL kernel path (K5): 8.7-15.5 us (K6 at 1 MiB: 18.9 us)
  c->proxy_cpu = -1;
  c->relay_slot_mib = 32;        // relay backup: 2 x 32 MiB staging per source on the relay GPU
  c->direct_max_kib = 16 * 1024; // AUTO: 256 KiB < n <= 16 MiB take the direct SM path (K6): 18-40 us vs 22-48 us on the copy-engine chain
  uint64_t u;
  int32_t i;
  if (env_u64("ICCL_CHUNK_BYTES", &u)) c->chunk_bytes = u;
  if (env_i32("ICCL_QP_NUM", &i)) c->streams_per_peer = i;
  if (env_i32("ICCL_SM_CAP", &i)) c->sm_cap = i;
  if (env_i32("ICCL_WINDOW_CHUNKS", &i)) c->window = i;
  if (env_i32("ICCL_MONITOR_WINDOW", &i)) c->monitor_window = i;
  if (env_i32("ICCL_MONITOR", &i)) c->monitor_enabled = i;
  if (env_i32("ICCL_BACKUP", &i)) c->backup_kind = i;
  if (env_i32("ICCL_TRANSPORT", &i)) c->transport = i;
  if (env_i32("ICCL_IB_TIMEOUT", &i)) c->timeout_exponent = i;
  if (env_i32("ICCL_IB_RETRY_CNT", &i)) c->retry_count = i;
  if (env_u64("ICCL_DELTA_US", &u)) c->delta_us = u;
  if (env_u64("ICCL_PROBE_PERIOD_US", &u)) c->probe_period_us = u;
  if (env_u64("ICCL_SM_SMALL_BYTES", &u)) c->sm_small_bytes = u;
  if (env_i32("ICCL_PROXY_CPU", &i)) c->proxy_cpu = i;
  if (env_i32("ICCL_RELAY_SLOT_MIB", &i)) c->relay_slot_mib = i;
  if (env_i32("ICCL_DIRECT_MAX_KIB", &i)) c->direct_max_kib = i;
  return ICCL_SUCCESS;
}

iccl_result_t iccl_config_validate(const iccl_config_t* c) {
  if (!c) return ICCL_ERR_INVALID_ARGUMENT;
  ICCL_RETURN_IF(c->chunk_bytes < 4096 || (c->chunk_bytes & 15), ICCL_ERR_INVALID_CONFIG,
                 "chunk_bytes must be >= 4096 and a multiple of 16");
  ICCL_RETURN_IF(c->streams_per_peer < 1 || c->streams_per_peer > 8, ICCL_ERR_INVALID_CONFIG,
                 "streams_per_peer must be in [1, 8]");
  ICCL_RETURN_IF(c->sm_cap < 1 || c->sm_cap > 148, ICCL_ERR_INVALID_CONFIG, "sm_cap must be in [1, 148]");
  ICCL_RETURN_IF(c->window < 1 || c->window > 1024, ICCL_ERR_INVALID_CONFIG, "window must be in [1, 1024]");
  ICCL_RETURN_IF(c->monitor_window < 1, ICCL_ERR_INVALID_CONFIG, "window size must be >= 1");
  ICCL_RETURN_IF(c->backup_kind != ICCL_BACKUP_SM && c->backup_kind != ICCL_BACKUP_RELAY, ICCL_ERR_INVALID_CONFIG,
                 "backup_kind must be ICCL_BACKUP_SM or ICCL_BACKUP_RELAY");
  ICCL_RETURN_IF(c->transport < ICCL_TRANSPORT_AUTO || c->transport > ICCL_TRANSPORT_SM, ICCL_ERR_INVALID_CONFIG,
                 "transport must be AUTO, CE or SM");
  ICCL_RETURN_IF(c->timeout_exponent < 0 || c->timeout_exponent > 31 || c->retry_count < 0 || c->retry_count > 7,
                 ICCL_ERR_INVALID_CONFIG, "timeout exponent in [0,31], retry count in [0,7]");
  ICCL_RETURN_IF(c->probe_period_us == 0, ICCL_ERR_INVALID_CONFIG, "probe period must be > 0");
  ICCL_RETURN_IF(c->relay_slot_mib < 1 || c->relay_slot_mib > 1024, ICCL_ERR_INVALID_CONFIG,
                 "relay_slot_mib must be in [1, 1024]");
  ICCL_RETURN_IF(c->direct_max_kib < 0, ICCL_ERR_INVALID_CONFIG, "direct_max_kib must be >= 0");
  return ICCL_SUCCESS;
}

// retry_timeout: (4.096 us x 2^exp) x (retry + 1).
uint64_t iccl_retry_timeout_ns(int timeout_exponent, int retry_count) {
  if (timeout_exponent < 0 || retry_count < 0) return 0;
  return 4096ull * (1ull << timeout_exponent) * (uint64_t)(retry_count + 1);
}

// switch_qp pointer retreat, receiver-driven.
int iccl_switch_pointers(iccl_xfer_state_t* s, iccl_xfer_state_t* r) {
  if (!s || !r) return -1;
  r->received = r->done;
  s->acked = r->done;
  s->posted = s->acked;
  s->transmitted = s->acked;
  return s->acked;
}

iccl_result_t iccl_per_message_throughput(const iccl_mon_rec_t* rec, double* bps) {
  if (!rec || !bps) return ICCL_ERR_INVALID_ARGUMENT;
  if (rec->t2_ns <= rec->t1_ns) {
    set_last_error("t2 <= t1");
    return ICCL_ERR_NON_POSITIVE_DURATION;
  }
  *bps = (double)rec->bytes / ((double)(rec->t2_ns - rec->t1_ns) * 1e-9);
  return ICCL_SUCCESS;
}

// window_throughput: sum(bytes) / (t2 of the last record - t1 of the first),
// records in completion order.
iccl_result_t iccl_window_throughput(const iccl_mon_rec_t* recs, int n, int window, double* bps) {
  if (!bps || window < 1) return ICCL_ERR_INVALID_ARGUMENT;
  if (n != window || !recs) {
    set_last_error("window not full");
    return ICCL_ERR_WINDOW_NOT_FULL;
  }
  uint64_t t1 = recs[0].t1_ns, t2 = recs[n - 1].t2_ns;
  if (t2 <= t1) {
    set_last_error("t2 <= t1");
    return ICCL_ERR_NON_POSITIVE_DURATION;
  }
  double bytes = 0;
  for (int i = 0; i < n; i++) bytes += (double)recs[i].bytes;
  *bps = bytes / ((double)(t2 - t1) * 1e-9);
  return ICCL_SUCCESS;
}

// sample_series: one sample per completion once W records are in
// (SPEC.md:340-348); count = n - W + 1.
iccl_result_t iccl_sample_series(const iccl_mon_rec_t* recs, int n, int window, double* out_bps, uint64_t* out_t,
                                 int* n_out) {
  if (!n_out || window < 1 || n < 0) return ICCL_ERR_INVALID_ARGUMENT;
  int m = n >= window ? n - window + 1 : 0;
  *n_out = m;
  for (int k = 0; k < m; k++) {
    double v = 0;
    iccl_result_t r = iccl_window_throughput(recs + k, window, window, &v);
    if (r != ICCL_SUCCESS) return r;
    if (out_bps) out_bps[k] = v;
    if (out_t) out_t[k] = recs[k + window - 1].t2_ns;
  }
  return ICCL_SUCCESS;
}

// detect_lagging_rank: unique strict minimum whose gap to
// the second smallest exceeds the threshold.
iccl_result_t iccl_detect_lagging_rank(const uint64_t* c, int n, uint64_t threshold, int* rank) {
  if (!c || !rank) return ICCL_ERR_INVALID_ARGUMENT;
  if (n < 2) return ICCL_ERR_GROUP_TOO_SMALL;
  int lo = 0;
  for (int i = 1; i < n; i++)
    if (c[i] < c[lo]) lo = i;
  uint64_t second = UINT64_MAX;
  for (int i = 0; i < n; i++)
    if (i != lo && c[i] < second) second = c[i];
  *rank = (second > c[lo] && second - c[lo] > threshold) ? lo : -1;
  return ICCL_SUCCESS;
}

}  // extern "C"

namespace iccl {

const Driver* driver() {
  static Driver d = [] {
    Driver x;
    memset(&x, 0, sizeof(x));
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !*fn)
        ok = false;
    };
    get("cuGetErrorString", (void**)&x.cuGetErrorString);
    get("cuInit", (void**)&x.cuInit);
    get("cuDeviceGet", (void**)&x.cuDeviceGet);
    get("cuDeviceGetAttribute", (void**)&x.cuDeviceGetAttribute);
    get("cuStreamWriteValue32", (void**)&x.cuStreamWriteValue32);
    get("cuStreamWaitValue32", (void**)&x.cuStreamWaitValue32);
    get("cuStreamBatchMemOp", (void**)&x.cuStreamBatchMemOp);
    get("cuMemcpyDtoDAsync", (void**)&x.cuMemcpyDtoDAsync);
    get("cuMemGetAddressRange", (void**)&x.cuMemGetAddressRange);
    get("cuPointerGetAttribute", (void**)&x.cuPointerGetAttribute);
    x.ok = ok;
    return x;
  }();
  if (!d.ok) {
    set_last_error("CUDA driver entry points unavailable (no GPU driver?)");
    return nullptr;
  }
  return &d;
}

}  // namespace iccl
