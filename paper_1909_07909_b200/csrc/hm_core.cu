// hm_core.cu — libhm plumbing shared by every call: thread-local error
// messages (hm_last_error), the launch trace (hm_profile_*), the tree check
// and the misc ABI queries. Paper: hm-toolbox (arXiv 1909.07909).
#include <mutex>

#include "hm_internal.cuh"

namespace hmi {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

hm_status fail(hm_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

hm_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return HM_OK;
}

int num_sms() {
  static int cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = sms > 0 ? sms : 1;
  }
  return cached[dev];
}

hm_status check_tree(const hm_tree* t) {
  if (!t) return fail(HM_ERR_INVALID_ARG, "tree is NULL");
  if (t->flags != 0) return fail(HM_ERR_UNSUPPORTED, "tree flags %d: only the balanced tree of P:86-91 is built", t->flags);
  if (t->n < 1 || t->leaf < 1 || t->levels < 0 || t->levels > 40)
    return fail(HM_ERR_INVALID_ARG, "tree: need n >= 1, leaf >= 1, 0 <= levels <= 40 (n=%lld leaf=%lld levels=%d)",
                (long long)t->n, (long long)t->leaf, t->levels);
  if ((t->leaf << t->levels) != t->n)
    return fail(HM_ERR_UNSUPPORTED, "n = %lld is not leaf * 2^levels = %lld * 2^%d (general endpoint vectors, P:560-565, not built)",
                (long long)t->n, (long long)t->leaf, t->levels);
  if (t->leaf + hm::kMaxRank * t->levels > kSmemBudgetDoubles)
    return fail(HM_ERR_UNSUPPORTED, "leaf size %lld exceeds the shared-memory staging limit", (long long)t->leaf);
  if (t->levels + 1 > hm::kMaxLevels) return fail(HM_ERR_UNSUPPORTED, "too many levels");
  return HM_OK;
}

hm_status check_part(const hm_tree* tree, const hm_part* part, DistPart* d) {
  if (!part) return fail(HM_ERR_INVALID_ARG, "part is NULL");
  const int P = part->nranks;
  if (P < 1 || (P & (P - 1)) != 0) return fail(HM_ERR_UNSUPPORTED, "nranks = %d is not a power of two", P);
  int q = 0;
  while ((1 << q) < P) ++q;
  if (q > tree->levels) return fail(HM_ERR_UNSUPPORTED, "nranks = %d > 2^levels", P);
  if (part->rank < 0 || part->rank >= P) return fail(HM_ERR_INVALID_ARG, "rank %d not in [0, %d)", part->rank, P);
  d->P = P; d->q = q; d->rank = part->rank;
  return HM_OK;
}

// ----------------------------------------------------------- launch trace --
// hm_profile_enable / hm_profile_collect: every launch bracketed by two events.
namespace {
struct TraceRec {
  const char* name;
  int32_t call;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
int32_t g_prof_call = -1;
std::vector<TraceRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_new_call() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_prof_on) ++g_prof_call;
}

int prof_begin(const char* name, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return -1;
  TraceRec r{name, g_prof_call, prof_event(), prof_event()};
  cudaEventRecord(r.a, s);
  g_prof_recs.push_back(r);
  return (int)g_prof_recs.size() - 1;
}

void prof_end(int slot, cudaStream_t s) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (slot < (int)g_prof_recs.size()) cudaEventRecord(g_prof_recs[slot].b, s);
}

}  // namespace hmi

using namespace hmi;

// Source hash of this build (paper_1909_07909_b200/build.py compares it with
// the sources on disk and rebuilds a stale library).
#ifndef HM_SRC_HASH_STR
#define HM_SRC_HASH_STR "HM_SRC_HASH=unknown"
#endif
extern "C" __attribute__((used)) const char hm_src_hash[] = HM_SRC_HASH_STR;

extern "C" {

const char* hm_last_error(void) { return g_err.c_str(); }

hm_status hm_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return HM_OK;
}

hm_status hm_profile_collect(hm_launch_record* out, int32_t cap, int32_t* count) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (cap > 0 && !out) return fail(HM_ERR_INVALID_ARG, "out is NULL");
  int32_t n = 0;
  hm_status st = HM_OK;
  for (const TraceRec& r : g_prof_recs) {
    if (n < cap) {
      float ms = 0.f, t0 = 0.f;
      if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess ||
          cudaEventElapsedTime(&t0, g_prof_recs.front().a, r.a) != cudaSuccess)
        st = cuda_check("hm_profile_collect");
      memset(&out[n], 0, sizeof out[n]);
      strncpy(out[n].name, r.name, sizeof out[n].name - 1);
      out[n].call = r.call;
      out[n].ms = ms;
      out[n].start_ms = t0;
    }
    ++n;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  g_prof_call = -1;
  if (count) *count = n;
  return st;
}
int32_t hm_abi_version(void) { return HM_ABI_VERSION; }
int32_t hm_last_launch_count(void) { return g_launches; }
}  // extern "C"
