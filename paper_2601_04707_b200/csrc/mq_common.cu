// Library plumbing: error strings, version, per-kernel event timing.
#include <stdarg.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "mq_common.cuh"
#include "mq_kernels.h"

namespace mq {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ---------------------------------------------------------------- profiling
struct PendingPair {
  int id;
  cudaEvent_t a, b;
};

static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<PendingPair> g_pending;
static std::vector<cudaEvent_t> g_free_events;
static double g_total_ms[K_COUNT];
static int64_t g_launches[K_COUNT];
static std::atomic<int64_t> g_launch_count{0};
static std::atomic<bool> g_pdl_on{true};
bool pdl_enabled() { return g_pdl_on.load(std::memory_order_relaxed); }

static cudaEvent_t take_event() {
  if (!g_free_events.empty()) {
    cudaEvent_t e = g_free_events.back();
    g_free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

static void settle_locked() {
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    g_total_ms[p.id] += ms;
    g_launches[p.id] += 1;
    g_free_events.push_back(p.a);
    g_free_events.push_back(p.b);
  }
  g_pending.clear();
}

ProfScope::ProfScope(int kernel_id, cudaStream_t stream) : id(kernel_id), s(stream), on(false) {
  g_launch_count.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_pending.size() > 8192) settle_locked();
  a = take_event();
  b = take_event();
  cudaEventRecord(a, s);
  on = true;
}

ProfScope::~ProfScope() {
  if (!on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEventRecord(b, s);
  g_pending.push_back(PendingPair{id, a, b});
}

static const char* kNames[K_COUNT] = {
#define MQ_KNAME(e, s) s,
    MQ_KERNEL_LIST(MQ_KNAME)
#undef MQ_KNAME
};

}  // namespace mq

extern "C" {

int mq_version(void) { return 1; }

const char* mq_last_error(void) { return mq::g_err; }

int mq_stream_check(void* stream) {
  MQ_CUDA(cudaStreamSynchronize(mq::as_stream(stream)));
  MQ_CUDA(cudaGetLastError());
  return MQ_OK;
}

int mq_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(mq::g_prof_mu);
  mq::g_prof_on = on != 0;
  return MQ_OK;
}

int mq_prof_reset(void) {
  std::lock_guard<std::mutex> lk(mq::g_prof_mu);
  mq::settle_locked();
  for (int i = 0; i < mq::K_COUNT; ++i) {
    mq::g_total_ms[i] = 0.0;
    mq::g_launches[i] = 0;
  }
  mq::g_launch_count.store(0);
  return MQ_OK;
}

int mq_prof_num_kernels(void) { return mq::K_COUNT; }

const char* mq_prof_kernel_name(int id) {
  if (id < 0 || id >= mq::K_COUNT) return "";
  return mq::kNames[id];
}

int mq_prof_read(double* total_ms, int64_t* launches, int32_t n) {
  std::lock_guard<std::mutex> lk(mq::g_prof_mu);
  mq::settle_locked();
  for (int i = 0; i < n && i < mq::K_COUNT; ++i) {
    total_ms[i] = mq::g_total_ms[i];
    launches[i] = mq::g_launches[i];
  }
  return MQ_OK;
}

int64_t mq_launch_count(void) { return mq::g_launch_count.load(); }

int mq_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  MQ_CHECK_ARG(bytes >= 0 && (bytes == 0 || (dst && src)), "mq_memcpy_async: bad arguments");
  if (bytes) MQ_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, mq::as_stream(stream)));
  return MQ_OK;
}

int mq_memset_async(void* dst, int32_t value, int64_t bytes, void* stream) {
  MQ_CHECK_ARG(bytes >= 0 && (bytes == 0 || dst), "mq_memset_async: bad arguments");
  if (bytes) MQ_CUDA(cudaMemsetAsync(dst, value, (size_t)bytes, mq::as_stream(stream)));
  return MQ_OK;
}

int mq_set_pdl(int32_t on) {
  mq::g_pdl_on.store(on != 0);
  return MQ_OK;
}

int mq_get_pdl(void) { return mq::g_pdl_on.load() ? 1 : 0; }

}  // extern "C"
