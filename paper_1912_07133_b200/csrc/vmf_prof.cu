// vmf_prof.cu -- see vmf_prof.cuh.
#include <atomic>
#include <mutex>
#include <vector>

#include "vmf_common.cuh"
#include "vmf_prof.cuh"

namespace vmf {

const char *const kKernelNames[K_NUM_IDS] = {
    "iir_carry", "iir_scan", "iir_apply", "iir_scale", "fir_rows", "fir_cols",
    "laplacian", "absmax", "nms_count", "nms_scan", "nms_write", "iir_rows_fused",
    "iir_cols_fused", "finalize", "col_carry", "col_scan", "sweep_border", "sweep_rows",
    "col_apply", "firtc_prep", "firtc_rows", "firtc_cols"};

namespace {
std::atomic<long long> g_launches{0};
std::mutex g_mu;
bool g_on = false;
struct Rec {
  int id;
  cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
// Inside a stream capture the event becomes a record node of the graph, so a
// replayed graph is timed launch by launch without host gaps.
void record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
}
}  // namespace

Launch::Launch(KernelId id, cudaStream_t st) : slot_(-1), st_(st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  Rec r{(int)id, get_event(), get_event()};
  record(r.a, st);
  g_recs.push_back(r);
  slot_ = (int)g_recs.size() - 1;
}

Launch::~Launch() {
  if (slot_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  record(g_recs[slot_].b, st_);
}

}  // namespace vmf

extern "C" {

long long vmf_launch_count(void) { return vmf::g_launches.load(); }

int vmf_num_kernel_ids(void) { return vmf::K_NUM_IDS; }

const char *vmf_kernel_name(int id) {
  return (id >= 0 && id < vmf::K_NUM_IDS) ? vmf::kKernelNames[id] : "";
}

void vmf_profile_begin(void) {
  std::lock_guard<std::mutex> lk(vmf::g_mu);
  for (auto &r : vmf::g_recs) {
    vmf::g_pool.push_back(r.a);
    vmf::g_pool.push_back(r.b);
  }
  vmf::g_recs.clear();
  vmf::g_on = true;
}

void vmf_profile_stop(void) {
  std::lock_guard<std::mutex> lk(vmf::g_mu);
  vmf::g_on = false;
}

// Waits for the recorded events; ms[id] = summed duration, counts[id] = launches.
int vmf_profile_read(double *ms, long long *counts, int n) {
  std::lock_guard<std::mutex> lk(vmf::g_mu);
  for (int i = 0; i < n; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  for (auto &r : vmf::g_recs) {
    cudaEventSynchronize(r.b);
    float t = 0.0f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (r.id < n) {
      ms[r.id] += t;
      counts[r.id] += 1;
    }
  }
  return vmf::K_NUM_IDS;
}

// The recorded launches in order: id, start and end in ms after the first
// recorded start (a concurrent replay's timeline).  Returns the count.
int vmf_profile_timeline(int *ids, float *t0, float *t1, int n) {
  std::lock_guard<std::mutex> lk(vmf::g_mu);
  int m = 0;
  if (vmf::g_recs.empty()) return 0;
  cudaEvent_t ref = vmf::g_recs[0].a;
  for (auto &r : vmf::g_recs) {
    if (m >= n) break;
    cudaEventSynchronize(r.b);
    float a = 0.0f, b = 0.0f;
    if (cudaEventElapsedTime(&a, ref, r.a) != cudaSuccess ||
        cudaEventElapsedTime(&b, ref, r.b) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    ids[m] = r.id;
    t0[m] = a;
    t1[m] = b;
    ++m;
  }
  return m;
}

int vmf_profile_end(double *ms, long long *counts, int n) {
  vmf_profile_stop();
  return vmf_profile_read(ms, counts, n);
}

}  // extern "C"
