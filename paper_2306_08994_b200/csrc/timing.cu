// Optional per-kernel-class device timing (CUDA events on the launch stream),
// used by bench.py to report the dominant kernel's roofline from the timed
// region itself.  Off by default: then begin/end are a single branch.
#include <algorithm>
#include <cstring>
#include <utility>
#include <vector>

#include "common.cuh"

namespace tfb {

static const char* kNames[K_COUNT] = {
    "factor_small_kernel", "factor_subtree_kernel", "large_assemble_kernel",
    "large_diag_kernel", "large_block_kernel", "large_update_kernel<2> (trsm)",
    "large_update_kernel<0> (panel)", "large_update_kernel<1> (schur)",
    "large_diag_finalize_kernel", "solve_fwd_small", "solve_bwd_small", "solve_gather_bwd",
    "solve_fwd_wave", "solve_bwd_wave", "permute_rows_kernel", "large_root_kernel"};

struct Pending {
  int cls;
  cudaEvent_t a, b;
};
static bool g_on = false;
static std::vector<cudaEvent_t> g_pool;
static std::vector<Pending> g_pending;
static Pending g_open = {-1, nullptr, nullptr};

static cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void timer_begin(int cls, cudaStream_t st) {
  if (!g_on) return;
  g_open.cls = cls;
  g_open.a = get_event();
  g_open.b = get_event();
  cudaEventRecord(g_open.a, st);
}

void timer_end(cudaStream_t st) {
  if (!g_on || g_open.cls < 0) return;
  cudaEventRecord(g_open.b, st);
  g_pending.push_back(g_open);
  g_open.cls = -1;
}

}  // namespace tfb

using namespace tfb;

extern "C" void tf_timing_enable(int32_t on) { g_on = on != 0; }

// Per class: the device time during which at least one of its launches was
// in flight (union of the launches' [begin, end] intervals, so launches of
// one class running concurrently on different streams -- lookahead chunks,
// concurrent top slices -- are not counted twice), and the launch count.
extern "C" int32_t tf_timing_collect(double* ms, int64_t* count, int32_t n) {
  if (ms) std::memset(ms, 0, sizeof(double) * n);
  if (count) std::memset(count, 0, sizeof(int64_t) * n);
  std::vector<std::vector<std::pair<float, float>>> iv(K_COUNT);
  if (!g_pending.empty()) {
    const cudaEvent_t ref = g_pending.front().a;
    for (const Pending& p : g_pending) {
      cudaEventSynchronize(p.b);
      float t0 = 0.f, t1 = 0.f;
      cudaEventElapsedTime(&t0, ref, p.a);
      cudaEventElapsedTime(&t1, ref, p.b);
      if (p.cls >= 0 && p.cls < K_COUNT) iv[p.cls].push_back({t0, t1});
    }
  }
  for (int c = 0; c < K_COUNT && c < n; c++) {
    auto& v = iv[c];
    std::sort(v.begin(), v.end());
    double tot = 0.0, s = 0.0, e = -1.0;
    for (const auto& x : v) {
      if (x.first > e) {
        if (e > s) tot += e - s;
        s = x.first;
        e = x.second;
      } else if (x.second > e) {
        e = x.second;
      }
    }
    if (e > s) tot += e - s;
    if (ms) ms[c] = tot;
    if (count) count[c] = (int64_t)v.size();
  }
  for (const Pending& p : g_pending) {
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
  return K_COUNT;
}

extern "C" const char* tf_timing_class_name(int32_t cls) {
  return (cls >= 0 && cls < K_COUNT) ? kNames[cls] : "";
}
