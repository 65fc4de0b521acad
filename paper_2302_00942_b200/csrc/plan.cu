#include <stdio.h>
// Host side of the C ABI (include/rfd.h): argument validation, the plan
// object (device buffers it owns), launch sequencing, status codes, launch
// counting and event-based per-kernel timing.  No arithmetic of the method
// runs here: every step of the path is one of the kernels in k_*.cu.  The
// one host-computed quantity is the constant C_R = P(||Z||_1 <= R) of the
// truncated proposal (A7), fixed by R alone.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rfd.h"
#include "rfd_internal.h"

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_last_error;

rfd_status fail(rfd_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

rfd_status cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? RFD_ENOMEM : RFD_ECUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define RFD_CUDA(call)                                     \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
  } while (0)

// ------------------------------------------------------------------ launches
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_profiling{0};
std::mutex g_prof_mu;
struct Pending {
  const char* name;
  cudaEvent_t a, b;
};
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_free_events;
std::map<std::string, std::pair<int64_t, double>> g_prof;
thread_local cudaEvent_t t_open_event = nullptr;
std::string g_prof_only;  // non-empty: profile only the launches of this name

cudaEvent_t take_event() {
  if (!g_free_events.empty()) {
    cudaEvent_t e = g_free_events.back();
    g_free_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

namespace rfd {
void launch_begin(const char* name, cudaStream_t s) {
  if (g_profiling.load(std::memory_order_relaxed)) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_only.empty() && g_prof_only != name) return;
    t_open_event = take_event();
    cudaEventRecord(t_open_event, s);
  }
}
void launch_end(const char* name, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  // RFD_SYNC_CHECK=1 (debugging): synchronize after every launch and name the
  // kernel that faulted.
  static const bool sync_check = [] {
    const char* e = getenv("RFD_SYNC_CHECK");
    return e && e[0] == '1';
  }();
  if (sync_check) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) fprintf(stderr, "rfd: kernel %s failed: %s\n", name, cudaGetErrorString(e));
  }
  if (t_open_event) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = take_event();
    cudaEventRecord(b, s);
    g_pending.push_back(Pending{name, t_open_event, b});
    t_open_event = nullptr;
  }
}
}  // namespace rfd

// ------------------------------------------------------------------ plan
struct rfd_plan {
  int device = 0;
  int sms = 148;
  int64_t n = 0;
  int batch = 1;
  int m = 0;
  int r = 0;
  double eps = 0, lambda = 0;
  uint64_t seed = 0;
  int scaling = 0;
  int symmetric = 1;
  // sharded cloud: this rank's shard of n_total points
  int rank = 0, world = 1;
  rfd_allgather_fn allgather = nullptr;
  void* ctx = nullptr;
  int64_t n_total = 0;
  // owned device state
  float4* pts = nullptr;      // batch*n
  float* pts16 = nullptr;     // batch*ceil(n/16)*48: SoA groups of 16 points (pass 1)
  float4* centre = nullptr;   // batch: bounding-box midpoint subtracted from the points
  float4* omega4 = nullptr;   // m
  float4* omega_rad4 = nullptr;  // m: fp32(2 pi omega) for the tensor-core kernels
  int64_t gram_nodes = 0;        // a4 through a spread grid of this many nodes (0: direct)
  double* nu = nullptr;       // m
  double* G = nullptr;        // batch*r*r (interleaved)
  double* C = nullptr;        // batch*r*r (interleaved)
  int* flags = nullptr;       // [0] nu/sampler flags, [2..3] ||Z||_1 bits, [4] overflow
  // integrate workspace (grows with d)
  int ws_d = 0;
  float* s_partial = nullptr; // batch*chunks*r*16
  double* S = nullptr;        // batch*r*d
  double* S_parts = nullptr;  // world*r*d (sharded plans: the gathered partials)
  float* small_part = nullptr;  // d <= 4 path: range x cloud-slot partials
  size_t small_part_elems = 0;
  unsigned int* bar = nullptr;  // d <= 4 path: grid barrier (2 words, self-resetting)
  float* Y = nullptr;         // batch*r*d
  int last_d = 0;
  // host-buffer staging (rfd_integrate_host / rfd_gfi_host)
  float* stage = nullptr;
  size_t stage_elems = 0;
  float* pipe_partial = nullptr;  // pass-1 partials of the chunked (pipelined) host path
  size_t pipe_partial_elems = 0;
  cudaStream_t cs_h2d = nullptr, cs_d2h = nullptr;  // copy streams of the host path
  cudaStream_t aux = nullptr;  // rfd_gfi: pass 1 beside the plan's core
  cudaEvent_t ev[2 * 16 + 2] = {};
  cudaStream_t stream = nullptr;  // stream of the last call (frees are ordered on it)
  bool core_pending = false;      // the core's overflow flag is read back but not yet checked
};

namespace {

double l1_ball_mass(double R) {
  // C_R = int_0^R int_0^{R-a} h(a) h(b) erf((R-a-b)/sqrt2) db da with the
  // half-normal density h(t) = 2 exp(-t^2/2)/sqrt(2 pi); composite 16-point
  // Gauss-Legendre in both variables.
  static const double xg[8] = {0.0950125098376374, 0.2816035507792589, 0.4580167776572274,
                               0.6178762444026438, 0.7554044083550030, 0.8656312023878318,
                               0.9445750230732326, 0.9894009349916499};
  static const double wg[8] = {0.1894506104550685, 0.1826034150449236, 0.1691565193950025,
                               0.1495959888165767, 0.1246289712555339, 0.0951585116824928,
                               0.0622535239386479, 0.0271524594117541};
  const int panels = 96;
  auto h = [](double t) { return 2.0 * exp(-0.5 * t * t) / sqrt(2.0 * M_PI); };
  auto inner = [&](double a) {
    const double L = R - a;
    double acc = 0.0;
    for (int p = 0; p < panels; ++p) {
      const double lo = L * p / panels, hi = L * (p + 1) / panels;
      const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
      for (int q = 0; q < 8; ++q)
        for (int sgn = -1; sgn <= 1; sgn += 2) {
          const double b = mid + sgn * half * xg[q];
          acc += half * wg[q] * h(b) * erf((R - a - b) / sqrt(2.0));
        }
    }
    return acc;
  };
  double acc = 0.0;
  for (int p = 0; p < panels; ++p) {
    const double lo = R * p / panels, hi = R * (p + 1) / panels;
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    for (int q = 0; q < 8; ++q)
      for (int sgn = -1; sgn <= 1; sgn += 2) {
        const double a = mid + sgn * half * xg[q];
        acc += half * wg[q] * h(a) * inner(a);
      }
  }
  return acc;
}

double cached_c_r() {
  static double c = -1.0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (c < 0) c = l1_ball_mass(RFD_TRUNCATION_R);
  return c;
}

bool is_device_pointer(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Stream-ordered allocations from a library-owned pool that keeps its
// memory (release threshold = max): plan creation and workspace growth then
// cost no cudaMalloc/cudaFree round trips after the first use.
cudaMemPool_t library_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  uint64_t thr = ~uint64_t(0);
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  pools[dev] = pool;
  return pool;
}

template <typename T>
cudaError_t dalloc(T** ptr, size_t count, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = library_pool(dev);
  const size_t bytes = count * sizeof(T) + 16;
  if (!pool) return cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, s);
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(ptr), bytes, pool, s);
}

template <typename T>
void dfree(T*& ptr, cudaStream_t s) {
  if (ptr) cudaFreeAsync(ptr, s);
  ptr = nullptr;
}

// sync = false: every free is stream-ordered on the plan's stream (pool
// memory: cudaFreeAsync), streams and events are destroyed deferred by the
// driver -- nothing waits on the host (rfd_gfi_host's internal plans).
void free_plan(rfd_plan* p, bool sync = true) {
  if (!p) return;
  cudaStream_t s = p->stream;
  if (p->aux) {  // the frees below (stream-ordered on s) come after its work
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(e, p->aux);
      cudaStreamWaitEvent(s, e, 0);
      cudaEventDestroy(e);
    } else {
      cudaStreamSynchronize(p->aux);
    }
    cudaStreamDestroy(p->aux);
    p->aux = nullptr;
  }
  if (sync) cudaStreamSynchronize(s);
  dfree(p->pts, s);
  dfree(p->pts16, s);
  dfree(p->centre, s);
  dfree(p->omega4, s);
  dfree(p->omega_rad4, s);
  dfree(p->nu, s);
  dfree(p->G, s);
  dfree(p->C, s);
  dfree(p->flags, s);
  dfree(p->s_partial, s);
  dfree(p->S, s);
  dfree(p->S_parts, s);
  dfree(p->small_part, s);
  dfree(p->bar, s);
  dfree(p->Y, s);
  dfree(p->stage, s);
  dfree(p->pipe_partial, s);
  if (p->cs_h2d) cudaStreamDestroy(p->cs_h2d);
  if (p->cs_d2h) cudaStreamDestroy(p->cs_d2h);
  for (cudaEvent_t e : p->ev)
    if (e) cudaEventDestroy(e);
  delete p;
}

struct TempBuffers {
  cudaStream_t s;
  std::vector<void*> bufs;
  explicit TempBuffers(cudaStream_t st) : s(st) {}
  ~TempBuffers() {
    for (void* b : bufs) cudaFreeAsync(b, s);
  }
  template <typename T>
  cudaError_t alloc(T** ptr, size_t count) {
    cudaError_t e = dalloc(ptr, count, s);
    if (e == cudaSuccess) bufs.push_back(*ptr);
    return e;
  }
};

// Host read-backs (the bounding box, omega and the frequency flags for a4's
// grid; ||Z||_1 and the overflow flag of the core) go through a per-thread
// pinned buffer and an event: a pageable cudaMemcpyAsync blocks the host for
// its own round trip (two in a row plus a stream synchronisation took ~44 us
// of idle GPU in the cfg-5 step), and an event wait does not wait for work
// enqueued behind the copy.  Slots: the core's flags, the box, the frequency
// flags, omega (RFD_MAX_M float4).
struct HostSlot {
  char* buf = nullptr;
  cudaEvent_t ev = nullptr, ev_src = nullptr, ev_join = nullptr;
  cudaStream_t side = nullptr;  // copies the work stream must not wait for
  int dev = -1;
};
constexpr size_t kSlotCore = 0, kSlotBox = 64, kSlotFlags = 128, kSlotOmega = 256;
constexpr size_t kSlotBytes = kSlotOmega + size_t(RFD_MAX_M) * sizeof(float4);
rfd_status host_slot(HostSlot** out) {
  thread_local HostSlot h;  // lives as long as the thread (not freed at exit)
  int dev = 0;
  RFD_CUDA(cudaGetDevice(&dev));
  if (h.dev != dev) {  // (a thread that moves to another device: fresh events, stream)
    RFD_CUDA(cudaEventCreateWithFlags(&h.ev, cudaEventDisableTiming));
    RFD_CUDA(cudaEventCreateWithFlags(&h.ev_src, cudaEventDisableTiming));
    RFD_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
    RFD_CUDA(cudaStreamCreateWithFlags(&h.side, cudaStreamNonBlocking));
    h.dev = dev;
  }
  if (!h.buf) RFD_CUDA(cudaMallocHost(&h.buf, kSlotBytes));
  *out = &h;
  return RFD_OK;
}
// wait for everything enqueued on st up to now (not for later work).  Used
// where the GPU idles until the host has read the result (a4's grid sizing),
// so the host polls the event instead of sleeping in cudaEventSynchronize
// (the wake-up is on the critical path; the wait is tens of microseconds).
rfd_status slot_wait(HostSlot* h, cudaStream_t st) {
  RFD_CUDA(cudaEventRecord(h->ev, st));
  cudaError_t e;
  while ((e = cudaEventQuery(h->ev)) == cudaErrorNotReady) {
  }
  RFD_CUDA(e);
  return RFD_OK;
}

// One kernel gathers what a4's grid sizing needs (the box, the frequency
// flags, omega) straight into the pinned slot buffer (mapped: cudaMallocHost
// memory is device-accessible under unified addressing) -- one small launch
// instead of three in-stream copies, each with the copy engine's latency.
__global__ void gather_readback_kernel(const unsigned int* __restrict__ bbox,
                                       const int* __restrict__ flags,
                                       const float4* __restrict__ omega4, int m,
                                       char* __restrict__ host) {
  unsigned int* hb = reinterpret_cast<unsigned int*>(host + kSlotBox);
  int* hf = reinterpret_cast<int*>(host + kSlotFlags);
  float4* ho = reinterpret_cast<float4*>(host + kSlotOmega);
  if (threadIdx.x < 6) hb[threadIdx.x] = bbox[threadIdx.x];
  if (threadIdx.x == 0) hf[0] = flags[0];
  for (int k = threadIdx.x; k < m; k += blockDim.x) ho[k] = omega4[k];
}

// D2H copy of what st has computed so far into the slot buffer, on the side
// stream: an in-stream copy delays st's next kernel by the copy's latency
// (~8-17 us measured between the core's kernels); h->ev marks its completion
rfd_status slot_copy_side(HostSlot* h, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  RFD_CUDA(cudaEventRecord(h->ev_src, st));
  RFD_CUDA(cudaStreamWaitEvent(h->side, h->ev_src, 0));
  RFD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->side));
  RFD_CUDA(cudaEventRecord(h->ev, h->side));
  return RFD_OK;
}

// the core's overflow flag, copied back by core_impl (deferred check)
rfd_status core_finish(rfd_plan* p) {
  if (!p->core_pending) return RFD_OK;
  p->core_pending = false;
  HostSlot* h = nullptr;
  const rfd_status hs = host_slot(&h);
  if (hs != RFD_OK) return hs;
  RFD_CUDA(cudaEventSynchronize(h->ev));
  int of = 0;
  memcpy(&of, h->buf + kSlotCore + 4 * sizeof(int), sizeof(int));
  if (of) return fail(RFD_ERANGE, "core: exp(lambda W~) overflows (lambda > 0 or negative nu)");
  return RFD_OK;
}

// a5 on the plan's G: C = lambda D phi1(lambda G D) for the given nu (its
// sign flags in flags[0]); ||Z||_1 is read back for the scaling exponent s.
// flags[2..4] are scratch.  known_sym: the route, when the host has already
// read the frequency flags (-1: not yet) -- the powers Z^2..Z^5 (independent
// of s, launch_core_powers with pw_alpha = 1) are then enqueued before the
// host waits, so the GEMM chain has no gap.  defer: the overflow flag is
// copied back but not waited for (p->core_pending; core_finish checks it once
// the caller has enqueued its next work); otherwise this blocks the host.
rfd_status core_impl(rfd_plan* p, const double* nu, int* flags, double lambda, double* C,
                     int* scaling_out, int* symmetric_out, cudaStream_t st, int known_sym = -1,
                     bool defer = false) {
  const int m = p->m, batch = p->batch;
  const size_t rr = size_t(p->r) * p->r;
  HostSlot* h = nullptr;
  const rfd_status hs = host_slot(&h);
  if (hs != RFD_OK) return hs;
  TempBuffers tmp(st);
  double *Z = nullptr, *work = nullptr;
  RFD_CUDA(tmp.alloc(&Z, rr * batch));
  RFD_CUDA(tmp.alloc(&work, rr * batch * rfd::kCoreWork));
  rfd::launch_core_prep(p->G, nu, flags, lambda, m, batch, Z,
                        reinterpret_cast<unsigned long long*>(flags + 2), st);
  RFD_CUDA(cudaGetLastError());
  int* hflags = reinterpret_cast<int*>(h->buf + kSlotCore);
  rfd_status xs = slot_copy_side(h, hflags, flags, 8 * sizeof(int), st);
  if (xs != RFD_OK) return xs;
  // unscaled powers are safe (no overflow) while ||Z||_1 <= 1e40
  constexpr double kUnscaledMax = 1e40;
  if (known_sym >= 0) rfd::launch_core_powers(Z, m, batch, known_sym == 1, 1.0, work, st);
  RFD_CUDA(cudaEventSynchronize(h->ev));
  if (hflags[0] & 2)
    return fail(RFD_ERANGE, "frequency sampler exhausted its attempts (R too small?)");
  const bool sym = (hflags[0] & 1) == 0;
  double znorm;
  memcpy(&znorm, hflags + 2, sizeof(double));
  // Scaling exponent: smallest s >= 0 with ||Z||_1 / 2^s <= kCoreTheta.
  if (!isfinite(znorm) || znorm > 1e60)
    return fail(RFD_ERANGE, "core: ||lambda G D|| is not finite or too large");
  int s_scale = 0;
  while (ldexp(znorm, -s_scale) > rfd::kCoreTheta) ++s_scale;
  double pw = 1.0;
  if (znorm > kUnscaledMax) {
    pw = ldexp(1.0, -s_scale);
    rfd::launch_core_powers(Z, m, batch, sym, pw, work, st);
  } else if (known_sym < 0) {
    rfd::launch_core_powers(Z, m, batch, sym, 1.0, work, st);
  }
  rfd::launch_core_eval(Z, nu, flags, lambda, m, batch, s_scale, sym, pw, work, C, flags + 4, st);
  RFD_CUDA(cudaGetLastError());
  *scaling_out = s_scale;
  *symmetric_out = sym ? 1 : 0;
  xs = slot_copy_side(h, hflags, flags, 8 * sizeof(int), st);
  if (xs != RFD_OK) return xs;
  p->core_pending = true;
  return defer ? RFD_OK : core_finish(p);
}

// all-gather of `count` fp64 through the caller's collective (sharded plans)
rfd_status exchange(const rfd_plan* p, const double* send, double* recv, size_t count,
                    cudaStream_t st) {
  if (p->allgather(p->ctx, send, recv, count, reinterpret_cast<rfd_stream>(st)) != 0)
    return fail(RFD_ECUDA, "sharded plan: the allgather callback failed");
  RFD_CUDA(cudaGetLastError());
  return RFD_OK;
}

// a4 path: RFD_GRAM_SPREAD=0 always direct, =2 spread whenever the grid is
// feasible (tests), unset/1: spread when the grid has <= n / kSpreadRatio nodes
// and n >= kSpreadMinPoints (below, the direct Gram is faster than the spread
// path's fixed costs: cfg 4, 200k points: 0.49 ms direct vs 0.63 ms spread).
constexpr int64_t kSpreadRatio = 8;
constexpr int64_t kSpreadMinPoints = int64_t(1) << 19;
int gram_spread_mode() {
  const char* e = getenv("RFD_GRAM_SPREAD");
  if (!e || !e[0]) return 1;
  return atoi(e);
}

// before_core (rfd_gfi): called once G, the points and omega are on the
// stream, before the core -- the one-shot GFI starts the field's pass 1 there.
rfd_status create_impl(const float* points, int batch, int64_t n, double eps, double lambda,
                       int m, uint64_t seed, const rfd_shard* shard, cudaStream_t st,
                       rfd_plan** plan_out,
                       const std::function<rfd_status(rfd_plan*)>& before_core = nullptr,
                       bool defer_core = false) {
  if (!plan_out) return fail(RFD_EINVAL, "plan_out is NULL");
  *plan_out = nullptr;
  if (!points) return fail(RFD_EINVAL, "points is NULL");
  if (n < 1) return fail(RFD_EINVAL, "n must be >= 1");
  if (batch < 1) return fail(RFD_EINVAL, "batch must be >= 1");
  if (m < 1 || m > RFD_MAX_M) return fail(RFD_EINVAL, "m must be in [1, RFD_MAX_M]");
  if (!(eps > 0.0) || !isfinite(eps)) return fail(RFD_EINVAL, "eps must be finite and > 0");
  if (!isfinite(lambda)) return fail(RFD_EINVAL, "lambda must be finite");
  if (reinterpret_cast<uintptr_t>(points) % 4 != 0)
    return fail(RFD_EINVAL, "points must be 4-byte aligned");
  const int world = shard ? shard->world : 1;
  if (shard && (shard->world < 1 || shard->rank < 0 || shard->rank >= shard->world ||
                (shard->world > 1 && !shard->allgather)))
    return fail(RFD_EINVAL, "shard: need 0 <= rank < world and an allgather for world > 1");
  if (world > 1 && batch != 1) return fail(RFD_EINVAL, "sharded plans hold one cloud");

  int dev = 0;
  RFD_CUDA(cudaGetDevice(&dev));
  rfd_plan* p = new rfd_plan();
  struct Guard {
    rfd_plan* p;
    bool keep = false;
    ~Guard() {
      if (!keep) free_plan(p);
    }
  } guard{p};
  p->device = dev;
  p->stream = st;
  RFD_CUDA(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, dev));
  p->n = n;
  p->batch = batch;
  p->m = m;
  p->r = 2 * m;
  p->eps = eps;
  p->lambda = lambda;
  p->seed = seed;
  p->n_total = n;
  if (shard) {
    p->rank = shard->rank;
    p->world = shard->world;
    p->allgather = shard->allgather;
    p->ctx = shard->ctx;
  }
  const int64_t total = n * batch;
  const size_t rr = size_t(p->r) * p->r;

  RFD_CUDA(dalloc(&p->pts, size_t(total), st));
  RFD_CUDA(dalloc(&p->pts16, size_t(batch) * size_t((n + 15) / 16) * 48, st));
  RFD_CUDA(dalloc(&p->centre, size_t(batch), st));
  RFD_CUDA(dalloc(&p->omega4, size_t(m), st));
  RFD_CUDA(dalloc(&p->omega_rad4, size_t(m), st));
  RFD_CUDA(dalloc(&p->nu, size_t(m), st));
  RFD_CUDA(dalloc(&p->G, rr * batch, st));
  RFD_CUDA(dalloc(&p->C, rr * batch, st));
  RFD_CUDA(dalloc(&p->flags, size_t(8), st));
  RFD_CUDA(cudaMemsetAsync(p->flags, 0, 8 * sizeof(int), st));
  RFD_CUDA(dalloc(&p->bar, size_t(rfd::kSmallBarWords), st));
  RFD_CUDA(cudaMemsetAsync(p->bar, 0, rfd::kSmallBarWords * sizeof(unsigned int), st));

  TempBuffers tmp(st);
  const float* dev_xyz = points;
  if (!is_device_pointer(points)) {
    float* staged = nullptr;
    RFD_CUDA(tmp.alloc(&staged, size_t(total) * 3));
    RFD_CUDA(cudaMemcpyAsync(staged, points, size_t(total) * 3 * sizeof(float),
                             cudaMemcpyHostToDevice, st));
    dev_xyz = staged;
  }
  unsigned int* bbox = nullptr;
  RFD_CUDA(tmp.alloc(&bbox, size_t(batch) * 6));
  unsigned int* bpart = nullptr;
  RFD_CUDA(tmp.alloc(&bpart, size_t(rfd::bbox_chunks(n, batch, p->sms)) * batch * 6 + batch));
  rfd::launch_bbox(dev_xyz, bbox, bpart, n, batch, p->sms, st);
  if (world > 1) {  // one centre for the whole cloud: merge the shards' boxes
    double *send = nullptr, *recv = nullptr;
    RFD_CUDA(tmp.alloc(&send, size_t(7)));
    RFD_CUDA(tmp.alloc(&recv, size_t(7) * world));
    rfd::launch_bbox_export(bbox, n, send, st);
    rfd_status xs = exchange(p, send, recv, 7, st);
    if (xs != RFD_OK) return xs;
    rfd::launch_bbox_merge(recv, world, bbox, st);
    std::vector<double> h(size_t(7) * world);
    RFD_CUDA(cudaMemcpyAsync(h.data(), recv, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    RFD_CUDA(cudaStreamSynchronize(st));
    p->n_total = 0;
    for (int q = 0; q < world; ++q) p->n_total += int64_t(h[size_t(q) * 7 + 6]);
  }
  rfd::launch_freq(p->omega4, p->omega_rad4, p->nu, p->flags, m, seed, eps, RFD_TRUNCATION_R, cached_c_r(), st);

  // a4: Gram on the tensor cores (tcgen05, fp16 hi/lo split): directly over
  // the points, or -- large single clouds -- over a spread grid (k_nufft.cu),
  // sized from the bounding box and omega read back here
  rfd::NufftGrid ng{};
  bool spread = false;
  int known_sym = -1;  // the core's route, once the frequency flags are read back
  const int spread_mode = gram_spread_mode();
  if (spread_mode != 0 && batch == 1 && rfd::gram_tc_pairs(m) &&
      (spread_mode == 2 || n >= kSpreadMinPoints)) {
    HostSlot* h = nullptr;
    const rfd_status hs = host_slot(&h);
    if (hs != RFD_OK) return hs;
    unsigned int* hb = reinterpret_cast<unsigned int*>(h->buf + kSlotBox);
    int* hf = reinterpret_cast<int*>(h->buf + kSlotFlags);
    float4* hom = reinterpret_cast<float4*>(h->buf + kSlotOmega);
    gather_readback_kernel<<<1, 256, 0, st>>>(bbox, p->flags, p->omega4, m, h->buf);
    RFD_CUDA(cudaGetLastError());
    const rfd_status ws = slot_wait(h, st);
    if (ws != RFD_OK) return ws;
    known_sym = (hf[0] & 1) ? 0 : 1;
    spread = rfd::nufft_grid(hb, hom, m, n, &ng) &&
             (spread_mode == 2 || (ng.nodes * kSpreadRatio <= n && n >= kSpreadMinPoints));
  }
  double* Gdst = p->G;
  double* parts = nullptr;
  if (world > 1) {  // this shard's partial, all-gathered, summed in rank order
    RFD_CUDA(tmp.alloc(&Gdst, rr));
    RFD_CUDA(tmp.alloc(&parts, rr * world));
  }
  if (spread) {  // the packing also counts the points into the grid's cells
    unsigned char* ws = nullptr;
    RFD_CUDA(tmp.alloc(&ws, rfd::nufft_workspace_bytes(ng, n, m, p->sms)));
    rfd::CellCount cc{};
    RFD_CUDA(rfd::nufft_cell_count(ng, n, m, p->sms, ws, &cc, st));
    // (the host's first launch after its wait: the packing -- then the grid's
    // zeroing and the phi^ tables on the side stream beside it, off the
    // critical path: 10-13 us at cfg 5)
    HostSlot* h = nullptr;
    const rfd_status hs = host_slot(&h);
    if (hs != RFD_OK) return hs;
    RFD_CUDA(cudaEventRecord(h->ev_src, st));  // (after the workspace's allocation)
    rfd::launch_pack_points(dev_xyz, bbox, p->pts, p->pts16, nullptr, n, p->centre, n, batch, &cc,
                            st);
    RFD_CUDA(cudaStreamWaitEvent(h->side, h->ev_src, 0));
    RFD_CUDA(rfd::launch_nufft_side(p->omega_rad4, m, n, ng, p->sms, ws, h->side));
    RFD_CUDA(cudaEventRecord(h->ev_join, h->side));
    RFD_CUDA(rfd::launch_gram_nufft(p->pts, n, p->omega_rad4, m, ng, p->sms, ws, Gdst, st,
                                    h->ev_join));
  } else {  // the packing writes the Gram's point layout into its workspace
    const rfd::GramGeom gg = rfd::gram_tc_geometry(m, n, batch, p->sms);
    float* gpart = nullptr;
    RFD_CUDA(tmp.alloc(&gpart, rfd::gram_tc_partial_elems(gg, batch)));
    int64_t gper = 0;
    float* gpts = rfd::gram_points(gg, batch, gpart, &gper);
    rfd::launch_pack_points(dev_xyz, bbox, p->pts, p->pts16, gpts, gper, p->centre, n, batch,
                            nullptr, st);
    rfd::launch_gram_tc(p->omega_rad4, m, n, batch, gg, gpart, Gdst, st);
  }
  p->gram_nodes = spread ? ng.nodes : 0;
  if (world > 1) {
    rfd_status xs = exchange(p, Gdst, parts, rr, st);
    if (xs != RFD_OK) return xs;
    rfd::launch_sum_parts(parts, world, int64_t(rr), p->G, st);
  }

  if (before_core) {
    const rfd_status hs = before_core(p);
    if (hs != RFD_OK) return hs;
  }

  // a5: core
  {
    int sc = 0, sym = 1;
    const rfd_status cs =
        core_impl(p, p->nu, p->flags, lambda, p->C, &sc, &sym, st, known_sym, defer_core);
    if (cs != RFD_OK) return cs;
    p->scaling = sc;
    p->symmetric = sym;
  }

  guard.keep = true;
  *plan_out = p;
  return RFD_OK;
}

// NEXT-4: new (eps, lambda) on the stored G (independent of both,
// PAPER.md:337): a2 and a5 only.  Computed into fresh buffers and swapped in
// on success, so the plan is untouched on error.  The results are copied into
// the plan's existing buffers (device addresses unchanged: CUDA graphs that
// captured rfd_integrate on this plan stay valid and see the new core).
rfd_status reparam_impl(rfd_plan* p, double eps, double lambda, cudaStream_t st) {
  if (!p) return fail(RFD_EINVAL, "plan is NULL");
  if (!(eps > 0.0) || !isfinite(eps)) return fail(RFD_EINVAL, "eps must be finite and > 0");
  if (!isfinite(lambda)) return fail(RFD_EINVAL, "lambda must be finite");
  p->stream = st;
  const size_t rr = size_t(p->r) * p->r;
  double *nu = nullptr, *C = nullptr;
  int* flags = nullptr;
  struct Owned {
    double **nu, **C;
    int** flags;
    cudaStream_t s;
    ~Owned() {
      dfree(*nu, s);
      dfree(*C, s);
      dfree(*flags, s);
    }
  } owned{&nu, &C, &flags, st};
  RFD_CUDA(dalloc(&nu, size_t(p->m), st));
  RFD_CUDA(dalloc(&C, rr * p->batch, st));
  RFD_CUDA(dalloc(&flags, size_t(8), st));
  RFD_CUDA(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st));
  rfd::launch_nu(p->omega4, nu, flags, p->m, eps, cached_c_r(), st);
  int sc = 0, sym = 1;
  const rfd_status cs = core_impl(p, nu, flags, lambda, C, &sc, &sym, st);
  if (cs != RFD_OK) return cs;
  RFD_CUDA(cudaMemcpyAsync(p->nu, nu, size_t(p->m) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  RFD_CUDA(cudaMemcpyAsync(p->C, C, rr * p->batch * sizeof(double), cudaMemcpyDeviceToDevice, st));
  RFD_CUDA(cudaMemcpyAsync(p->flags, flags, 8 * sizeof(int), cudaMemcpyDeviceToDevice, st));
  p->eps = eps;
  p->lambda = lambda;
  p->scaling = sc;
  p->symmetric = sym;
  return RFD_OK;
}

// NEXT-3: the k smallest eigenvalues of exp(lambda W~) per cloud from the
// plan's G and nu (symmetric route: all nu > 0).
rfd_status spectrum_impl(rfd_plan* p, int k, double* out, cudaStream_t st) {
  if (!p) return fail(RFD_EINVAL, "plan is NULL");
  if (!out) return fail(RFD_EINVAL, "out is NULL");
  if (k < 1 || int64_t(k) > p->n_total) return fail(RFD_EINVAL, "k must be in [1, n]");
  if (!p->symmetric)
    return fail(RFD_EINVAL, "spectrum needs all nu > 0 (symmetric route D^1/2 G D^1/2)");
  p->stream = st;
  const int r = p->r, B = p->batch;
  TempBuffers tmp(st);
  double *W = nullptr, *P = nullptr, *dg = nullptr, *of = nullptr, *mu = nullptr, *o = nullptr;
  unsigned int* bar = nullptr;
  RFD_CUDA(tmp.alloc(&W, size_t(B) * r * r));
  RFD_CUDA(tmp.alloc(&P, size_t(B) * r));
  RFD_CUDA(tmp.alloc(&dg, size_t(B) * r));
  RFD_CUDA(tmp.alloc(&of, size_t(B) * r));
  RFD_CUDA(tmp.alloc(&mu, size_t(B) * r));
  RFD_CUDA(tmp.alloc(&o, size_t(B) * k));
  RFD_CUDA(tmp.alloc(&bar, size_t(2)));
  RFD_CUDA(rfd::launch_spectrum(p->G, p->nu, p->m, B, p->n_total, p->lambda, k, W, P, dg, of, mu, bar,
                                o, st));
  RFD_CUDA(cudaMemcpyAsync(out, o, size_t(B) * k * sizeof(double), cudaMemcpyDefault, st));
  RFD_CUDA(cudaStreamSynchronize(st));
  return RFD_OK;
}

rfd_status ensure_workspace(rfd_plan* p, int d, cudaStream_t st) {
  if (p->ws_d >= d) return RFD_OK;
  dfree(p->s_partial, st);
  dfree(p->S, st);
  dfree(p->S_parts, st);
  dfree(p->Y, st);
  p->ws_d = 0;
  const int ranges = rfd::pass1_tc_ranges(p->m, p->n, p->batch, p->sms);
  // pass-1 partials: ranges x r x (column chunk <= 64)
  const size_t part = size_t(p->batch) * ranges * p->r * size_t(d < 64 ? d : 64);
  RFD_CUDA(dalloc(&p->s_partial, part, st));
  RFD_CUDA(dalloc(&p->S, size_t(p->batch) * p->r * d, st));
  RFD_CUDA(dalloc(&p->Y, size_t(p->batch) * p->r * d, st));
  if (p->world > 1) RFD_CUDA(dalloc(&p->S_parts, size_t(p->world) * p->r * d, st));
  p->ws_d = d;
  return RFD_OK;
}

// narrow fields: the whole inference in one cooperative SIMT launch
// (k_small.cu) for d = 1, batched, tiny and large clouds; single clouds of
// 4097 .. 65536 points with 2 <= d <= 4 are faster on the tensor-core passes
// (measured, graph replay: cfg 2 d = 3 16.1 vs 24.2 us; 18,944 points d = 3
// (barycenter) faster too; cfg 4 (200k) even; at 4M points d = 3 the narrow
// kernel wins: its contraction costs 2d FMA, the passes' split and MMA a
// fixed 16 columns).  RFD_NARROW=0 / 2 force either side (tests).
bool use_narrow(const rfd_plan* p, int d) {
  const char* ne = getenv("RFD_NARROW");
  const int narrow_env = (ne && ne[0]) ? atoi(ne) : 1;
  return d <= 4 && p->world == 1 && narrow_env != 0 &&
         (narrow_env == 2 || d == 1 || p->batch > 1 || p->n <= 4096 || p->n > 65536);
}

// Small r (<= 128) with d in one chunk and few partials: a7 (S reduction and
// Y = C^ S) runs fused in pass 2's prologue -- two launches fewer per call
// (every pass-2 CTA re-reduces its cloud's partials, hence the bound).
bool fuse_a7(const rfd_plan* p, int d, int ranges) {
  return p->world == 1 && p->r <= 128 && d <= 64 && int64_t(ranges) * p->r * d <= 16384;
}

// a6 (+ the S reduction unless fused): pass 1 on the tensor cores takes up to
// 64 columns per launch (MMA N = the chunk's columns): the features are
// regenerated once per chunk (NEXT-2).  Needs the plan's points, omega and
// workspace (ensure_workspace) but not its core.
void pass1_part(rfd_plan* p, const float* F, int d, cudaStream_t st) {
  const int ranges = rfd::pass1_tc_ranges(p->m, p->n, p->batch, p->sms);
  const bool fuse = fuse_a7(p, d, ranges);
  const int w1 = 64;
  for (int c0 = 0; c0 < d; c0 += w1) {
    const int dc = (d - c0 < w1) ? d - c0 : w1;
    rfd::launch_pass1_tc(p->pts16, p->omega_rad4, p->m, p->n, p->batch, p->sms, ranges, F, d, c0,
                         dc, p->s_partial, st);
    if (!fuse) rfd::launch_reduce_S(p->s_partial, p->m, p->batch, ranges, d, c0, dc, p->S, st);
  }
}

// the rest of the inference after pass1_part: the shards' S exchange, a7
// (unless fused into pass 2) and a8
rfd_status tail_part(rfd_plan* p, const float* F, int d, float* out, cudaStream_t st) {
  const int ranges = rfd::pass1_tc_ranges(p->m, p->n, p->batch, p->sms);
  const bool fuse = fuse_a7(p, d, ranges);
  if (p->world > 1) {  // S = sum over the shards' partials, rank order
    rfd_status xs = exchange(p, p->S, p->S_parts, size_t(p->r) * d, st);
    if (xs != RFD_OK) return xs;
    rfd::launch_sum_parts(p->S_parts, p->world, int64_t(p->r) * d, p->S, st);
  }
  if (!fuse) rfd::launch_core_apply(p->C, p->S, p->m, p->batch, d, p->Y, st);
  // a8: pass 2 on the tensor cores takes up to 64 columns per launch (MMA N =
  // the chunk's columns): the features are regenerated once per chunk (NEXT-2)
  const int w2 = rfd::pass2_tc_width(p->m);
  for (int c0 = 0; c0 < d; c0 += w2) {
    const int dc = (d - c0 < w2) ? d - c0 : w2;
    rfd::launch_pass2_tc(p->pts, p->omega_rad4, p->m, p->n, p->batch, p->sms, p->Y, F, out, d, c0,
                         dc, fuse ? p->s_partial : nullptr, ranges, p->C, p->S, p->Y, st);
  }
  RFD_CUDA(cudaGetLastError());
  p->last_d = d;
  return RFD_OK;
}

rfd_status check_field(const float* F, int d, const float* out) {
  if (!F || !out) return fail(RFD_EINVAL, "F/out is NULL");
  if (d < 1) return fail(RFD_EINVAL, "d must be >= 1");
  if (reinterpret_cast<uintptr_t>(F) % 16 != 0 || reinterpret_cast<uintptr_t>(out) % 16 != 0)
    return fail(RFD_EINVAL, "F/out must be 16-byte aligned");
  return RFD_OK;
}

rfd_status integrate_impl(rfd_plan* p, const float* F, int d, float* out, cudaStream_t st) {
  if (!p) return fail(RFD_EINVAL, "plan is NULL");
  const rfd_status cf = check_field(F, d, out);
  if (cf != RFD_OK) return cf;
  p->stream = st;
  rfd_status rs = ensure_workspace(p, d, st);
  if (rs != RFD_OK) return rs;
  if (use_narrow(p, d)) {
    const size_t need = rfd::small_partial_elems(p->m, p->n, p->batch, d, p->sms);
    if (p->small_part_elems < need) {
      dfree(p->small_part, st);
      p->small_part_elems = 0;
      RFD_CUDA(dalloc(&p->small_part, need, st));
      p->small_part_elems = need;
    }
    RFD_CUDA(rfd::launch_integrate_small(p->pts, p->omega_rad4, p->m, p->n, p->batch, p->sms, F, d,
                                         out, p->C, p->small_part, p->S, p->Y, p->bar, st));
    p->last_d = d;
    return RFD_OK;
  }
  pass1_part(p, F, d, st);
  return tail_part(p, F, d, out, st);
}

// One-shot GFI on device fields (rfd_gfi): plan and inference with pass 1
// (which needs only the points, omega and the field) on a second stream
// beside the plan's core -- the core's small DMMA GEMMs (128 threads, no
// TMEM) fit on the SMs next to pass 1's persistent CTAs.  Same kernels and
// results as rfd_plan_create + rfd_integrate.
rfd_status gfi_impl(const float* points, int64_t n, double eps, double lambda, int m,
                    uint64_t seed, const float* F, int d, float* out, cudaStream_t st,
                    rfd_plan** plan_out) {
  const rfd_status cf = check_field(F, d, out);
  if (cf != RFD_OK) return cf;
  if (!is_device_pointer(F) || !is_device_pointer(out))
    return fail(RFD_EINVAL, "rfd_gfi: F and out must be device memory (rfd_gfi_host for host)");
  rfd_plan* p = nullptr;
  bool early = false;
  auto hook = [&](rfd_plan* q) -> rfd_status {
    q->stream = st;
    if (use_narrow(q, d)) return RFD_OK;  // one launch after the plan
    rfd_status rs = ensure_workspace(q, d, st);
    if (rs != RFD_OK) return rs;
    if (!q->aux) {
      // pass 1 (persistent, one CTA per SM) must be placed before the core's
      // GEMM CTAs, which are launched right behind it on `st` now that the
      // powers of Z no longer wait for the host: two GEMM CTAs on one SM
      // leave no room for pass 1's CTA there.  The higher-priority stream's
      // pending CTAs are dispatched first.
      int lo = 0, hi = 0;
      RFD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      RFD_CUDA(cudaStreamCreateWithPriority(&q->aux, cudaStreamNonBlocking, hi));
    }
    if (!q->ev[0]) RFD_CUDA(cudaEventCreateWithFlags(&q->ev[0], cudaEventDisableTiming));
    if (!q->ev[1]) RFD_CUDA(cudaEventCreateWithFlags(&q->ev[1], cudaEventDisableTiming));
    RFD_CUDA(cudaEventRecord(q->ev[0], st));
    RFD_CUDA(cudaStreamWaitEvent(q->aux, q->ev[0], 0));
    pass1_part(q, F, d, q->aux);
    RFD_CUDA(cudaGetLastError());
    RFD_CUDA(cudaEventRecord(q->ev[1], q->aux));
    early = true;
    return RFD_OK;
  };
  // the core's overflow check waits until the inference is enqueued behind it
  // (no idle GPU while the host reads the flag back)
  const rfd_status cs =
      create_impl(points, 1, n, eps, lambda, m, seed, nullptr, st, &p, hook, true);
  if (cs != RFD_OK) return cs;
  rfd_status rs = RFD_OK;
  if (early) {
    rs = cudaStreamWaitEvent(st, p->ev[1], 0) == cudaSuccess ? RFD_OK
                                                            : fail(RFD_ECUDA, "rfd_gfi: event wait");
    if (rs == RFD_OK) rs = tail_part(p, F, d, out, st);
  } else {
    rs = integrate_impl(p, F, d, out, st);
  }
  const rfd_status fs = core_finish(p);  // (out is unspecified on RFD_ERANGE)
  if (rs == RFD_OK) rs = fs;
  if (rs != RFD_OK || !plan_out) {
    free_plan(p, false);  // stream-ordered (after the aux stream's work)
    if (plan_out) *plan_out = nullptr;
    return rs;
  }
  *plan_out = p;
  return RFD_OK;
}

// Host buffers, pipelined: the field travels in K point-range chunks.  The
// H2D copy of chunk c (copy stream) overlaps pass 1 of the chunks before it
// (each chunk's pass 1 is its own launch writing its own partial slots; S =
// the fixed-order sum of all slots, chunk-major); pass 2 runs per chunk too
// and the D2H copy of chunk c (second copy stream) overlaps pass 2 of the
// chunks after it.  `h2d_issued`: the caller has already enqueued the H2D
// copies into p->stage on cs_h2d with events ev[0..K) (rfd_gfi_host starts
// them before the plan exists).  Single-cloud plans, d <= 64 (one pass-1
// column chunk); otherwise the serial path.
constexpr int kPipeChunks = 8;

int64_t pipe_chunk_begin(int64_t n, int c) {
  // boundaries at multiples of 2048 points (whole pass-1 groups and pass-2
  // tiles; F blocks stay 16-byte aligned for any d)
  return std::min<int64_t>(n, ((n * c / kPipeChunks) + 2047) / 2048 * 2048);
}

rfd_status pipe_streams(rfd_plan* p) {
  if (!p->cs_h2d) RFD_CUDA(cudaStreamCreateWithFlags(&p->cs_h2d, cudaStreamNonBlocking));
  if (!p->cs_d2h) RFD_CUDA(cudaStreamCreateWithFlags(&p->cs_d2h, cudaStreamNonBlocking));
  for (cudaEvent_t& e : p->ev)
    if (!e) RFD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return RFD_OK;
}

rfd_status ensure_stage(rfd_plan* p, size_t elems, cudaStream_t st) {
  if (p->stage_elems >= elems) return RFD_OK;
  dfree(p->stage, st);
  p->stage_elems = 0;
  RFD_CUDA(dalloc(&p->stage, elems, st));
  p->stage_elems = elems;
  return RFD_OK;
}

// enqueue the H2D copies of F's chunks on cs_h2d (after `st`'s prior work)
rfd_status pipe_h2d(rfd_plan* p, const float* F_host, int d, cudaStream_t st) {
  RFD_CUDA(cudaEventRecord(p->ev[2 * kPipeChunks], st));
  RFD_CUDA(cudaStreamWaitEvent(p->cs_h2d, p->ev[2 * kPipeChunks], 0));
  for (int c = 0; c < kPipeChunks; ++c) {
    const int64_t a = pipe_chunk_begin(p->n, c), b = pipe_chunk_begin(p->n, c + 1);
    if (b > a)
      RFD_CUDA(cudaMemcpyAsync(p->stage + a * d, F_host + a * d, size_t(b - a) * d * sizeof(float),
                               cudaMemcpyHostToDevice, p->cs_h2d));
    RFD_CUDA(cudaEventRecord(p->ev[c], p->cs_h2d));
  }
  return RFD_OK;
}

rfd_status integrate_host_pipelined(rfd_plan* p, const float* F_host, int d, float* out_host,
                                    bool h2d_issued, cudaStream_t st) {
  p->stream = st;
  rfd_status rs = ensure_workspace(p, d, st);
  if (rs != RFD_OK) return rs;
  const int r = p->r;
  // partial slots of every chunk's pass 1
  int rg[kPipeChunks];
  int64_t slots = 0;
  for (int c = 0; c < kPipeChunks; ++c) {
    const int64_t nc = pipe_chunk_begin(p->n, c + 1) - pipe_chunk_begin(p->n, c);
    rg[c] = nc > 0 ? rfd::pass1_tc_ranges(p->m, nc, 1, p->sms) : 0;
    slots += rg[c];
  }
  const size_t need = size_t(slots) * r * d;
  if (p->pipe_partial_elems < need) {
    dfree(p->pipe_partial, st);
    p->pipe_partial_elems = 0;
    RFD_CUDA(dalloc(&p->pipe_partial, need, st));
    p->pipe_partial_elems = need;
  }
  if (!h2d_issued) {
    rs = pipe_h2d(p, F_host, d, st);
    if (rs != RFD_OK) return rs;
  }
  // a6 per chunk, each as soon as its field has arrived
  int64_t slot = 0;
  for (int c = 0; c < kPipeChunks; ++c) {
    const int64_t a = pipe_chunk_begin(p->n, c), nc = pipe_chunk_begin(p->n, c + 1) - a;
    if (nc <= 0) continue;
    RFD_CUDA(cudaStreamWaitEvent(st, p->ev[c], 0));
    rfd::launch_pass1_tc(p->pts16 + (a / 16) * 48, p->omega_rad4, p->m, nc, 1, p->sms, rg[c],
                         p->stage + a * d, d, 0, d, p->pipe_partial + size_t(slot) * r * d, st);
    slot += rg[c];
  }
  // a7
  rfd::launch_reduce_S(p->pipe_partial, p->m, 1, int(slots), d, 0, d, p->S, st);
  if (p->world > 1) {
    rs = exchange(p, p->S, p->S_parts, size_t(r) * d, st);
    if (rs != RFD_OK) return rs;
    rfd::launch_sum_parts(p->S_parts, p->world, int64_t(r) * d, p->S, st);
  }
  rfd::launch_core_apply(p->C, p->S, p->m, 1, d, p->Y, st);
  // a8 per chunk (in place in the stage), each chunk's D2H right behind it
  const int w2 = rfd::pass2_tc_width(p->m);
  for (int c = 0; c < kPipeChunks; ++c) {
    const int64_t a = pipe_chunk_begin(p->n, c), nc = pipe_chunk_begin(p->n, c + 1) - a;
    if (nc <= 0) continue;
    float* f = p->stage + a * d;
    for (int c0 = 0; c0 < d; c0 += w2) {
      const int dc = (d - c0 < w2) ? d - c0 : w2;
      rfd::launch_pass2_tc(p->pts + a, p->omega_rad4, p->m, nc, 1, p->sms, p->Y, f, f, d, c0, dc,
                           nullptr, 0, p->C, p->S, p->Y, st);
    }
    RFD_CUDA(cudaEventRecord(p->ev[kPipeChunks + c], st));
    RFD_CUDA(cudaStreamWaitEvent(p->cs_d2h, p->ev[kPipeChunks + c], 0));
    RFD_CUDA(cudaMemcpyAsync(out_host + a * d, f, size_t(nc) * d * sizeof(float),
                             cudaMemcpyDeviceToHost, p->cs_d2h));
  }
  // the caller's stream resumes after the last copy (stream semantics)
  RFD_CUDA(cudaEventRecord(p->ev[2 * kPipeChunks + 1], p->cs_d2h));
  RFD_CUDA(cudaStreamWaitEvent(st, p->ev[2 * kPipeChunks + 1], 0));
  RFD_CUDA(cudaGetLastError());
  p->last_d = d;
  return RFD_OK;
}

// NEXT-1: Alg. 1 with FM_K = rfd_integrate on the
// N x k field of the k distributions (k_sinkhorn.cu).
rfd_status barycenter_impl(rfd_plan* p, const float* mu_in, const float* area,
                           const double* alpha, int k, int max_iter, double tol, float* out,
                           int32_t* iters_out, cudaStream_t st) {
  if (!p) return fail(RFD_EINVAL, "plan is NULL");
  if (p->batch != 1) return fail(RFD_EINVAL, "barycenter needs a single-cloud plan");
  if (p->world != 1) return fail(RFD_EINVAL, "barycenter: sharded plans are not supported");
  if (!mu_in || !area || !alpha || !out) return fail(RFD_EINVAL, "NULL argument");
  if (k < 1 || k > 16) return fail(RFD_EINVAL, "k must be in [1, 16]");
  if (max_iter < 1) return fail(RFD_EINVAL, "max_iter must be >= 1");
  if (!(tol >= 0.0)) return fail(RFD_EINVAL, "tol must be >= 0");
  double asum = 0.0;
  for (int i = 0; i < k; ++i) {
    if (!(alpha[i] > 0.0) || !isfinite(alpha[i])) return fail(RFD_EINVAL, "alpha must be > 0");
    asum += alpha[i];
  }
  if (fabs(asum - 1.0) > 1e-6) return fail(RFD_EINVAL, "alpha must sum to 1");
  if (!is_device_pointer(mu_in) || !is_device_pointer(area) || !is_device_pointer(out))
    return fail(RFD_EINVAL, "mu, area and out must be device pointers");
  p->stream = st;
  const int64_t n = p->n;
  const char* fe = getenv("RFD_BARY_FUSED");  // "0": the unfused path (tests compare the two)
  const bool no_fused = fe && fe[0] == '0';
  if (!no_fused && p->m <= 32 && k <= 4 && n <= rfd::bary_fused_max_points(p->sms)) {
    // the whole loop in one launch, feature rows cached on chip (k_bary_fused.cu)
    TempBuffers tmp(st);
    const int ctas = int((n + 511) / 512);
    double *part = nullptr, *S = nullptr, *red = nullptr;
    int* status = nullptr;
    RFD_CUDA(tmp.alloc(&part, size_t(2) * ctas * p->r * k));
    RFD_CUDA(tmp.alloc(&S, size_t(p->r) * k));
    RFD_CUDA(tmp.alloc(&red, size_t(3) * ctas));
    RFD_CUDA(tmp.alloc(&status, size_t(2)));
    RFD_CUDA(cudaMemsetAsync(status, 0, 2 * sizeof(int), st));
    RFD_CUDA(rfd::launch_bary_fused(p->pts, p->omega_rad4, p->C, mu_in, area, alpha, p->m, k, n,
                                    max_iter, tol, part, S, red, p->bar, status, out, st));
    int hs[2] = {0, 0};
    RFD_CUDA(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
    RFD_CUDA(cudaStreamSynchronize(st));
    if (hs[0])
      return fail(RFD_ERANGE, "barycenter: non-finite iterate at iteration " + std::to_string(hs[1]));
    if (iters_out) *iters_out = hs[1];
    return RFD_OK;
  }
  const size_t nk = size_t(n) * k;
  const int nb = rfd::bary_blocks(n);
  TempBuffers tmp(st);
  float *Mt = nullptr, *X = nullptr, *Y = nullptr;
  double *V = nullptr, *W = nullptr, *mu = nullptr, *sc = nullptr, *part = nullptr,
         *dpart = nullptr, *red = nullptr;
  int* flag = nullptr;
  RFD_CUDA(tmp.alloc(&Mt, nk));
  RFD_CUDA(tmp.alloc(&X, nk));
  RFD_CUDA(tmp.alloc(&Y, nk));
  RFD_CUDA(tmp.alloc(&V, nk));
  RFD_CUDA(tmp.alloc(&W, nk));
  RFD_CUDA(tmp.alloc(&mu, size_t(n)));
  RFD_CUDA(tmp.alloc(&sc, size_t(16)));
  RFD_CUDA(tmp.alloc(&part, size_t(nb) * 16));
  RFD_CUDA(tmp.alloc(&dpart, size_t(nb)));
  RFD_CUDA(tmp.alloc(&red, size_t(2)));
  RFD_CUDA(tmp.alloc(&flag, size_t(1)));
  RFD_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  rfd::launch_bary_init(mu_in, area, n, k, Mt, V, mu, part, sc, flag, X, st);  // X = a v s
  int it = 0;
  for (it = 1; it <= max_iter; ++it) {
    rfd_status rs = integrate_impl(p, X, k, Y, st);                   // FM_K(a v^i) s_i
    if (rs != RFD_OK) return rs;
    rfd::launch_bary_step1(area, Mt, Y, sc, n, k, W, part, st);       // w^i
    rfd::launch_bary_input(area, W, part, n, k, sc, flag, X, st);     // X = a w s
    rs = integrate_impl(p, X, k, Y, st);                               // FM_K(a w^i) s_i
    if (rs != RFD_OK) return rs;
    rfd::launch_bary_step2(area, Y, alpha, sc, n, k, V, mu, dpart, part, red, flag, st);
    rfd::launch_bary_input(area, V, part, n, k, sc, flag, X, st);     // next X = a v s
    if (tol > 0.0 || it == max_iter) {
      double delta = 0.0;
      int hflag = 0;
      RFD_CUDA(cudaMemcpyAsync(&delta, red, sizeof(double), cudaMemcpyDeviceToHost, st));
      RFD_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
      RFD_CUDA(cudaStreamSynchronize(st));
      if (hflag) return fail(RFD_ERANGE, "barycenter: non-finite iterate at iteration " +
                                             std::to_string(it));
      if (tol > 0.0 && delta < tol) break;
    }
  }
  if (it > max_iter) it = max_iter;
  rfd::launch_bary_finish(area, mu, n, dpart, red + 1, out, st);
  RFD_CUDA(cudaGetLastError());
  RFD_CUDA(cudaStreamSynchronize(st));
  if (iters_out) *iters_out = it;
  return RFD_OK;
}

// interleaved feature index (2k + t) for the paper's blocked index (t m + k)
inline int interleaved(int a, int m) { return a < m ? 2 * a : 2 * (a - m) + 1; }

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

rfd_status rfd_plan_create(const float* points, int64_t n, double eps, double lambda, int32_t m,
                           uint64_t seed, rfd_stream stream, rfd_plan** plan_out) {
  return create_impl(points, 1, n, eps, lambda, m, seed, nullptr,
                     reinterpret_cast<cudaStream_t>(stream), plan_out);
}

rfd_status rfd_plan_create_sharded(const float* points, int64_t n_local, double eps, double lambda,
                                   int32_t m, uint64_t seed, const rfd_shard* shard,
                                   rfd_stream stream, rfd_plan** plan_out) {
  if (!shard) return fail(RFD_EINVAL, "shard is NULL");
  return create_impl(points, 1, n_local, eps, lambda, m, seed, shard,
                     reinterpret_cast<cudaStream_t>(stream), plan_out);
}

rfd_status rfd_plan_create_batched(const float* points, int32_t batch, int64_t n, double eps,
                                   double lambda, int32_t m, uint64_t seed, rfd_stream stream,
                                   rfd_plan** plan_out) {
  return create_impl(points, batch, n, eps, lambda, m, seed, nullptr,
                     reinterpret_cast<cudaStream_t>(stream), plan_out);
}

rfd_status rfd_plan_reparam(rfd_plan* plan, double eps, double lambda, rfd_stream stream) {
  return reparam_impl(plan, eps, lambda, reinterpret_cast<cudaStream_t>(stream));
}

rfd_status rfd_barycenter(rfd_plan* plan, const float* mu, const float* area, const double* alpha,
                          int32_t k, int32_t max_iter, double tol, float* out, int32_t* iters,
                          rfd_stream stream) {
  return barycenter_impl(plan, mu, area, alpha, k, max_iter, tol, out, iters,
                         reinterpret_cast<cudaStream_t>(stream));
}

rfd_status rfd_plan_spectrum(rfd_plan* plan, int32_t k, double* out, rfd_stream stream) {
  return spectrum_impl(plan, k, out, reinterpret_cast<cudaStream_t>(stream));
}

rfd_status rfd_integrate(rfd_plan* plan, const float* F, int32_t d, float* out,
                         rfd_stream stream) {
  return integrate_impl(plan, F, d, out, reinterpret_cast<cudaStream_t>(stream));
}

rfd_status rfd_gfi(const float* points, int64_t n, double eps, double lambda, int32_t m,
                   uint64_t seed, const float* F, int32_t d, float* out, rfd_stream stream,
                   rfd_plan** plan_out) {
  return gfi_impl(points, n, eps, lambda, m, seed, F, d, out,
                  reinterpret_cast<cudaStream_t>(stream), plan_out);
}

rfd_status rfd_integrate_host(rfd_plan* plan, const float* F_host, int32_t d, float* out_host,
                              rfd_stream stream) {
  if (!plan) return fail(RFD_EINVAL, "plan is NULL");
  if (!F_host || !out_host) return fail(RFD_EINVAL, "F/out is NULL");
  if (d < 1) return fail(RFD_EINVAL, "d must be >= 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t elems = size_t(plan->batch) * plan->n * d;
  RFD_CUDA(ensure_stage(plan, elems, st) == RFD_OK ? cudaSuccess : cudaErrorMemoryAllocation);
  if (plan->batch == 1 && d > 4 && d <= 64 && plan->n >= 2048 * kPipeChunks) {
    const rfd_status ps = pipe_streams(plan);
    if (ps != RFD_OK) return ps;
    return integrate_host_pipelined(plan, F_host, d, out_host, false, st);
  }
  RFD_CUDA(cudaMemcpyAsync(plan->stage, F_host, elems * sizeof(float), cudaMemcpyHostToDevice, st));
  rfd_status rs = integrate_impl(plan, plan->stage, d, plan->stage, st);
  if (rs != RFD_OK) return rs;
  RFD_CUDA(cudaMemcpyAsync(out_host, plan->stage, elems * sizeof(float), cudaMemcpyDeviceToHost, st));
  return RFD_OK;
}

rfd_status rfd_gfi_host(const float* points, int64_t n, double eps, double lambda, int32_t m,
                        uint64_t seed, const float* F_host, int32_t d, float* out_host,
                        rfd_stream stream, rfd_plan** plan_out) {
  if (plan_out) *plan_out = nullptr;
  if (!points || !F_host || !out_host) return fail(RFD_EINVAL, "NULL argument");
  if (d < 1) return fail(RFD_EINVAL, "d must be >= 1");
  if (n < 1) return fail(RFD_EINVAL, "n must be >= 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (d <= 4 || d > 64 || n < 2048 * kPipeChunks || is_device_pointer(points)) {  // nothing to overlap
    rfd_plan* p = nullptr;
    rfd_status rs = create_impl(points, 1, n, eps, lambda, m, seed, nullptr, st, &p);
    if (rs != RFD_OK) return rs;
    rs = rfd_integrate_host(p, F_host, d, out_host, stream);
    if (rs != RFD_OK || !plan_out) rfd_destroy(p);
    else *plan_out = p;
    return rs;
  }
  // The field's H2D copies start right behind the points' and run while the
  // plan (Gram, core) computes; pass 1 consumes each chunk as it lands.
  rfd_plan* stub = new rfd_plan();  // holds the streams, events and stage until the plan exists
  struct StubGuard {
    rfd_plan* s;
    ~StubGuard() {
      if (s) free_plan(s, false);
    }
  } sg{stub};
  stub->stream = st;
  stub->n = n;
  rfd_status rs = pipe_streams(stub);
  if (rs != RFD_OK) return rs;
  rs = ensure_stage(stub, size_t(n) * d, st);
  if (rs != RFD_OK) return rs;
  float* pts_dev = nullptr;
  RFD_CUDA(dalloc(&pts_dev, size_t(n) * 3, st));
  struct PtsGuard {
    float* p;
    cudaStream_t s;
    ~PtsGuard() { dfree(p, s); }
  } pg{pts_dev, st};
  RFD_CUDA(cudaEventRecord(stub->ev[2 * kPipeChunks], st));
  RFD_CUDA(cudaStreamWaitEvent(stub->cs_h2d, stub->ev[2 * kPipeChunks], 0));
  RFD_CUDA(cudaMemcpyAsync(pts_dev, points, size_t(n) * 3 * sizeof(float), cudaMemcpyHostToDevice,
                           stub->cs_h2d));
  RFD_CUDA(cudaEventRecord(stub->ev[2 * kPipeChunks + 1], stub->cs_h2d));
  rs = pipe_h2d(stub, F_host, d, stub->cs_h2d);
  if (rs != RFD_OK) return rs;
  RFD_CUDA(cudaStreamWaitEvent(st, stub->ev[2 * kPipeChunks + 1], 0));
  rfd_plan* p = nullptr;
  rs = create_impl(pts_dev, 1, n, eps, lambda, m, seed, nullptr, st, &p);
  if (rs != RFD_OK) {
    cudaStreamSynchronize(stub->cs_h2d);
    return rs;
  }
  // hand the streams, events and staged field over to the plan
  std::swap(p->stage, stub->stage);
  std::swap(p->stage_elems, stub->stage_elems);
  std::swap(p->cs_h2d, stub->cs_h2d);
  std::swap(p->cs_d2h, stub->cs_d2h);
  for (int i = 0; i < 2 * kPipeChunks + 2; ++i) std::swap(p->ev[i], stub->ev[i]);
  rs = integrate_host_pipelined(p, F_host, d, out_host, true, st);
  if (rs != RFD_OK || !plan_out) {
    free_plan(p, false);  // stream-ordered: the host does not wait for the step
  } else {
    *plan_out = p;
  }
  return rs;
}

void rfd_destroy(rfd_plan* plan) { free_plan(plan); }

const char* rfd_last_error(void) { return g_last_error.c_str(); }

rfd_status rfd_plan_info(const rfd_plan* p, rfd_plan_info_t* info) {
  if (!p || !info) return fail(RFD_EINVAL, "NULL argument");
  info->n = p->n;
  info->batch = p->batch;
  info->m = p->m;
  info->r = p->r;
  info->scaling = p->scaling;
  info->symmetric = p->symmetric;
  info->eps = p->eps;
  info->lambda = p->lambda;
  info->seed = p->seed;
  info->n_total = p->n_total;
  info->rank = p->rank;
  info->world = p->world;
  info->gram_nodes = p->gram_nodes;
  return RFD_OK;
}

rfd_status rfd_plan_export(const rfd_plan* p, rfd_field which, void* host_dst, size_t bytes) {
  if (!p || !host_dst) return fail(RFD_EINVAL, "NULL argument");
  const int m = p->m, r = p->r, B = p->batch, d = p->last_d;
  RFD_CUDA(cudaDeviceSynchronize());
  switch (which) {
    case RFD_OMEGA: {
      if (bytes != size_t(m) * 3 * sizeof(float)) return fail(RFD_EINVAL, "size mismatch");
      std::vector<float4> w(m);
      RFD_CUDA(cudaMemcpy(w.data(), p->omega4, m * sizeof(float4), cudaMemcpyDeviceToHost));
      float* o = static_cast<float*>(host_dst);
      for (int k = 0; k < m; ++k) {
        o[3 * k] = w[k].x;
        o[3 * k + 1] = w[k].y;
        o[3 * k + 2] = w[k].z;
      }
      return RFD_OK;
    }
    case RFD_NU:
      if (bytes != size_t(m) * sizeof(double)) return fail(RFD_EINVAL, "size mismatch");
      RFD_CUDA(cudaMemcpy(host_dst, p->nu, bytes, cudaMemcpyDeviceToHost));
      return RFD_OK;
    case RFD_GRAM:
    case RFD_CORE:
    case RFD_S:
    case RFD_Y: {
      // device state is in the centred basis: rotate back (rfd_export_rotate)
      const bool sq = which == RFD_GRAM || which == RFD_CORE;
      if (!sq && d < 1) return fail(RFD_EINVAL, "no integrate has run on this plan");
      const int cols = sq ? r : d;
      const size_t cnt = size_t(B) * r * cols;
      const size_t es = which == RFD_Y ? sizeof(float) : sizeof(double);
      if (bytes != cnt * es) return fail(RFD_EINVAL, "size mismatch");
      double* rot = nullptr;
      RFD_CUDA(cudaMalloc(&rot, cnt * sizeof(double)));
      rfd::launch_rotate(which == RFD_GRAM ? p->G : which == RFD_CORE ? p->C : which == RFD_S ? p->S : nullptr,
                         which == RFD_Y ? p->Y : nullptr, r, cols, B, sq, p->omega4, p->centre, rot,
                         nullptr);
      std::vector<double> tmp(cnt);
      const cudaError_t e1 = cudaMemcpy(tmp.data(), rot, cnt * sizeof(double), cudaMemcpyDeviceToHost);
      cudaFree(rot);
      RFD_CUDA(e1);
      for (int b = 0; b < B; ++b)
        for (int a = 0; a < r; ++a)
          for (int c = 0; c < cols; ++c) {
            const double v = tmp[(size_t(b) * r + interleaved(a, m)) * cols + (sq ? interleaved(c, m) : c)];
            const size_t o = (size_t(b) * r + a) * cols + c;
            if (which == RFD_Y)
              static_cast<float*>(host_dst)[o] = float(v);
            else
              static_cast<double*>(host_dst)[o] = v;
          }
      return RFD_OK;
    }
  }
  return fail(RFD_EINVAL, "unknown field");
}

uint64_t rfd_launch_count(void) { return g_launches.load(); }

rfd_status rfd_profile_enable(int on) {
  g_profiling.store(on ? 1 : 0);
  return RFD_OK;
}

rfd_status rfd_profile_only(const char* name) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_only = name ? name : "";
  return RFD_OK;
}

int32_t rfd_profile_read(rfd_profile_entry* entries, int32_t cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  // RFD_TIMELINE=path (instrumentation): also append every launch's start and
  // end (ms from the first recorded launch) -- the overlap of the streams
  if (const char* tl = getenv("RFD_TIMELINE")) {
    if (FILE* f = (tl[0] && !g_pending.empty()) ? fopen(tl, "a") : nullptr) {
      const cudaEvent_t t0 = g_pending.front().a;
      for (const Pending& pe : g_pending) {
        float s0 = 0.0f, s1 = 0.0f;
        cudaEventSynchronize(pe.b);
        cudaEventElapsedTime(&s0, t0, pe.a);
        cudaEventElapsedTime(&s1, t0, pe.b);
        fprintf(f, "%s %.4f %.4f\n", pe.name, s0, s1);
      }
      fprintf(f, "--\n");
      fclose(f);
    }
  }
  for (const Pending& pe : g_pending) {
    float ms = 0.0f;
    cudaEventSynchronize(pe.b);
    cudaEventElapsedTime(&ms, pe.a, pe.b);
    auto& agg = g_prof[pe.name];
    agg.first += 1;
    agg.second += ms;
    g_free_events.push_back(pe.a);
    g_free_events.push_back(pe.b);
  }
  g_pending.clear();
  int32_t i = 0;
  for (const auto& kv : g_prof) {
    if (i >= cap || !entries) break;
    strncpy(entries[i].name, kv.first.c_str(), sizeof(entries[i].name) - 1);
    entries[i].name[sizeof(entries[i].name) - 1] = '\0';
    entries[i].launches = kv.second.first;
    entries[i].total_ms = kv.second.second;
    ++i;
  }
  g_prof.clear();
  return i;
}

}  // extern "C"
