// Shared device/host infrastructure of libpmx_cuda.so (sm_100a only).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pmx.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libpmx_cuda is written for sm_100a (B200) only"
#endif

namespace pmx {

// ----------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PMX_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::pmx::Error(e_ == cudaErrorMemoryAllocation ? PMX_ERR_OUT_OF_MEMORY         \
                                                         : PMX_ERR_CUDA,                 \
                         std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

inline void require(bool ok, const char* msg) {
  if (!ok) throw Error(PMX_ERR_INVALID_ARGUMENT, msg);
}

// --------------------------------------------------------------- context
struct ProfEvent {
  const char* name;
  cudaEvent_t start, stop;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t copy_in = nullptr, copy_out = nullptr;  // pipelined host staging (created on first use)
  cudaStream_t copy_in2 = nullptr;                      // small pinned inputs by SM copy (PMX_SM_SMALL_COPIES)
  cudaStream_t aux = nullptr;  // high-priority side stream of the overlapped matcher (created on first use)
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;
  bool profiling = false;
  bool graphs = true;      // device-side loops as CUDA graphs (pmx_set_device_graphs)
  bool capturing = false;  // a graph body is being captured: no per-kernel event brackets
  std::vector<ProfEvent> prof;  // unresolved event pairs (pmx_profile_*)
  std::map<std::string, int64_t> counters;  // profiling counters (pmx_profile_get, total_ms = 0)
  std::map<std::string, unsigned long long*> dev_counters;  // device-side counters, read at pmx_profile_get
  // NCCL communicator of the edge-sharded backend (pmx_nccl_init; ncclComm_t)
  void* nccl_comm = nullptr;
  int nccl_rank = 0, nccl_nranks = 1;
};

// Device-side profiling counter `name` (allocated on first use, zeroed).
inline unsigned long long* dev_counter(Context& ctx, const char* name) {
  auto it = ctx.dev_counters.find(name);
  if (it != ctx.dev_counters.end()) return it->second;
  unsigned long long* p = nullptr;
  if (cudaMalloc(&p, sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  cudaMemsetAsync(p, 0, sizeof(unsigned long long), ctx.stream);
  ctx.dev_counters[name] = p;
  return p;
}

// CUDA-event bracket around one kernel launch on ctx.stream (when profiling).
struct ProfScope {
  Context& c;
  ProfEvent ev{nullptr, nullptr, nullptr};
  bool on;
  ProfScope(Context& ctx, const char* name) : c(ctx), on(ctx.profiling && !ctx.capturing) {
    if (!on) return;
    ev.name = name;
    cudaEventCreate(&ev.start);
    cudaEventCreate(&ev.stop);
    cudaEventRecord(ev.start, c.stream);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(ev.stop, c.stream);
    c.prof.push_back(ev);
  }
};

// Device scratch owned for the duration of one API call (stream-ordered).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) : bytes(n), s(st) {
    if (n) PMX_CUDA(cudaMallocAsync(&p, n, st));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p;
    bytes = o.bytes;
    s = o.s;
    o.p = nullptr;
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

inline void launch_check(Context& c, const char* what) {
  c.launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(PMX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Copies host arrays to scratch device memory when mem == HOST; passes
// device pointers through when mem == DEVICE.
struct Stager {
  Context& ctx;
  pmx_memory mem;
  std::vector<DevBuf> bufs;
  Stager(Context& c, pmx_memory m) : ctx(c), mem(m) {}
  template <class T>
  const T* in(const T* host_or_dev, size_t count) {
    if (host_or_dev == nullptr || mem == PMX_MEM_DEVICE || count == 0) return host_or_dev;
    bufs.emplace_back(sizeof(T) * count, ctx.stream);
    PMX_CUDA(cudaMemcpyAsync(bufs.back().p, host_or_dev, sizeof(T) * count, cudaMemcpyHostToDevice,
                             ctx.stream));
    return bufs.back().as<T>();
  }
  template <class T>
  T* inout(T* host_or_dev, size_t count) {
    return const_cast<T*>(in<T>(host_or_dev, count));
  }
  template <class T>
  T* out(T* host_or_dev, size_t count) {
    if (host_or_dev == nullptr || mem == PMX_MEM_DEVICE || count == 0) return host_or_dev;
    bufs.emplace_back(sizeof(T) * count, ctx.stream);
    return bufs.back().as<T>();
  }
  template <class T>
  void back(T* host, const T* dev, size_t count) {
    if (host == nullptr || mem == PMX_MEM_DEVICE || count == 0) return;
    PMX_CUDA(cudaMemcpyAsync(host, dev, sizeof(T) * count, cudaMemcpyDeviceToHost, ctx.stream));
  }
};

// ----------------------------------------------------------- device math
struct DSim3 {  // Sim(3) in FP64: x -> s R x + t (lie.hpp:36-70)
  double R[9];
  double t[3];
  double s;
};

inline DSim3 to_dsim3(const pmx_sim3& T) {
  DSim3 d;
  for (int i = 0; i < 9; ++i) d.R[i] = T.R[i];
  for (int i = 0; i < 3; ++i) d.t[i] = T.t[i];
  d.s = T.s;
  return d;
}

__host__ __device__ inline DSim3 sim3_mul(const DSim3& a, const DSim3& b) {  // lie.cpp:131-140
  DSim3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.R[3 * i + j] = a.R[3 * i] * b.R[j] + a.R[3 * i + 1] * b.R[3 + j] + a.R[3 * i + 2] * b.R[6 + j];
  r.s = a.s * b.s;
  for (int i = 0; i < 3; ++i)
    r.t[i] = a.s * (a.R[3 * i] * b.t[0] + a.R[3 * i + 1] * b.t[1] + a.R[3 * i + 2] * b.t[2]) + a.t[i];
  return r;
}

__host__ __device__ inline DSim3 sim3_inv(const DSim3& a) {  // lie.cpp:121-129
  DSim3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.R[3 * i + j] = a.R[3 * j + i];
  r.s = 1.0 / a.s;
  for (int i = 0; i < 3; ++i)
    r.t[i] = -r.s * (r.R[3 * i] * a.t[0] + r.R[3 * i + 1] * a.t[1] + r.R[3 * i + 2] * a.t[2]);
  return r;
}

// Sim(3) exponential, lie.cpp:23-32, 51-90, 99-108 (tangent order rho, omega, sigma).
__host__ __device__ inline DSim3 sim3_exp(const double* tau) {
  const double rho[3] = {tau[0], tau[1], tau[2]};
  const double w[3] = {tau[3], tau[4], tau[5]};
  const double sigma = tau[6];
  const double theta = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double O[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double O2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) O2[3 * i + j] = O[3 * i] * O[j] + O[3 * i + 1] * O[3 + j] + O[3 * i + 2] * O[6 + j];
  const double kSmall = 1e-8;
  DSim3 r;
  double a1, a2;
  if (theta < kSmall) {
    a1 = 1.0;
    a2 = 0.5;
  } else {
    a1 = sin(theta) / theta;
    a2 = (1.0 - cos(theta)) / (theta * theta);
  }
  for (int i = 0; i < 9; ++i) r.R[i] = ((i % 4 == 0) ? 1.0 : 0.0) + a1 * O[i] + a2 * O2[i];
  const double scale = exp(sigma);
  r.s = scale;
  double A, B, Cc;
  if (fabs(sigma) < kSmall) {
    Cc = 1.0 + 0.5 * sigma + sigma * sigma / 6.0;
    if (theta < kSmall) {
      A = 0.5 + sigma / 3.0;
      B = 1.0 / 6.0 + sigma / 8.0;
    } else {
      const double th2 = theta * theta, den = sigma * sigma + th2;
      A = (scale * (sigma * sin(theta) - theta * cos(theta)) + theta) / (theta * den);
      B = (Cc - (scale * (sigma * cos(theta) + theta * sin(theta)) - sigma) / den) / th2;
    }
  } else {
    Cc = (scale - 1.0) / sigma;
    if (theta < kSmall) {
      const double s2 = sigma * sigma;
      A = (scale * (sigma - 1.0) + 1.0) / s2;
      B = (scale * (s2 - 2.0 * sigma + 2.0) - 2.0) / (2.0 * s2 * sigma);
    } else {
      const double th2 = theta * theta, den = sigma * sigma + th2;
      A = (scale * (sigma * sin(theta) - theta * cos(theta)) + theta) / (theta * den);
      B = (Cc - (scale * (sigma * cos(theta) + theta * sin(theta)) - sigma) / den) / th2;
    }
  }
  double Wm[9];
  for (int i = 0; i < 9; ++i) Wm[i] = ((i % 4 == 0) ? Cc : 0.0) + A * O[i] + B * O2[i];
  for (int i = 0; i < 3; ++i) r.t[i] = Wm[3 * i] * rho[0] + Wm[3 * i + 1] * rho[1] + Wm[3 * i + 2] * rho[2];
  return r;
}

// 7x7 adjoint, lie.cpp:155-163 (row-major)
__host__ __device__ inline void sim3_adjoint(const DSim3& T, double* ad) {
  for (int i = 0; i < 49; ++i) ad[i] = 0.0;
  const double* R = T.R;
  const double* t = T.t;
  const double S[9] = {0, -t[2], t[1], t[2], 0, -t[0], -t[1], t[0], 0};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      ad[r * 7 + c] = T.s * R[3 * r + c];
      ad[r * 7 + 3 + c] = S[3 * r] * R[c] + S[3 * r + 1] * R[3 + c] + S[3 * r + 2] * R[6 + c];
      ad[(3 + r) * 7 + 3 + c] = R[3 * r + c];
    }
  for (int r = 0; r < 3; ++r) ad[r * 7 + 6] = -t[r];
  ad[48] = 1.0;
}

__host__ __device__ inline pmx_sim3 to_pmx(const DSim3& d) {
  pmx_sim3 T;
  for (int i = 0; i < 9; ++i) T.R[i] = d.R[i];
  for (int i = 0; i < 3; ++i) T.t[i] = d.t[i];
  T.s = d.s;
  return T;
}

// Eigen-style pivoted LDL^T solve (LDLT.h restated; see oracle.cpp) for n<=7,
// used for the tracking 7x7 step (tracking.cpp:203) on host and device.
__host__ __device__ inline void ldlt_pivoted_solve(int n, const double* A_in, const double* b, double* x) {
  double M[49];
  for (int i = 0; i < n * n; ++i) M[i] = A_in[i];
  int tr[7];
  double temp[7];
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bigv = fabs(M[k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(M[i * n + i]) > bigv) {
        bigv = fabs(M[i * n + i]);
        big = i;
      }
    tr[k] = big;
    if (k != big) {
      for (int c = 0; c < k; ++c) {
        double t = M[k * n + c];
        M[k * n + c] = M[big * n + c];
        M[big * n + c] = t;
      }
      for (int r = big + 1; r < n; ++r) {
        double t = M[r * n + k];
        M[r * n + k] = M[r * n + big];
        M[r * n + big] = t;
      }
      double t = M[k * n + k];
      M[k * n + k] = M[big * n + big];
      M[big * n + big] = t;
      for (int i = k + 1; i < big; ++i) {
        double tmp = M[i * n + k];
        M[i * n + k] = M[big * n + i];
        M[big * n + i] = tmp;
      }
    }
    if (k > 0) {
      for (int c = 0; c < k; ++c) temp[c] = M[c * n + c] * M[k * n + c];
      double acc = 0.0;
      for (int c = 0; c < k; ++c) acc += M[k * n + c] * temp[c];
      M[k * n + k] -= acc;
      for (int r = k + 1; r < n; ++r) {
        double a = 0.0;
        for (int c = 0; c < k; ++c) a += M[r * n + c] * temp[c];
        M[r * n + k] -= a;
      }
    }
    const double akk = M[k * n + k];
    const bool ok = fabs(akk) > 0.0;
    if (k == 0 && !ok) {
      for (int i = 0; i < n; ++i) x[i] = 0.0;
      return;
    }
    if (ok)
      for (int r = k + 1; r < n; ++r) M[r * n + k] /= akk;
  }
  double d[7];
  for (int i = 0; i < n; ++i) d[i] = b[i];
  for (int k = 0; k < n; ++k) {
    double t = d[k];
    d[k] = d[tr[k]];
    d[tr[k]] = t;
  }
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < i; ++c) d[i] -= M[i * n + c] * d[c];
  for (int i = 0; i < n; ++i) {
    if (fabs(M[i * n + i]) > 2.2250738585072014e-308)
      d[i] /= M[i * n + i];
    else
      d[i] = 0.0;
  }
  for (int i = n - 1; i >= 0; --i)
    for (int r = i + 1; r < n; ++r) d[i] -= M[r * n + i] * d[r];
  for (int k = n - 1; k >= 0; --k) {
    double t = d[k];
    d[k] = d[tr[k]];
    d[tr[k]] = t;
  }
  for (int i = 0; i < n; ++i) x[i] = d[i];
}

// Shared-memory histogram increment aggregated over the warp's lanes that hit
// the same bin (keys of one image cluster in a few bins: plain atomics would
// serialise on them).  Call from every lane of the converged warp; `take` =
// this lane has a key.
// Checked builds (-DPMX_CHECKED, tools/gpu_checked.sh): every gather index
// of the hot kernels is range-checked on the device; a violation is counted
// (per translation unit, read by pmx_checked_violations) and the access is
// redirected to element 0, so a bad index shows up as a non-zero count
// instead of a fault.  Substitutes for compute-sanitizer, which this pool
// does not offer.  Release builds compile the checks away.
#ifdef PMX_CHECKED
static __device__ unsigned long long g_pmx_violations;
#define PMX_CHECK_INDEX(i, n)                                                        \
  do {                                                                              \
    if ((unsigned long long)(long long)(i) >= (unsigned long long)(long long)(n)) { \
      atomicAdd(&g_pmx_violations, 1ull);                                           \
      (i) = 0;                                                                      \
    }                                                                               \
  } while (0)
#define PMX_DEFINE_VIOLATION_READER(fn)                                                 \
  extern "C" unsigned long long fn() {                                                  \
    unsigned long long v = 0;                                                           \
    cudaMemcpyFromSymbol(&v, g_pmx_violations, sizeof(v));                              \
    return v;                                                                           \
  }
#else
#define PMX_CHECK_INDEX(i, n) \
  do {                        \
  } while (0)
#define PMX_DEFINE_VIOLATION_READER(fn) \
  extern "C" unsigned long long fn() { return 0; }
#endif

// FP64 reciprocal from the MUFU seed + two Newton steps (within 1 ulp of the
// correctly rounded 1/d; zero, non-finite and extreme inputs take the IEEE
// division).
__device__ __forceinline__ double rcp64(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  e = fma(e, e, e);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  const double ad = fabs(d);
  if (!(ad > 1e-300 && ad < 1e300)) r = 1.0 / d;
  return r;
}

__device__ __forceinline__ void hist_add(uint32_t* sh, uint32_t bin, bool take) {
  const unsigned active = __activemask();
  const unsigned with = __ballot_sync(active, take);
  if (!take) return;
  const unsigned peers = __match_any_sync(with, bin);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh[bin], (uint32_t)__popc(peers));
}

// --------------------------------------------------------- reductions
__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace pmx
