// Frontend tracking (BASELINE path 2): IRLS/Huber Gauss-Newton over one
// Sim(3) on ray + distance residuals, and confidence-weighted fusion.
//
// Reference: /root/reference/proj/src/tracking.cpp:149-247 (solve_pose,
// fuse_canonical), :249-257 (keyframe_decision); camera.cpp:10-28
// (valid_count, unique_pixel_fraction).
//
//   K5 k_track_gn   one cooperative persistent kernel runs the whole LM-damped
//                   GN loop of tracking.cpp:184-224 on the device: one fused
//                   residual + H/g + cost pass per iteration at the trial pose
//                   (its H/g are reused when the step is accepted, exactly as
//                   the reference reuses blocks_new), a deterministic FP64
//                   block/grid reduction, and the 7x7 pivoted LDL^T solve +
//                   retract + accept test replicated in every block (one grid
//                   barrier per iteration).  Nothing per-match is written to
//                   HBM.
//   K6 k_fuse       one thread per pixel, in place.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <unordered_set>
#include <vector>

#include "residual.cuh"
#include "select.cuh"

namespace cg = cooperative_groups;

namespace pmx {

// Fused residual pass over all matches at pose T -> per-block partials.
// Td (the GN loop): the cost slot (35) takes the FP64 block_cost of the
// FP64-evaluated residuals instead of the fp32 sum, so the accept / stop
// decisions (tracking.cpp:210-223) are taken on the reference's arithmetic
// (as ray mode's ray_cost64 does).
__device__ void eval_pass(const PoseR<float>& T, const MatchesDev& M, const CloudDev& Xref, const CloudDev& Xsrc,
                          int mode, const WeightsDev& wp, const IntrDev& K, double* __restrict__ partials,
                          const PoseR<double>* Td = nullptr) {
  float acc[kAcc];
#pragma unroll
  for (int i = 0; i < kAcc; ++i) acc[i] = 0.0f;
  double cost64 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M.count; k += stride) {
    if (Td) {  // residuals in FP64 (they cancel in point / pixel mode), products accumulated in fp32
      MatchEval<double> md;
      eval_match<double>(*Td, M, Xref, Xsrc, mode, wp, K, k, md);
      accumulate<double>(md, mode, wp, acc);
      if (md.used) cost64 += block_cost_one<double>(md, mode, wp);
    } else {
      MatchEval<float> m;
      eval_match<float>(T, M, Xref, Xsrc, mode, wp, K, k, m);
      accumulate<float>(m, mode, wp, acc);
    }
  }
  block_reduce_to(acc, partials + (size_t)blockIdx.x * kAcc);
  if (Td) {  // deterministic: warp sums in lane order, warps in order
    __shared__ double wc[32];
    cost64 = warp_sum(cost64);
    if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = cost64;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wc[w];
      partials[(size_t)blockIdx.x * kAcc + 35] = t;
    }
    __syncthreads();
  }
}

// Ray mode (the tracking configuration): closed-form sums with the cancelling
// parts of the residual in FP64 (residual.cuh ray_accumulate) -> kRayAcc
// partials per block (stride kAcc).  Same skips as eval_match.
// with_count: the pass also counts the valid flags of all matches (the lost
// test's valid_count, camera.cpp:10-14) into slot kAcc - 1 of the partials.
__device__ void eval_pass_ray(const PoseR<double>& T, const MatchesDev& M, const CloudDev& Xref,
                              const CloudDev& Xsrc, const WeightsDev& wp, double* __restrict__ partials,
                              bool with_count = false) {
  float acc[kRayAcc];
#pragma unroll
  for (int i = 0; i < kRayAcc; ++i) acc[i] = 0.0f;
  const RayW c{(float)wp.huber_delta, (float)(wp.huber_delta * wp.huber_delta), (float)wp.distance_weight};
  double cost64 = 0.0;
  int nvalid = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M.count; k += stride) {
    const int pa = M.pa ? __ldg(M.pa + k) : (int)k;
    const int pb = M.pb ? __ldg(M.pb + k) : (int)k;
    const bool mv = M.valid ? __ldg(M.valid + k) != 0 : true;
    nvalid += mv ? 1 : 0;
    if (!mv || pa < 0 || pb < 0 || pb >= Xref.H * Xref.W || pa >= Xsrc.H * Xsrc.W) continue;
    float rf[3], sf[3];
    if (!load_point(Xref, pb, rf) || !load_point(Xsrc, pa, sf)) continue;
    const double q = (double)__ldg(M.q + k);
    if (!(q > wp.q_min)) continue;  // robust_weight: infinite denom -> excluded
    const float info = (float)(1.0 / (wp.sigma2 / q));
    const double rd[3] = {rf[0], rf[1], rf[2]}, sd[3] = {sf[0], sf[1], sf[2]};
    const float rrf = fmaf(rf[0], rf[0], fmaf(rf[1], rf[1], rf[2] * rf[2]));
    if (!(rrf >= 1e-24f)) continue;  // |ref| < 1e-12 (tracking.cpp:78)
    const float ir = rsqrt_nr(rrf);
    ray_accumulate(T, rd, rrf * ir, ir, rf, sd, info, c, acc);
    cost64 += ray_cost64(T, rd, sd, 1.0 / (wp.sigma2 / q), wp.distance_weight, wp.huber_delta);
  }
  block_reduce_n<kRayAcc>(acc, partials + (size_t)blockIdx.x * kAcc);
  // the cost slot takes the FP64 sum (deterministic: warp sums in lane order, warps in order)
  __shared__ double wc[32];
  __shared__ int wn[32];
  cost64 = warp_sum(cost64);
  for (int o = 16; o > 0; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
  if ((threadIdx.x & 31) == 0) {
    wc[threadIdx.x >> 5] = cost64;
    wn[threadIdx.x >> 5] = nvalid;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    int nv = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t += wc[w];
      nv += wn[w];
    }
    partials[(size_t)blockIdx.x * kAcc + kRayAcc - 1] = t;
    if (with_count) partials[(size_t)blockIdx.x * kAcc + kAcc - 1] = (double)nv;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_normal_eq(PoseR<float> T, MatchesDev M, CloudDev Xref, CloudDev Xsrc,
                                                   int mode, WeightsDev wp, const double* qmin_dev, IntrDev K,
                                                   double* partials) {
  if (qmin_dev) wp.q_min = *qmin_dev;
  eval_pass(T, M, Xref, Xsrc, mode, wp, K, partials);
}

__global__ void k_sum_partials(const double* __restrict__ partials, int nblocks, double* out) {
  for (int i = threadIdx.x; i < kAcc; i += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partials[(size_t)b * kAcc + i];
    out[i] = s;
  }
}

__global__ void __launch_bounds__(256) k_residual_blocks(PoseR<double> T, MatchesDev M, CloudDev Xref,
                                                         CloudDev Xsrc, int mode, WeightsDev wp, IntrDev K,
                                                         double* res, double* jac, double* wt, double* info,
                                                         uint8_t* used) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M.count) return;
  MatchEval<double> m;
  eval_match<double>(T, M, Xref, Xsrc, mode, wp, K, k, m);
  for (int r = 0; r < 4; ++r) {
    res[4 * k + r] = m.r[r];
    wt[4 * k + r] = m.w[r];
    for (int c = 0; c < 7; ++c) jac[28 * k + 7 * r + c] = m.J[r][c];
  }
  info[k] = m.info;
  used[k] = m.used ? 1 : 0;
}

// --------------------------------------------------------------- GN loop
struct GNState {
  DSim3 T;        // current estimate
  DSim3 Ttrial;   // candidate
  double H[49];   // normal equations at T
  double g[7];
  double tau[7];
  double cost;
  double lambda;
  double q_min;
  int64_t valid_count;
  int iterations;
  int stop;
  int trial_ok;
  int lost;
  int trace_len;
  double trace[PMX_MAX_TRACE];
};

struct TrackArgs {
  MatchesDev M;
  CloudDev Xref, Xsrc;
  int mode;
  WeightsDev wp;
  IntrDev K;
  int max_iterations;
  double update_tol;
  int min_valid;
  double q_min_fraction;
  const double* median_dev;  // median of valid q
  double* partials;
  GNState* st;
};

__device__ void load_sums(const double* __restrict__ partials, int nblocks, bool ray, double* H, double* g,
                          double* cost) {
  // one block, all threads: fixed-order sum (deterministic), columns x 8 row
  // groups in parallel, then the groups in order; results into shared
  __shared__ double s[kAcc];
  __shared__ double grp[8][kAcc];
  const int n = ray ? kRayAcc : kAcc;
  for (int t = threadIdx.x; t < 8 * n; t += blockDim.x) {
    const int i = t % n, q = t / n;
    const int b0 = (int)((int64_t)nblocks * q / 8), b1 = (int)((int64_t)nblocks * (q + 1) / 8);
    double a = 0.0;
#pragma unroll 4
    for (int b = b0; b < b1; ++b) a += partials[(size_t)b * kAcc + i];
    grp[q][i] = a;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double a = 0.0;
    for (int q = 0; q < 8; ++q) a += grp[q][i];
    s[i] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0 && ray) {
    ray_expand(s, H, g, cost);
  } else if (threadIdx.x == 0) {
    int idx = 0;
    for (int a = 0; a < 7; ++a)
      for (int b = a; b < 7; ++b) {
        H[a * 7 + b] = s[idx];
        H[b * 7 + a] = s[idx];
        ++idx;
      }
    for (int a = 0; a < 7; ++a) g[a] = s[28 + a];
    *cost = s[35];
  }
  __syncthreads();
}

// ldlt_pivoted_solve(7, ...) (pmx_common.cuh, Eigen's pivoted LDLT) on one
// warp with the matrix in shared memory: the same operations in the same
// order on every element (bit-identical), lanes over rows / columns where the
// reference's loops are independent.  H, g: this warp's inputs; tau out.
__device__ void ldlt7_solve_warp(const double* H, const double* mg, double* tau, double* M, double* tmp, int* tr) {
  constexpr int n = 7;
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < n * n; i += 32) M[i] = H[i];
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    int big = k;
    if (lane == 0) {  // first largest |diagonal| (strict '>', as the scan of the reference)
      double bigv = fabs(M[k * n + k]);
      for (int i = k + 1; i < n; ++i)
        if (fabs(M[i * n + i]) > bigv) {
          bigv = fabs(M[i * n + i]);
          big = i;
        }
      tr[k] = big;
    }
    big = __shfl_sync(0xffffffffu, big, 0);
    if (k != big) {
      if (lane < k) {
        const double t = M[k * n + lane];
        M[k * n + lane] = M[big * n + lane];
        M[big * n + lane] = t;
      }
      if (lane > big && lane < n) {
        const double t = M[lane * n + k];
        M[lane * n + k] = M[lane * n + big];
        M[lane * n + big] = t;
      }
      if (lane == 0) {
        const double t = M[k * n + k];
        M[k * n + k] = M[big * n + big];
        M[big * n + big] = t;
      }
      if (lane > k && lane < big) {
        const double t = M[lane * n + k];
        M[lane * n + k] = M[big * n + lane];
        M[big * n + lane] = t;
      }
    }
    __syncwarp();
    if (k > 0) {
      if (lane < k) tmp[lane] = M[lane * n + lane] * M[k * n + lane];
      __syncwarp();
      if (lane >= k && lane < n) {
        double a = 0.0;
        for (int c = 0; c < k; ++c) a += M[lane * n + c] * tmp[c];
        M[lane * n + k] -= a;  // lane k: the diagonal (acc of the reference)
      }
      __syncwarp();
    }
    const double akk = M[k * n + k];
    const bool ok = fabs(akk) > 0.0;
    if (k == 0 && !ok) {
      if (lane < n) tau[lane] = 0.0;
      __syncwarp();
      return;
    }
    if (ok && lane > k && lane < n) M[lane * n + k] /= akk;
    __syncwarp();
  }
  if (lane == 0) {  // substitutions: sequential, as the reference
    double d[n];
    for (int i = 0; i < n; ++i) d[i] = mg[i];
    for (int k = 0; k < n; ++k) {
      const double t = d[k];
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
      const double t = d[k];
      d[k] = d[tr[k]];
      d[tr[k]] = t;
    }
    for (int i = 0; i < n; ++i) tau[i] = d[i];
  }
  __syncwarp();
}

// The loop state is replicated in every block (shared memory): after the
// one grid barrier of an iteration every block sums the partials in the same
// fixed order, solves the same 7x7 system and takes the same accept
// decision, so the replicas stay bit-identical and the next residual pass
// starts without a second barrier.  The partials alternate between two
// buffers: a block can be at most one pass ahead of the slowest reader.
// Block 0 publishes the state (pose, iterations, cost trace) to A.st.
template <bool RAY>
__global__ void __launch_bounds__(256, 2) k_track_gn(TrackArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double s_Hd[49], s_mg[7], s_tau[7], s_M[49], s_tmp[7];  // the 7x7 solve (warp 0)
  __shared__ int s_tr[7];
  __shared__ GNState L;  // this block's replica of the loop state
  const int nb = gridDim.x;
  const size_t half = (size_t)nb * kAcc;
  const bool pub = blockIdx.x == 0 && threadIdx.x == 0;  // publishes to A.st
  if (threadIdx.x == 0) L = *A.st;  // initial pose (host-written)
  __syncthreads();
  constexpr bool ray = RAY;  // ray mode gets its own instance (register budget)
  WeightsDev wp = A.wp;
  wp.q_min = A.q_min_fraction * (*A.median_dev);  // tracking.cpp:170-171
  int buf = 1;
  double* part = A.partials + buf * half;
  if (ray) {
    // the first residual pass at the initial pose also counts the valid
    // matches; the lost test (tracking.cpp:165-168) then discards it if needed
    eval_pass_ray(make_pose<double>(L.T), A.M, A.Xref, A.Xsrc, wp, part, true);
  } else {
    // valid_count (camera.cpp:10-14) for the lost test (tracking.cpp:165-168)
    float acc[kAcc];
    for (int i = 0; i < kAcc; ++i) acc[i] = 0.0f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int cnt = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < A.M.count; k += stride)
      cnt += (A.M.valid ? A.M.valid[k] != 0 : 1);
    acc[kAcc - 1] = (float)cnt;
    block_reduce_to(acc, A.partials + (size_t)blockIdx.x * kAcc);  // buffer 0
  }
  grid.sync();
  if (threadIdx.x == 0) {
    const double* cp = ray ? part : A.partials;
    double c = 0.0;
    for (int b = 0; b < nb; ++b) c += cp[(size_t)b * kAcc + kAcc - 1];
    L.valid_count = (int64_t)c;
    L.lost = c < (double)A.min_valid ? 1 : 0;
    L.stop = L.lost;
    L.q_min = wp.q_min;
    L.lambda = 1e-8;
    L.iterations = 0;
    L.trace_len = 0;
  }
  __syncthreads();
  if (!L.stop) {
    if (!ray) {
      const PoseR<float> T = make_pose<float>(L.T);
      const PoseR<double> Td = make_pose<double>(L.T);
      eval_pass(T, A.M, A.Xref, A.Xsrc, A.mode, wp, A.K, part, &Td);
      grid.sync();
    }
    {
      double H[49], g[7], c;
      load_sums(part, nb, ray, H, g, &c);
      if (threadIdx.x == 0) {
        for (int i = 0; i < 49; ++i) L.H[i] = H[i];
        for (int i = 0; i < 7; ++i) L.g[i] = g[i];
        L.cost = c;
        L.trace[L.trace_len++] = c;
      }
      __syncthreads();
    }
    for (int it = 0; it < A.max_iterations; ++it) {
      if (threadIdx.x < 32) {
        // tracking.cpp:200-206 (the 7x7 pivoted LDLT on warp 0, bit-identical)
        for (int i = threadIdx.x; i < 49; i += 32) s_Hd[i] = L.H[i];
        __syncwarp();
        if (threadIdx.x < 7) {
          s_Hd[threadIdx.x * 8] += L.lambda * fmax(L.H[threadIdx.x * 8], 1e-12);
          s_mg[threadIdx.x] = -L.g[threadIdx.x];
        }
        __syncwarp();
        ldlt7_solve_warp(s_Hd, s_mg, s_tau, s_M, s_tmp, s_tr);
      }
      if (threadIdx.x == 0) {
        L.iterations++;
        double tau[7];
        for (int k = 0; k < 7; ++k) tau[k] = s_tau[k];
        bool fin = true;
        double inf = 0.0;
        for (int k = 0; k < 7; ++k) {
          fin = fin && isfinite(tau[k]);
          inf = fmax(inf, fabs(tau[k]));
          L.tau[k] = tau[k];
        }
        if (fin && inf < 1e3) {
          L.Ttrial = sim3_mul(sim3_exp(tau), L.T);  // left-plus retract, lie.hpp:54
          L.trial_ok = 1;
        } else {
          L.trial_ok = 0;
          L.lambda *= 10.0;
          if (L.lambda > 1e8) L.stop = 1;
        }
      }
      __syncthreads();
      if (L.stop) break;
      if (!L.trial_ok) continue;
      buf ^= 1;
      part = A.partials + buf * half;
      if (ray) {
        eval_pass_ray(make_pose<double>(L.Ttrial), A.M, A.Xref, A.Xsrc, wp, part);
      } else {
        const PoseR<float> T = make_pose<float>(L.Ttrial);
        const PoseR<double> Td = make_pose<double>(L.Ttrial);
        eval_pass(T, A.M, A.Xref, A.Xsrc, A.mode, wp, A.K, part, &Td);
      }
      grid.sync();
      double H[49], g[7], c;
      load_sums(part, nb, ray, H, g, &c);
      if (threadIdx.x == 0) {
        // tracking.cpp:210-223
        if (c <= L.cost * (1.0 + 1e-12) + 1e-300) {
          L.T = L.Ttrial;
          for (int i = 0; i < 49; ++i) L.H[i] = H[i];
          for (int i = 0; i < 7; ++i) L.g[i] = g[i];
          L.cost = c;
          if (L.trace_len < PMX_MAX_TRACE) L.trace[L.trace_len++] = c;
          L.lambda = fmax(L.lambda * 0.3, 1e-10);
          double n2 = 0.0;
          for (int k = 0; k < 7; ++k) n2 += L.tau[k] * L.tau[k];
          if (sqrt(n2) < A.update_tol) L.stop = 1;
        } else {
          L.lambda *= 10.0;
          if (L.lambda > 1e8) L.stop = 1;
        }
      }
      __syncthreads();
      if (L.stop) break;
    }
  }
  if (pub) *A.st = L;
}

// ----------------------------------------------------------------- fusion
__global__ void __launch_bounds__(256) k_fuse(int n, float* __restrict__ cxyz, uint8_t* __restrict__ cvalid,
                                              float* __restrict__ cconf, const float* __restrict__ xk,
                                              const uint8_t* __restrict__ vk, const float* __restrict__ conf,
                                              DSim3 T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (vk && !vk[i]) return;  // tracking.cpp:233
  const double c = conf[i];
  const double cp = cconf[i];
  if (cp + c <= 0.0) return;
  const double p0 = xk[3 * i], p1 = xk[3 * i + 1], p2 = xk[3 * i + 2];
  double o[3];
  for (int r = 0; r < 3; ++r)
    o[r] = T.s * (T.R[3 * r] * p0 + T.R[3 * r + 1] * p1 + T.R[3 * r + 2] * p2) + T.t[r];
  if (cp <= 0.0 || !cvalid[i]) {
    for (int r = 0; r < 3; ++r) cxyz[3 * i + r] = (float)o[r];
  } else {
    const double inv = 1.0 / (cp + c);
    for (int r = 0; r < 3; ++r) cxyz[3 * i + r] = (float)((cp * (double)cxyz[3 * i + r] + c * o[r]) * inv);
  }
  cvalid[i] = 1;
  cconf[i] = (float)(cp + c);
}

// ------------------------------------------------------------ match stats
__global__ void k_match_stats(MatchesDev M, int num_pixels_a, uint32_t* bitmap, unsigned long long* count,
                              int* oob, int* oob_n, int oob_cap) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool v = false;
  if (k < M.count) v = M.valid ? M.valid[k] != 0 : true;
  const unsigned ballot = __ballot_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(count, (unsigned long long)__popc(ballot));
  if (!v) return;
  const int pa = M.pa[k];
  if (pa >= 0 && pa < num_pixels_a) {
    atomicOr(&bitmap[pa >> 5], 1u << (pa & 31));
  } else {
    const int slot = atomicAdd(oob_n, 1);
    if (slot < oob_cap) oob[slot] = pa;
  }
}

__global__ void k_popcount(const uint32_t* bitmap, int words, unsigned long long* out) {
  unsigned long long s = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x)
    s += __popc(bitmap[i]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// ------------------------------------------------------------------ host
static WeightsDev make_weights(const pmx_robust_weight_params& p, int mode) {
  WeightsDev w;
  w.sigma2 = mode == PMX_TRACK_RAY ? p.sigma2_ray : mode == PMX_TRACK_POINT ? p.sigma2_point : p.sigma2_pixel;
  w.q_min = p.q_min;
  w.huber_delta = p.huber_delta;
  w.distance_weight = p.distance_weight;
  return w;
}

static IntrDev make_intr(const pmx_intrinsics* K) {
  IntrDev k{0, 0, 0, 0, 0};
  if (K) k = IntrDev{K->fx, K->fy, K->cx, K->cy, 1};
  return k;
}

static DSim3 checked_pose(const pmx_sim3* T) {
  require(T != nullptr, "null pose");
  require(T->s > 0.0, "Sim3Pose: scale must be positive");  // lie.cpp:94-96
  return to_dsim3(*T);
}

static MatchesDev stage_matches(Stager& st, const pmx_matchset* m) {
  require(m && m->count >= 0 && (m->count == 0 || (m->pixel_a && m->confidence)), "matchset: null arrays");
  MatchesDev d;
  d.count = m->count;
  d.pa = st.in(m->pixel_a, (size_t)m->count);
  d.pb = st.in(m->pixel_b, (size_t)m->count);
  d.q = st.in(m->confidence, (size_t)m->count);
  d.valid = st.in(m->valid, (size_t)m->count);
  return d;
}

static CloudDev stage_cloud(Stager& st, const pmx_pointmap* p) {
  require(p && p->xyz && p->height > 0 && p->width > 0, "pointmap: empty or null");
  const size_t hw = (size_t)p->height * p->width;
  return CloudDev{st.in(p->xyz, 3 * hw), st.in(p->valid, hw), p->height, p->width};
}

static int grid_for(Context& ctx, const void* kernel, int threads) {
  int per_sm = 0;
  PMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0));
  return std::max(1, per_sm) * ctx.num_sms;
}

}  // namespace pmx

using namespace pmx;

int pmx_impl_match_stats_dev(Context& ctx, const MatchesDev& M, int num_pixels_a, int64_t* valid_count,
                             double* unique_fraction);

extern "C" int pmx_impl_residual_blocks(pmx_context* c, pmx_memory mem, const pmx_sim3* Tp, const pmx_matchset* m,
                                        const pmx_pointmap* X_ref, const pmx_pointmap* X_src, pmx_track_mode mode,
                                        const pmx_robust_weight_params* params, const pmx_intrinsics* K,
                                        double* residual, double* jacobian, double* weight, double* info,
                                        uint8_t* used) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  if (mode == PMX_TRACK_PIXEL && K == nullptr)
    throw Error(PMX_ERR_INVALID_ARGUMENT, "residual_blocks: pixel mode requires intrinsics");  // tracking.cpp:50-52
  pmx_robust_weight_params p;
  pmx_default_robust_weight_params(&p);
  if (params) p = *params;
  const DSim3 T = checked_pose(Tp);
  Stager st(ctx, mem);
  const MatchesDev M = stage_matches(st, m);
  const CloudDev R = stage_cloud(st, X_ref), S = stage_cloud(st, X_src);
  const size_t n = (size_t)M.count;
  double* dr = st.out(residual, 4 * n);
  double* dj = st.out(jacobian, 28 * n);
  double* dw = st.out(weight, 4 * n);
  double* di = st.out(info, n);
  uint8_t* du = st.out(used, n);
  if (n) {
    k_residual_blocks<<<(unsigned)((n + 255) / 256), 256, 0, ctx.stream>>>(
        make_pose<double>(T), M, R, S, mode, make_weights(p, mode), make_intr(K), dr, dj, dw, di, du);
    launch_check(ctx, "k_residual_blocks");
  }
  st.back(residual, dr, 4 * n);
  st.back(jacobian, dj, 28 * n);
  st.back(weight, dw, 4 * n);
  st.back(info, di, n);
  st.back(used, du, n);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

extern "C" int pmx_impl_normal_equations(pmx_context* c, pmx_memory mem, const pmx_sim3* Tp, const pmx_matchset* m,
                                         const pmx_pointmap* X_ref, const pmx_pointmap* X_src, pmx_track_mode mode,
                                         const pmx_robust_weight_params* params, const pmx_intrinsics* K, double* H,
                                         double* g, double* cost, int64_t* used) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  if (mode == PMX_TRACK_PIXEL && K == nullptr)
    throw Error(PMX_ERR_INVALID_ARGUMENT, "residual_blocks: pixel mode requires intrinsics");
  require(H && g && cost, "normal_equations: null outputs");
  pmx_robust_weight_params p;
  pmx_default_robust_weight_params(&p);
  if (params) p = *params;
  const DSim3 T = checked_pose(Tp);
  Stager st(ctx, mem);
  const MatchesDev M = stage_matches(st, m);
  const CloudDev R = stage_cloud(st, X_ref), S = stage_cloud(st, X_src);
  const int nb = grid_for(ctx, (const void*)k_normal_eq, 256);
  DevBuf partials(sizeof(double) * kAcc * nb, ctx.stream), sums(sizeof(double) * kAcc, ctx.stream);
  k_normal_eq<<<nb, 256, 0, ctx.stream>>>(make_pose<float>(T), M, R, S, mode, make_weights(p, mode), nullptr,
                                          make_intr(K), partials.as<double>());
  launch_check(ctx, "k_normal_eq");
  k_sum_partials<<<1, 64, 0, ctx.stream>>>(partials.as<double>(), nb, sums.as<double>());
  launch_check(ctx, "k_sum_partials");
  double s[kAcc];
  PMX_CUDA(cudaMemcpyAsync(s, sums.p, sizeof(s), cudaMemcpyDeviceToHost, ctx.stream));
  PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  int idx = 0;
  for (int a = 0; a < 7; ++a)
    for (int b = a; b < 7; ++b) {
      H[a * 7 + b] = s[idx];
      H[b * 7 + a] = s[idx];
      ++idx;
    }
  for (int a = 0; a < 7; ++a) g[a] = s[28 + a];
  *cost = s[35];
  if (used) *used = (int64_t)s[36];
  return PMX_OK;
}

extern "C" int pmx_impl_track_given_matches(pmx_context* c, pmx_memory mem, const pmx_pointmap* canonical,
                                            const pmx_pointmap* X_f_f, const pmx_matchset* matches,
                                            const pmx_sim3* init, pmx_track_mode mode,
                                            const pmx_solve_pose_params* params, pmx_track_result* result) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(result, "track: null result");
  pmx_solve_pose_params sp;
  pmx_default_solve_pose_params(&sp);
  if (params) sp = *params;
  const DSim3 T0 = checked_pose(init);
  Stager st(ctx, mem);
  TrackArgs A;
  std::memset(&A, 0, sizeof(A));
  A.M = stage_matches(st, matches);
  A.Xref = stage_cloud(st, canonical);
  A.Xsrc = stage_cloud(st, X_f_f);
  A.mode = mode;
  A.wp = make_weights(sp.weights, mode);
  A.K = make_intr(sp.has_intrinsics ? &sp.intrinsics : nullptr);
  A.max_iterations = sp.max_iterations;
  A.update_tol = sp.update_tol;
  A.min_valid = sp.min_valid_matches;
  A.q_min_fraction = sp.weights.q_min_fraction;
  // median of valid match confidences (tracking.cpp:170-171)
  DevBuf median(sizeof(double), ctx.stream), segbuf(sizeof(SelSeg), ctx.stream), selscratch;
  SelSeg seg{A.M.q, A.M.valid, A.M.count, median.as<double>(), 1.0};
  PMX_CUDA(cudaMemcpyAsync(segbuf.p, &seg, sizeof(seg), cudaMemcpyHostToDevice, ctx.stream));
  segmented_median(ctx, segbuf.as<SelSeg>(), 1, A.M.count, selscratch);
  A.median_dev = median.as<double>();
  const void* kern = mode == PMX_TRACK_RAY ? (const void*)k_track_gn<true> : (const void*)k_track_gn<false>;
  const int nb = grid_for(ctx, kern, 256);
  DevBuf partials(2 * sizeof(double) * kAcc * nb, ctx.stream), state(sizeof(GNState), ctx.stream);  // two buffers
  GNState init_state;
  std::memset(&init_state, 0, sizeof(init_state));
  init_state.T = T0;
  PMX_CUDA(cudaMemcpyAsync(state.p, &init_state, sizeof(init_state), cudaMemcpyHostToDevice, ctx.stream));
  A.partials = partials.as<double>();
  A.st = state.as<GNState>();
  // solve_pose's lost test precedes everything (tracking.cpp:165-168); pixel
  // mode without intrinsics throws on the first residual evaluation.
  void* args[] = {&A};
  if (mode == PMX_TRACK_PIXEL && !sp.has_intrinsics) {
    // evaluate the lost test first: the reference only throws if it gets to residual_blocks
    int64_t vc = 0;
    double uf = 0;
    pmx_impl_match_stats_dev(ctx, A.M, 1, &vc, &uf);
    if (vc >= sp.min_valid_matches)
      throw Error(PMX_ERR_INVALID_ARGUMENT, "residual_blocks: pixel mode requires intrinsics");
  }
  {
    ProfScope ps(ctx, "k_track_gn");
    PMX_CUDA(cudaLaunchCooperativeKernel(kern, dim3(nb), dim3(256), args, 0, ctx.stream));
  }
  launch_check(ctx, "k_track_gn");
  GNState out;
  PMX_CUDA(cudaMemcpyAsync(&out, state.p, sizeof(out), cudaMemcpyDeviceToHost, ctx.stream));
  PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  result->T_kf = to_pmx(out.lost ? T0 : out.T);
  result->iterations = out.iterations;
  result->lost = out.lost;
  result->cost_trace_len = out.trace_len;
  for (int i = 0; i < out.trace_len && i < PMX_MAX_TRACE; ++i) result->cost_trace[i] = out.trace[i];
  return PMX_OK;
}

extern "C" int pmx_impl_fuse_canonical(pmx_context* c, pmx_memory mem, int32_t height, int32_t width,
                                       float* cxyz, uint8_t* cvalid, float* cconf, const pmx_pointmap* X_k_f,
                                       const float* confidence, const pmx_sim3* Tp) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(cxyz && cvalid && cconf && X_k_f && confidence, "fuse_canonical: null arguments");
  require(X_k_f->height == height && X_k_f->width == width, "fuse_canonical: size mismatch");
  const DSim3 T = checked_pose(Tp);
  const size_t n = (size_t)height * width;
  Stager st(ctx, mem);
  float* dx = st.inout(cxyz, 3 * n);
  uint8_t* dv = st.inout(cvalid, n);
  float* dc = st.inout(cconf, n);
  const float* xk = st.in(X_k_f->xyz, 3 * n);
  const uint8_t* vk = st.in(X_k_f->valid, n);
  const float* cf = st.in(confidence, n);
  if (n) {
    k_fuse<<<(unsigned)((n + 255) / 256), 256, 0, ctx.stream>>>((int)n, dx, dv, dc, xk, vk, cf, T);
    launch_check(ctx, "k_fuse");
  }
  st.back(cxyz, dx, 3 * n);
  st.back(cvalid, dv, n);
  st.back(cconf, dc, n);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

int pmx_impl_match_stats_dev(Context& ctx, const MatchesDev& M, int num_pixels_a, int64_t* valid_count,
                             double* unique_fraction) {
  const int words = (std::max(num_pixels_a, 0) + 31) / 32;
  const int cap = 4096;
  DevBuf bm(sizeof(uint32_t) * std::max(words, 1), ctx.stream), cnt(sizeof(unsigned long long) * 2, ctx.stream),
      oob(sizeof(int) * cap, ctx.stream), oobn(sizeof(int), ctx.stream);
  PMX_CUDA(cudaMemsetAsync(bm.p, 0, bm.bytes, ctx.stream));
  PMX_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, ctx.stream));
  PMX_CUDA(cudaMemsetAsync(oobn.p, 0, oobn.bytes, ctx.stream));
  if (M.count > 0) {
    k_match_stats<<<(unsigned)((M.count + 255) / 256), 256, 0, ctx.stream>>>(
        M, num_pixels_a, bm.as<uint32_t>(), cnt.as<unsigned long long>(), oob.as<int>(), oobn.as<int>(), cap);
    launch_check(ctx, "k_match_stats");
  }
  if (words > 0) {
    k_popcount<<<std::min(1024, (words + 255) / 256), 256, 0, ctx.stream>>>(bm.as<uint32_t>(), words,
                                                                           cnt.as<unsigned long long>() + 1);
    launch_check(ctx, "k_popcount");
  }
  unsigned long long h[2];
  int on = 0;
  PMX_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  PMX_CUDA(cudaMemcpyAsync(&on, oobn.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  uint64_t distinct = h[1];
  if (on > 0) {
    require(on <= cap, "match_stats: too many out-of-range pixel_a values");
    std::vector<int> v(on);
    PMX_CUDA(cudaMemcpy(v.data(), oob.p, sizeof(int) * on, cudaMemcpyDeviceToHost));
    distinct += std::unordered_set<int>(v.begin(), v.end()).size();
  }
  *valid_count = (int64_t)h[0];
  *unique_fraction = num_pixels_a > 0 ? (double)distinct / (double)num_pixels_a : 0.0;
  return PMX_OK;
}

extern "C" int pmx_impl_match_stats(pmx_context* c, pmx_memory mem, const pmx_matchset* m, int32_t num_pixels_a,
                                    int64_t* valid_count, double* unique_fraction) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(m && valid_count && unique_fraction, "match_stats: null arguments");
  Stager st(ctx, mem);
  MatchesDev M;
  M.count = m->count;
  M.pa = st.in(m->pixel_a, (size_t)m->count);
  M.pb = nullptr;
  M.q = nullptr;
  M.valid = st.in(m->valid, (size_t)m->count);
  if (num_pixels_a <= 0) {  // camera.cpp:22
    *unique_fraction = 0.0;
    int64_t vc = 0;
    double uf;
    pmx_impl_match_stats_dev(ctx, M, 0, &vc, &uf);
    *valid_count = vc;
    return PMX_OK;
  }
  return pmx_impl_match_stats_dev(ctx, M, num_pixels_a, valid_count, unique_fraction);
}
