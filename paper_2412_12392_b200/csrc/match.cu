// Iterative projective matching + descriptor refinement (BASELINE path 1).
//
// Reference: /root/reference/proj/src/camera.cpp:39-271
//   normalize_rays (39-56), interpolate_ray (58-100), iterative_project
//   (115-174), median_scene_distance (178-191), match_pointmaps (195-237),
//   feature_refine (239-271).
//
// Kernels (one CUDA grid dimension per pair):
//   K2 k_keys / k_sel_scan / k_sel_hist   (all pairs of a batch at once)
//                    fp32 keys of the FP64 point norms, then an exact
//                    rank-floor(n/2) radix select (12+12+8 bits): the upper
//                    median of median_scene_distance's nth_element.
//   then per chunk of pairs (all pairs of a device-memory batch at once):
//   K1 k_prep        one thread per a-pixel: FP64 unit ray + validity into a
//                    32-byte ray map, and the int8 image of the descriptor
//                    (24 B) for the refinement.
//   K3+K4 k_match_refine  one thread per b-pixel: FP64 Levenberg-Marquardt on
//                    the ray-angle error, lround + clamp, q = sqrt(Q_a Q_b),
//                    the 3D invalidation test (K3; k_match alone when no
//                    refinement is asked), then the coarse-to-fine descriptor
//                    refinement of the valid matches on exact int8 scores with
//                    a rigorous uniqueness gap (K4); undecided pixels (near
//                    ties) take the exact path, so the argmax equals the
//                    reference's exact-arithmetic argmax (strict '>' scan,
//                    ties keep the centre / first raster).
#include <math_constants.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <type_traits>
#include <vector>

#include "pmx_common.cuh"

// Build-time variants (dev ablations; defaults are the product).
#ifndef PMX_PRUNE
#define PMX_PRUNE 0  // head-bound pruning of level-1 refinement candidates
#endif
#ifndef PMX_LD256
#define PMX_LD256 1  // one 256-bit load per ray-map support
#endif
#ifndef PMX_RCP
#define PMX_RCP 1  // LM quotients as products with reciprocals
#endif
#ifndef PMX_LM_F32
#define PMX_LM_F32 1  // LM step direction (Jacobian, normal equations, 2x2 solve) in fp32
#endif
#ifndef PMX_PAIRLD
#define PMX_PAIRLD 0  // level-1 window rows as aligned pixel pairs (16-B heads, 32-B tails): identical outputs, 1.50 -> 1.61 ms
#endif
#ifndef PMX_SEL_DIRECT_ATOMICS
#define PMX_SEL_DIRECT_ATOMICS 1  // median select passes 2-3: plain shared atomics instead of warp-aggregated ones
#endif
#ifndef PMX_ROW_WITH_GATHERS
#define PMX_ROW_WITH_GATHERS 1  // the refinement's target row loaded with the LM result's gathers
#endif
#ifndef PMX_PRELOAD_SEED
#define PMX_PRELOAD_SEED 0  // the identity seed's supports loaded together with X_b (spills 112 -> 128 B: 1.297 -> 1.377 ms)
#endif
#ifndef PMX_VALID_BITS
#define PMX_VALID_BITS 1  // support validity from the high words of the ray map's w (1.0 / 0.0)
#endif
#ifndef PMX_JDIFF_F32
#define PMX_JDIFF_F32 0  // Jacobian support differences from fp32-rounded supports (1.252 -> 1.245 ms; valid matches identical, a few invalid pixels' pixel_a differ)
#endif
#ifndef PMX_SPLIT
#define PMX_SPLIT 0  // LM (k_match) and refinement (k_refine_tiles) as two kernels (1.250 -> 1.434 ms at the best occupancy: the fused kernel overlaps the phases)
#endif
#ifndef PMX_PREFETCH
#define PMX_PREFETCH 0  // L2 prefetch of the target descriptor row before the LM (neutral at first; with the row loaded among the post-LM gathers, 1.296 -> 1.306 ms)
#endif
#ifndef PMX_EAGER_F32
#define PMX_EAGER_F32 1  // fp32 LM: Jacobian support differences formed in interp_eval, so the FP64 supports die there (with the normal-equation loop state: spills 156 -> 116 B, 1.425 -> 1.422 ms)
#endif
#ifndef PMX_RAY24
#define PMX_RAY24 0  // LM gathers 24 B (x, y, z: 16 + 8 B loads) per support, NaN-marked invalid rays: 1.500 -> 1.551 ms
#endif
#ifndef PMX_SM_COPY_MAX_KB
#define PMX_SM_COPY_MAX_KB 1024  // inputs below this size qualify for the SM copy
#endif
#ifndef PMX_SM_SMALL_COPIES
#define PMX_SM_SMALL_COPIES 1  // host path: small pinned inputs copied by one SM kernel instead of DMA
#endif
#ifndef PMX_HOST_CHUNK
#define PMX_HOST_CHUNK 4  // host path: pairs per full chunk (~95 MB of inputs: ~1.8 ms of H2D against ~0.2 ms of compute)
#endif
#ifndef PMX_J_SMEM
#define PMX_J_SMEM 0  // LM fp32 Jacobian in shared memory instead of registers (spills 180 -> 172 B; neutral: 1.502 vs 1.495 ms)
#endif
#ifndef PMX_LM_NE_STATE
#define PMX_LM_NE_STATE 1  // fp32 LM: carry J^T J, J^T r across iterations instead of J and the FP64 ray
#endif
#ifndef PMX_OVERLAP
#define PMX_OVERLAP 0  // pairs per chunk of the overlapped device path (0: one chunk; 8 / 16 / 32 measured 7-17% slower)
#endif

namespace pmx {

constexpr int kHist1 = 4096, kHist2 = 4096, kHist3 = 256;
constexpr int kHistTotal = kHist1 + kHist2 + kHist3;
constexpr uint32_t kNoKey = 0xffffffffu;

constexpr int kSelCap = 64;  // FP64 candidates kept per pair for the exact tie resolution

struct SelState {
  uint32_t n;       // number of keys
  uint32_t k;       // target rank (n / 2)
  uint32_t prefix;  // resolved high bits so far
  uint32_t krem;    // rank within the current bucket
  double threshold; // invalidation_median_fraction * median
  int a1max;        // max over a-pixels of sum |q8(D_a)| (int8 refinement error bound)
  int qbad;         // some |D_a component| * 127 >= 127.5: no int8 fast path for this pair
  // exact FP64 median: the fp32 key of the rank-k element, how many norms
  // share that key, and their FP64 values (the rank-krem one is the median)
  uint32_t key, ties, cnt, pad_;
  double median;
  double cand[kSelCap];
};

struct PairDev {
  int Ha, Wa, Hb, Wb, dim;
  const float* xa;
  const uint8_t* va;
  const float* xb;
  const uint8_t* vb;
  const __half* da;
  const float* qa;
  const __half* db;
  const float* qb;
  // optional seed (init MatchSet): last valid k per pixel_b, and the init pixel_a
  const int32_t* seed_last;
  const int32_t* init_pa;
  // outputs
  int32_t* out_pa;
  int32_t* out_pb;
  float* out_q;
  uint8_t* out_valid;
  // per-pair scratch
  double4* rays;
  uint32_t* keys;
  uint32_t* hist;
  SelState* sel;
  // descriptor pruning aux (dim == 24, 16-byte rows): planar 8-dim heads and
  // {||a||_2, ||a[8:24]||_2} upper bounds of every a-pixel (L2-resident)
  float4* dnorm;  // {||a||, ||a[16:24]||, ||a[8:24]||} upper bounds, .w = qa (standalone refine)
  // int8 descriptors of every a-pixel, round(127 x) (batched refine), planar
  // (a warp's 32 neighbouring candidates read contiguous bytes): q8h = dims
  // 0-7, q8n = nt = ceil(sqrt(sum of squares of dims 8-23)) (the
  // Cauchy-Schwarz bound of the tail), q8t = dims 8-23
  uint2* q8h;
  uint16_t* q8n;
  uint4* q8t;
};

struct LMParams {
  double lambda_init, lambda_up, lambda_down;
  double cos_tol;  // exact threshold: acos(clamp(d,-1,1)) < tol  <=>  d >= cos_tol
  int max_iterations;
  double median_fraction;
};

struct RefineLevels {
  int n;
  int stride[PMX_MAX_REFINE_LEVELS];
  int radius[PMX_MAX_REFINE_LEVELS];
};

// fp32 FMA with fp16 sources (SASS FHFMA, .H0/.H1 half selects): the fp16 x
// fp16 product is exact, one rounding per accumulation.
__device__ __forceinline__ float fh_lo(uint32_t a, uint32_t b, float c) {
  float r;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;"
      : "=f"(r)
      : "h"((unsigned short)(a & 0xffffu)), "h"((unsigned short)(b & 0xffffu)), "f"(c));
  return r;
}
__device__ __forceinline__ float fh_hi(uint32_t a, uint32_t b, float c) {
  float r;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(r) : "h"((unsigned short)(a >> 16)), "h"((unsigned short)(b >> 16)), "f"(c));
  return r;
}
// 8-term fp16 dot accumulated onto s in two independent FHFMA chains (half the
// dependency latency); at most 8 roundings, so the n*u error bounds used
// below stay valid for any chaining of these calls.
__device__ __forceinline__ float dot8(const uint4& a, const uint4& b, float s) {
  float t = fh_hi(a.x, b.x, 0.0f);
  s = fh_lo(a.x, b.x, s);
  t = fh_hi(a.y, b.y, t);
  s = fh_lo(a.y, b.y, s);
  t = fh_hi(a.z, b.z, t);
  s = fh_lo(a.z, b.z, s);
  t = fh_hi(a.w, b.w, t);
  s = fh_lo(a.w, b.w, s);
  return s + t;
}
// 16-term dot in four independent 4-deep chains (<= 6 roundings on any path,
// within the 16u bound).
__device__ __forceinline__ float dot16(const uint4& a0, const uint4& a1, const uint4& b0, const uint4& b1) {
  float p = fh_lo(a0.x, b0.x, 0.0f), q = fh_hi(a0.x, b0.x, 0.0f);
  float r = fh_lo(a1.x, b1.x, 0.0f), t = fh_hi(a1.x, b1.x, 0.0f);
  p = fh_lo(a0.y, b0.y, p);
  q = fh_hi(a0.y, b0.y, q);
  r = fh_lo(a1.y, b1.y, r);
  t = fh_hi(a1.y, b1.y, t);
  p = fh_lo(a0.z, b0.z, p);
  q = fh_hi(a0.z, b0.z, q);
  r = fh_lo(a1.z, b1.z, r);
  t = fh_hi(a1.z, b1.z, t);
  p = fh_lo(a0.w, b0.w, p);
  q = fh_hi(a0.w, b0.w, q);
  r = fh_lo(a1.w, b1.w, r);
  t = fh_hi(a1.w, b1.w, t);
  return (p + q) + (r + t);
}
constexpr float kU = 5.9604645e-08f;  // fp32 unit roundoff 2^-24

// Upper bound of sqrt(sum of squares) accumulated by an n-term FHFMA chain.
__device__ __forceinline__ float norm_ub(float ss, int n) {
  return sqrtf(ss * (1.0f + (n + 2) * kU)) * (1.0f + 2.0f * kU);
}

// Norm bounds of one 24-dim descriptor row (+ the pixel's match confidence).
__device__ __forceinline__ void desc_aux(const __half* row, float q, float4* nrm) {
  const uint4* p = reinterpret_cast<const uint4*>(row);
  const uint4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  const float s0 = dot8(a, a, 0.0f), s1 = dot8(b, b, 0.0f), s2 = dot8(c, c, 0.0f);
  *nrm = make_float4(norm_ub(s0 + s1 + s2, 24), norm_ub(s2, 8), norm_ub(s1 + s2, 16), q);
}

// int8 image of a 24-dim fp16 descriptor: q_k = rne(127 x_k), computed
// exactly in fp16 as the low byte of fma(x, 127, 1536) (the product is exact
// in the FMA, and 1536 + q is representable with ulp 1 for |q| <= 511).
// Valid (|127 x| <= 127.49, so q fits int8) iff max |x_k| <= 1 + 2^-8.
// l1 = sum |q_k| (exact: per-byte |q| summed by DP4A).
struct Q8 {
  uint4 a;  // dims 0-15
  uint2 b;  // dims 16-23
  int l1;   // sum of |q_k|, all dims
  int nt;   // ceil(sqrt(sum of squares of dims 8-23))
  int bad;
};
__device__ __forceinline__ uint32_t q8_word(uint32_t w0, uint32_t w1, __half2& amax) {
  const __half2 k127 = __float2half2_rn(127.0f), k1536 = __float2half2_rn(1536.0f);
  __half2 x0, x1;
  memcpy(&x0, &w0, 4);
  memcpy(&x1, &w1, 4);
  amax = __hmax2_nan(amax, __habs2(x0));  // NaN-propagating
  amax = __hmax2_nan(amax, __habs2(x1));
  const __half2 r0 = __hfma2(x0, k127, k1536), r1 = __hfma2(x1, k127, k1536);
  uint32_t u0, u1;
  memcpy(&u0, &r0, 4);
  memcpy(&u1, &r1, 4);
  return __byte_perm(u0, u1, 0x6420);  // low bytes of the four fp16 results
}
__device__ __forceinline__ Q8 quantize24(const uint4 d0, const uint4 d1, const uint4 d2) {
  Q8 q;
  __half2 amax = __float2half2_rn(0.0f);
  q.a.x = q8_word(d0.x, d0.y, amax);
  q.a.y = q8_word(d0.z, d0.w, amax);
  q.a.z = q8_word(d1.x, d1.y, amax);
  q.a.w = q8_word(d1.z, d1.w, amax);
  q.b.x = q8_word(d2.x, d2.y, amax);
  q.b.y = q8_word(d2.z, d2.w, amax);
  const float2 m = __half22float2(amax);
  q.bad = !(m.x <= 1.00390625f && m.y <= 1.00390625f);  // also NaN / inf
  constexpr int kOnes = 0x01010101;  // |q| <= 127 for a valid row, so the bytes stay positive as int8
  int l1 = __dp4a((int)__vabsss4(q.a.x), kOnes, 0);
  l1 = __dp4a((int)__vabsss4(q.a.y), kOnes, l1);
  l1 = __dp4a((int)__vabsss4(q.a.z), kOnes, l1);
  l1 = __dp4a((int)__vabsss4(q.a.w), kOnes, l1);
  l1 = __dp4a((int)__vabsss4(q.b.x), kOnes, l1);
  q.l1 = __dp4a((int)__vabsss4(q.b.y), kOnes, l1);
#if PMX_PRUNE  // the tail bound only feeds the pruned form
  int l2t = __dp4a((int)q.a.z, (int)q.a.z, 0);
  l2t = __dp4a((int)q.a.w, (int)q.a.w, l2t);
  l2t = __dp4a((int)q.b.x, (int)q.b.x, l2t);
  l2t = __dp4a((int)q.b.y, (int)q.b.y, l2t);
  int nt = (int)ceilf(sqrtf((float)l2t));  // exact integer ceil(sqrt): l2t < 2^24
  if (nt * nt < l2t) ++nt;
  q.nt = nt;
#else
  q.nt = 0;
#endif
  return q;
}

// ---------------------------------------------------------------- K1
// Norm keys of median_scene_distance (camera.cpp:181-186: valid pixels with
// |p| > 1e-12, FP64 norm as normalize_rays) + pass 1 of the radix select.
__global__ void __launch_bounds__(256) k_keys(const PairDev* __restrict__ pairs, int px_per_block) {
  const PairDev& P = pairs[blockIdx.y];
  const int HW = P.Ha * P.Wa;
  __shared__ uint32_t sh[kHist1];
  for (int i = threadIdx.x; i < kHist1; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int begin = blockIdx.x * px_per_block;
  const int end = min(HW, begin + px_per_block);
  for (int i = begin + threadIdx.x; i < end; i += blockDim.x) {
    const double x = P.xa[3 * i], y = P.xa[3 * i + 1], z = P.xa[3 * i + 2];
    const bool v = P.va ? P.va[i] != 0 : true;
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    uint32_t key = kNoKey;
    if (v && nrm > 1e-12) key = __float_as_uint((float)nrm);
    hist_add(sh, key >> 20, key != kNoKey);
    P.keys[i] = key;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHist1; i += blockDim.x)
    if (sh[i]) atomicAdd(&P.hist[i], sh[i]);
}

// Per-chunk a-side maps: FP64 unit rays (camera.cpp:39-56: norm in FP64,
// exact division as the reference), the int8 descriptor image for the
// refinement (+ its per-pair error-bound statistics), or the fp32 norm bounds
// of the standalone refine.
__global__ void __launch_bounds__(256) k_prep(const PairDev* __restrict__ pairs, int px_per_block, bool with_keys) {
  const PairDev& P = pairs[blockIdx.y];
  const int HW = P.Ha * P.Wa;
  const int begin = blockIdx.x * px_per_block;
  const int end = min(HW, begin + px_per_block);
  // with_keys: also the median's norm keys and their first histogram level
  // (k_keys folded in: one read of X_a instead of two)
  __shared__ uint32_t sh[kHist1];
  if (with_keys) {
    for (int i = threadIdx.x; i < kHist1; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  int a1max = 0, qbad = 0;
  for (int i = begin + threadIdx.x; i < end; i += blockDim.x) {
    const double x = P.xa[3 * i], y = P.xa[3 * i + 1], z = P.xa[3 * i + 2];
    const bool v = P.va ? P.va[i] != 0 : true;
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    if (with_keys) {  // k_keys
      uint32_t key = kNoKey;
      if (v && nrm > 1e-12) key = __float_as_uint((float)nrm);
      hist_add(sh, key >> 20, key != kNoKey);
      P.keys[i] = key;
    }
    // invalid: w = 0, and (PMX_RAY24) NaN components, so the LM's 24-byte
    // gathers see an invalid support through the NaN its weighted sum takes
    double4 r = PMX_RAY24 ? make_double4(CUDART_NAN, CUDART_NAN, CUDART_NAN, 0.0) : make_double4(0.0, 0.0, 1.0, 0.0);
    if (v && !(nrm < 1e-12) && isfinite(nrm)) r = make_double4(x / nrm, y / nrm, z / nrm, 1.0);
    P.rays[i] = r;
    if (P.dnorm) desc_aux(P.da + (size_t)i * 24, P.qa[i], P.dnorm + i);
    if (P.q8h) {
      const uint4* row = reinterpret_cast<const uint4*>(P.da) + 3 * (size_t)i;
      const Q8 q = quantize24(__ldg(row), __ldg(row + 1), __ldg(row + 2));
      P.q8h[i] = make_uint2(q.a.x, q.a.y);
      if (PMX_PRUNE) P.q8n[i] = (uint16_t)q.nt;  // the tail bound only feeds the pruned form
      P.q8t[i] = make_uint4(q.a.z, q.a.w, q.b.x, q.b.y);
      a1max = max(a1max, q.l1);
      qbad |= q.bad;
    }
  }
  if (P.q8h) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a1max = max(a1max, __shfl_xor_sync(0xffffffffu, a1max, o));
      qbad |= __shfl_xor_sync(0xffffffffu, qbad, o);
    }
    if ((threadIdx.x & 31) == 0) {
      if (a1max) atomicMax(&P.sel->a1max, a1max);
      if (qbad) atomicOr(&P.sel->qbad, qbad);
    }
  }
  if (with_keys) {
    __syncthreads();
    for (int i = threadIdx.x; i < kHist1; i += blockDim.x)
      if (sh[i]) atomicAdd(&P.hist[i], sh[i]);
  }
}

__global__ void __launch_bounds__(256) k_desc_prep(const __half* __restrict__ da, const float* __restrict__ qa,
                                                   int hw, float4* dnorm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hw) desc_aux(da + (size_t)i * 24, qa[i], dnorm + i);
}

// ---------------------------------------------------------------- K2
// One block per pair: locate the bucket holding rank krem.
template <int PASS>
__global__ void __launch_bounds__(1024) k_sel_scan(const PairDev* __restrict__ pairs, double fraction) {
  const PairDev& P = pairs[blockIdx.x];
  constexpr int NB = PASS == 1 ? kHist1 : PASS == 2 ? kHist2 : kHist3;
  const uint32_t* h = P.hist + (PASS == 1 ? 0 : PASS == 2 ? kHist1 : kHist1 + kHist2);
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t total;
  const int t = threadIdx.x;
  constexpr int PER = (NB + 1023) / 1024;
  uint32_t local[PER];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int b = t * PER + j;
    local[j] = b < NB ? h[b] : 0u;
    s += local[j];
  }
  // block exclusive scan of per-thread sums
  uint32_t incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += y;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    uint32_t w = wsum[t];
    uint32_t wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (t >= o) wi += y;
    }
    wsum[t] = wi - w;
    if (t == 31) total = wi;
  }
  __syncthreads();
  uint32_t excl = wsum[t >> 5] + incl - s;
  SelState* st = P.sel;
  __shared__ uint32_t krem_s;
  if (t == 0) {
    if (PASS == 1) {
      st->n = total;
      st->k = total / 2;
      st->krem = total / 2;
    }
    krem_s = st->krem;  // read once: the matching thread rewrites st->krem below
  }
  __syncthreads();
  const uint32_t krem = krem_s;
  if (total == 0) {
    if (t == 0) {
      st->prefix = 0;
      if (PASS == 3 || PASS == 1) st->threshold = fraction * 0.0;  // empty -> median 0
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int b = t * PER + j;
    if (b < NB && local[j] > 0 && excl <= krem && krem < excl + local[j]) {
      if (PASS == 1) {
        st->prefix = (uint32_t)b;
      } else if (PASS == 2) {
        st->prefix = (st->prefix << 12) | (uint32_t)b;
      } else {
        // the fp32 key of the rank-k norm; k_sel_exact resolves it to the
        // FP64 norm (the keys are fp32 roundings of FP64 norms: monotone, so
        // the median is the krem-th smallest FP64 norm among those with this key)
        const uint32_t key = (st->prefix << 8) | (uint32_t)b;
        st->key = key;
        st->ties = local[j];
        st->threshold = fraction * (double)__uint_as_float(key);
      }
      st->krem = krem - excl;
    }
    excl += local[j];
  }
}

template <int PASS>
__global__ void __launch_bounds__(256) k_sel_hist(const PairDev* __restrict__ pairs, int px_per_block) {
  const PairDev& P = pairs[blockIdx.y];
  const int HW = P.Ha * P.Wa;
  if (P.sel->n == 0) return;
  constexpr int NB = PASS == 2 ? kHist2 : kHist3;
  uint32_t* h = P.hist + (PASS == 2 ? kHist1 : kHist1 + kHist2);
  __shared__ uint32_t sh[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t prefix = P.sel->prefix;
  const int begin = blockIdx.x * px_per_block;
  const int end = min(HW, begin + px_per_block);
  auto add = [&](uint32_t key) {
    const bool take = key != kNoKey && (PASS == 2 ? (key >> 20) == prefix : (key >> 8) == prefix);
#if PMX_SEL_DIRECT_ATOMICS
    // the low bits of keys inside one bucket spread over the bins: plain
    // shared-memory atomics (rarely conflicting) beat warp aggregation
    if (take) atomicAdd(&sh[PASS == 2 ? (key >> 8) & 0xfff : key & 0xff], 1u);
#else
    hist_add(sh, PASS == 2 ? (key >> 8) & 0xfff : key & 0xff, take);
#endif
  };
  int i0 = begin;
  if ((reinterpret_cast<uintptr_t>(P.keys + begin) & 15) == 0) {  // 16-byte body
    const int nv = (end - begin) >> 2;
    const uint4* v = reinterpret_cast<const uint4*>(P.keys + begin);
    for (int j = threadIdx.x; j < nv; j += blockDim.x) {
      const uint4 k4 = v[j];
      add(k4.x);
      add(k4.y);
      add(k4.z);
      add(k4.w);
    }
    i0 = begin + 4 * nv;
  }
  for (int i = i0 + threadIdx.x; i < end; i += blockDim.x) add(P.keys[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += blockDim.x)
    if (sh[i]) atomicAdd(&h[i], sh[i]);
}

// FP64 norm of an a-pixel exactly as normalize_rays / median_scene_distance
// compute it (camera.cpp:49, 183: x*x + y*y + z*z in order, no FMA, sqrt).
__device__ __forceinline__ double norm64(const float* __restrict__ xa, int i) {
  const double x = xa[3 * i], y = xa[3 * i + 1], z = xa[3 * i + 2];
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// Exact median, step 1: the FP64 norms whose fp32 key equals the selected key
// (st->ties of them; kept when there are at most kSelCap).
__global__ void __launch_bounds__(256) k_sel_collect(const PairDev* __restrict__ pairs, int px_per_block) {
  const PairDev& P = pairs[blockIdx.y];
  SelState* st = P.sel;
  if (st->n == 0 || st->ties > (uint32_t)kSelCap) return;
  const uint32_t key = st->key;
  const int HW = P.Ha * P.Wa;
  const int begin = blockIdx.x * px_per_block;
  const int end = min(HW, begin + px_per_block);
  auto take = [&](uint32_t k, int i) {
    if (k != key) return;
    const uint32_t slot = atomicAdd(&st->cnt, 1u);
    if (slot < (uint32_t)kSelCap) st->cand[slot] = norm64(P.xa, i);
  };
  int i0 = begin;
  if ((reinterpret_cast<uintptr_t>(P.keys + begin) & 15) == 0) {  // 16-byte body
    const int nv = (end - begin) >> 2;
    const uint4* v = reinterpret_cast<const uint4*>(P.keys + begin);
    for (int j = threadIdx.x; j < nv; j += blockDim.x) {
      const uint4 k4 = v[j];
      const int i = begin + 4 * j;
      take(k4.x, i);
      take(k4.y, i + 1);
      take(k4.z, i + 2);
      take(k4.w, i + 3);
    }
    i0 = begin + 4 * nv;
  }
  for (int i = i0 + threadIdx.x; i < end; i += blockDim.x) take(P.keys[i], i);
}

// Exact median, step 2 (one block per pair): the krem-th smallest of the
// tied FP64 norms -> median and threshold = fraction * median (camera.cpp:
// 188-190, 199-200).  More than kSelCap ties (adversarial inputs): exact
// bisection over the FP64 bit patterns of the tied norms (positive doubles
// order as their bit patterns), one counting pass over the pair per step.
__global__ void __launch_bounds__(256) k_sel_exact(const PairDev* __restrict__ pairs, double fraction) {
  const PairDev& P = pairs[blockIdx.x];
  SelState* st = P.sel;
  if (st->n == 0) {
    if (threadIdx.x == 0) st->median = 0.0;
    return;
  }
  const uint32_t krem = st->krem, ties = st->ties;
  if (ties <= (uint32_t)kSelCap) {
    for (uint32_t t = threadIdx.x; t < ties; t += blockDim.x) {
      const double v = st->cand[t];
      uint32_t less = 0, eq = 0;
      for (uint32_t o = 0; o < ties; ++o) {
        less += st->cand[o] < v;
        eq += st->cand[o] == v;
      }
      if (less <= krem && krem < less + eq) {  // equal values write the same result
        st->median = v;
        st->threshold = fraction * v;
      }
    }
    return;
  }
  __shared__ unsigned long long lo_s, hi_s;
  __shared__ uint32_t count_s;
  const uint32_t key = st->key;
  const int HW = P.Ha * P.Wa;
  if (threadIdx.x == 0) {
    lo_s = 0ull;
    hi_s = 0x7ff0000000000000ull;  // +inf
  }
  __syncthreads();
  for (int step = 0; step < 64; ++step) {
    const unsigned long long lo = lo_s, hi = hi_s;
    if (lo >= hi) break;
    const unsigned long long mid = lo + (hi - lo) / 2;
    if (threadIdx.x == 0) count_s = 0;
    __syncthreads();
    uint32_t c = 0;
    for (int i = threadIdx.x; i < HW; i += blockDim.x)
      if (P.keys[i] == key && (unsigned long long)__double_as_longlong(norm64(P.xa, i)) <= mid) ++c;
    atomicAdd(&count_s, c);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (count_s >= krem + 1)
        hi_s = mid;
      else
        lo_s = mid + 1;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double v = __longlong_as_double((long long)lo_s);
    st->median = v;
    st->threshold = fraction * v;
  }
}

// ---------------------------------------------------------------- LM
#ifndef PMX_LM_RSQRT
#define PMX_LM_RSQRT 1  // the LM's ray normalisation: MUFU estimate + two Newton steps (~1 ulp) instead of rsqrt()
#endif
__device__ __forceinline__ double lm_rsqrt(double x) {
#if PMX_LM_RSQRT
  // x = |g|^2 of an interpolated unit-ray combination: within [1e-24, 1],
  // far from the subnormal range ftz touches
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x * y, y, 1.0);
  return fma(0.5 * y, e, y);
#else
  return rsqrt(x);
#endif
}

// One 256-bit load per support (LDG.E.ENL2.256 on sm_100: 32-byte aligned
// double4 through the read-only path).
__device__ __forceinline__ double4 ld_ray(const double4* __restrict__ rays, int i) {
#if PMX_LD256
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(rays + i));
  return v;
#else
  const double2* p = reinterpret_cast<const double2*>(rays + i);
  const double2 a = __ldg(p), b = __ldg(p + 1);
  return make_double4(a.x, a.y, b.x, b.y);
#endif
}

// interpolate_ray, camera.cpp:58-100, split so the 3x2 Jacobian is only
// formed for accepted points (the reference computes it for every trial;
// the value is identical, it is just never used when a trial is rejected).
// (An eager-Jacobian form that lets the supports die early measured ~1%
// slower: the extra FP64 work of rejected trials outweighs the registers.)
struct Interp {
  double r0, r1, r2;  // unit ray g / |g|
  double rs;          // 1 / |g|
  double fu, fv;
  double4 c00, c10, c01, c11;
};

// All four supports are loaded before any test (no load -> branch -> load
// round trips); the validity and |g| tests are applied to the result.
__device__ __forceinline__ bool interp_eval(const double4* __restrict__ rays, int W, int H, double u, double v,
                                            Interp& I) {
  if (u < 0.0 || v < 0.0 || u > (double)(W - 1) || v > (double)(H - 1)) return false;
  int u0 = (int)floor(u);
  int v0 = (int)floor(v);
  u0 = min(u0, W - 2 >= 0 ? W - 2 : 0);
  v0 = min(v0, H - 2 >= 0 ? H - 2 : 0);
  const int du = min(u0 + 1, W - 1) - u0, dv = (min(v0 + 1, H - 1) - v0) * W;
  int base = v0 * W + u0;
  PMX_CHECK_INDEX(base, W * H - dv - du);  // all four supports inside the map
  const double4* p = rays + base;
  I.fu = u - u0;
  I.fv = v - v0;
  I.c00 = ld_ray(p, 0);
  I.c10 = ld_ray(p, du);
  I.c01 = ld_ray(p, dv);
  I.c11 = ld_ray(p, dv + du);
  const double fu = I.fu, fv = I.fv;
  const double w00 = (1 - fu) * (1 - fv), w10 = fu * (1 - fv), w01 = (1 - fu) * fv, w11 = fu * fv;
  const double g0 = w00 * I.c00.x + w10 * I.c10.x + w01 * I.c01.x + w11 * I.c11.x;
  const double g1 = w00 * I.c00.y + w10 * I.c10.y + w01 * I.c01.y + w11 * I.c11.y;
  const double g2 = w00 * I.c00.z + w10 * I.c10.z + w01 * I.c01.z + w11 * I.c11.z;
  const double gg = g0 * g0 + g1 * g1 + g2 * g2;
  const bool valid = I.c00.w != 0.0 && I.c10.w != 0.0 && I.c01.w != 0.0 && I.c11.w != 0.0;
  if (!valid || gg < 1e-24) return false;  // an invalid support / |g| < 1e-12
  I.rs = lm_rsqrt(gg);
  I.r0 = g0 * I.rs;
  I.r1 = g1 * I.rs;
  I.r2 = g2 * I.rs;
  return true;
}

// The LM's form of interp_eval (PMX_RAY24): 24-byte supports (x, y, z: one
// 16-byte + one 8-byte load), validity from the NaN an invalid support puts
// into the weighted sum (weights are finite, 0 x NaN = NaN).  8 fewer
// registers per live support set and 25% fewer L1 wavefronts than the
// 256-bit form; same values.
struct Interp3 {
  double r0, r1, r2;
  double rs;
  double fu, fv;
  double3 c00, c10, c01, c11;
};

__device__ __forceinline__ double3 ld_ray3(const double4* __restrict__ rays, int i) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(rays + i));
  const double c = __ldg(reinterpret_cast<const double*>(rays + i) + 2);
  return make_double3(a.x, a.y, c);
}

__device__ __forceinline__ bool interp_eval(const double4* __restrict__ rays, int W, int H, double u, double v,
                                            Interp3& I) {
  if (u < 0.0 || v < 0.0 || u > (double)(W - 1) || v > (double)(H - 1)) return false;
  int u0 = (int)floor(u);
  int v0 = (int)floor(v);
  u0 = min(u0, W - 2 >= 0 ? W - 2 : 0);
  v0 = min(v0, H - 2 >= 0 ? H - 2 : 0);
  const int du = min(u0 + 1, W - 1) - u0, dv = (min(v0 + 1, H - 1) - v0) * W;
  int base = v0 * W + u0;
  PMX_CHECK_INDEX(base, W * H - dv - du);
  I.fu = u - u0;
  I.fv = v - v0;
  I.c00 = ld_ray3(rays, base);
  I.c10 = ld_ray3(rays, base + du);
  I.c01 = ld_ray3(rays, base + dv);
  I.c11 = ld_ray3(rays, base + dv + du);
  const double fu = I.fu, fv = I.fv;
  const double w00 = (1 - fu) * (1 - fv), w10 = fu * (1 - fv), w01 = (1 - fu) * fv, w11 = fu * fv;
  const double g0 = w00 * I.c00.x + w10 * I.c10.x + w01 * I.c01.x + w11 * I.c11.x;
  const double g1 = w00 * I.c00.y + w10 * I.c10.y + w01 * I.c01.y + w11 * I.c11.y;
  const double g2 = w00 * I.c00.z + w10 * I.c10.z + w01 * I.c01.z + w11 * I.c11.z;
  const double gg = g0 * g0 + g1 * g1 + g2 * g2;
  if (!(gg >= 1e-24)) return false;  // an invalid support (NaN) / |g| < 1e-12
  I.rs = lm_rsqrt(gg);
  I.r0 = g0 * I.rs;
  I.r1 = g1 * I.rs;
  I.r2 = g2 * I.rs;
  return true;
}

// J = (I - r r^T) / |g| [dg/du, dg/dv]  (camera.cpp:92-98)
__device__ __forceinline__ void interp_jac(const Interp& I, double J[6]) {
  const double fu = I.fu, fv = I.fv;
  const double du0 = (1 - fv) * (I.c10.x - I.c00.x) + fv * (I.c11.x - I.c01.x);
  const double du1 = (1 - fv) * (I.c10.y - I.c00.y) + fv * (I.c11.y - I.c01.y);
  const double du2 = (1 - fv) * (I.c10.z - I.c00.z) + fv * (I.c11.z - I.c01.z);
  const double dv0 = (1 - fu) * (I.c01.x - I.c00.x) + fu * (I.c11.x - I.c10.x);
  const double dv1 = (1 - fu) * (I.c01.y - I.c00.y) + fu * (I.c11.y - I.c10.y);
  const double dv2 = (1 - fu) * (I.c01.z - I.c00.z) + fu * (I.c11.z - I.c10.z);
  const double rdu = I.r0 * du0 + I.r1 * du1 + I.r2 * du2;
  const double rdv = I.r0 * dv0 + I.r1 * dv1 + I.r2 * dv2;
  J[0] = (du0 - I.r0 * rdu) * I.rs;
  J[1] = (du1 - I.r1 * rdu) * I.rs;
  J[2] = (du2 - I.r2 * rdu) * I.rs;
  J[3] = (dv0 - I.r0 * rdv) * I.rs;
  J[4] = (dv1 - I.r1 * rdv) * I.rs;
  J[5] = (dv2 - I.r2 * rdv) * I.rs;
}

// Full form (ray + Jacobian), kept for the fine-grained entry points.
__device__ __forceinline__ bool interp_ray(const double4* __restrict__ rays, int W, int H, double u,
                                           double v, double ray[3], double J[6]) {
  Interp I;
  if (!interp_eval(rays, W, H, u, v, I)) return false;
  ray[0] = I.r0;
  ray[1] = I.r1;
  ray[2] = I.r2;
  interp_jac(I, J);
  return true;
}

// PMX_LM_F32: the LM's step direction in fp32.  Only the decisions need
// FP64 - the ray, r = ray - t (a difference of nearly equal unit vectors),
// the cost |r|^2 and the convergence dot are kept FP64; the Jacobian, J^T J,
// J^T r and the 2x2 damped solve only steer the step, and a ~1e-7 relative
// change of a step moves the next iterate by ~1e-7 of the step (the same
// class of perturbation as the rsqrt normalisation), far from the decision
// boundaries except in the rare stalled-LM end game.
// Jacobian storage of the fp32 LM: registers, or (JSm) a thread's column
// of a shared-memory array - the loop-carried J otherwise spills to local
// memory at 64 registers.
struct JReg {
  float v[6];
  __device__ __forceinline__ float& operator[](int k) { return v[k]; }
};
template <int STRIDE>
struct JSm {
  float* p;
  __device__ __forceinline__ float& operator[](int k) { return p[k * STRIDE]; }
};

template <class IP, class JT>
__device__ __forceinline__ void interp_jac_f(const IP& I, JT& J) {
  const float fu = (float)I.fu, fv = (float)I.fv;
  const float a0 = (float)(I.c10.x - I.c00.x), a1 = (float)(I.c10.y - I.c00.y), a2 = (float)(I.c10.z - I.c00.z);
  const float b0 = (float)(I.c11.x - I.c01.x), b1 = (float)(I.c11.y - I.c01.y), b2 = (float)(I.c11.z - I.c01.z);
  const float c0 = (float)(I.c01.x - I.c00.x), c1 = (float)(I.c01.y - I.c00.y), c2 = (float)(I.c01.z - I.c00.z);
  const float e0 = (float)(I.c11.x - I.c10.x), e1 = (float)(I.c11.y - I.c10.y), e2 = (float)(I.c11.z - I.c10.z);
  const float du0 = fmaf(fv, b0 - a0, a0), du1 = fmaf(fv, b1 - a1, a1), du2 = fmaf(fv, b2 - a2, a2);
  const float dv0 = fmaf(fu, e0 - c0, c0), dv1 = fmaf(fu, e1 - c1, c1), dv2 = fmaf(fu, e2 - c2, c2);
  const float r0 = (float)I.r0, r1 = (float)I.r1, r2 = (float)I.r2, rs = (float)I.rs;
  const float rdu = fmaf(r0, du0, fmaf(r1, du1, r2 * du2)), rdv = fmaf(r0, dv0, fmaf(r1, dv1, r2 * dv2));
  J[0] = fmaf(-r0, rdu, du0) * rs;
  J[1] = fmaf(-r1, rdu, du1) * rs;
  J[2] = fmaf(-r2, rdu, du2) * rs;
  J[3] = fmaf(-r0, rdv, dv0) * rs;
  J[4] = fmaf(-r1, rdv, dv1) * rs;
  J[5] = fmaf(-r2, rdv, dv2) * rs;
}

// Eager form of the fp32 path: interp_eval_f keeps only what the step needs
// - the FP64 unit ray, and the fp32 dg/du, dg/dv and 1/|g| - so the four
// FP64 supports (32 registers) die inside the interpolation instead of
// living until the accept test.  Same operations as interp_jac_f on the
// same values (identical Jacobian); the differences are also formed for
// trials that end up rejected (rare at lambda = 1e-8).
struct InterpF {
  double r0, r1, r2;  // unit ray g / |g|
  float rs;           // 1 / |g|
  float du[3], dv[3];
};

// The four supports of an interpolation and the fractional offsets.
struct Corners {
  double4 c00, c10, c01, c11;
  double fu, fv;
};

__device__ __forceinline__ void corners_load(const double4* __restrict__ rays, int W, int H, double u, double v,
                                             Corners& C) {
  int u0 = (int)floor(u);
  int v0 = (int)floor(v);
  u0 = min(u0, W - 2 >= 0 ? W - 2 : 0);
  v0 = min(v0, H - 2 >= 0 ? H - 2 : 0);
  const int du = min(u0 + 1, W - 1) - u0, dv = (min(v0 + 1, H - 1) - v0) * W;
  int base = v0 * W + u0;
  PMX_CHECK_INDEX(base, W * H - dv - du);
  const double4* p = rays + base;
  C.fu = u - u0;
  C.fv = v - v0;
  C.c00 = ld_ray(p, 0);
  C.c10 = ld_ray(p, du);
  C.c01 = ld_ray(p, dv);
  C.c11 = ld_ray(p, dv + du);
}

__device__ __forceinline__ bool interp_math_f(const Corners& C, InterpF& I) {
  const double4 &c00 = C.c00, &c10 = C.c10, &c01 = C.c01, &c11 = C.c11;
  const double fu = C.fu, fv = C.fv;
  const double w00 = (1 - fu) * (1 - fv), w10 = fu * (1 - fv), w01 = (1 - fu) * fv, w11 = fu * fv;
  const double g0 = w00 * c00.x + w10 * c10.x + w01 * c01.x + w11 * c11.x;
  const double g1 = w00 * c00.y + w10 * c10.y + w01 * c01.y + w11 * c11.y;
  const double g2 = w00 * c00.z + w10 * c10.z + w01 * c01.z + w11 * c11.z;
  const double gg = g0 * g0 + g1 * g1 + g2 * g2;
#if PMX_VALID_BITS
  // w is exactly 1.0 (valid) or 0.0 (k_prep): all four valid iff the AND of
  // their high words (0x3ff00000 or 0) is non-zero - integer ops, not DSETPs
  const bool valid = (__double2hiint(c00.w) & __double2hiint(c10.w) & __double2hiint(c01.w) & __double2hiint(c11.w)) != 0;
#else
  const bool valid = c00.w != 0.0 && c10.w != 0.0 && c01.w != 0.0 && c11.w != 0.0;
#endif
  if (!valid || gg < 1e-24) return false;
  const double rs = lm_rsqrt(gg);
  I.r0 = g0 * rs;
  I.r1 = g1 * rs;
  I.r2 = g2 * rs;
  I.rs = (float)rs;
  const float ffu = (float)fu, ffv = (float)fv;
#if PMX_JDIFF_F32
  // differences of the fp32-rounded supports (steering only; ~2e-5 relative)
  const float x00 = (float)c00.x, y00 = (float)c00.y, z00 = (float)c00.z;
  const float x10 = (float)c10.x, y10 = (float)c10.y, z10 = (float)c10.z;
  const float x01 = (float)c01.x, y01 = (float)c01.y, z01 = (float)c01.z;
  const float x11 = (float)c11.x, y11 = (float)c11.y, z11 = (float)c11.z;
  const float a0 = x10 - x00, a1 = y10 - y00, a2 = z10 - z00;
  const float b0 = x11 - x01, b1 = y11 - y01, b2 = z11 - z01;
  const float d0 = x01 - x00, d1 = y01 - y00, d2 = z01 - z00;
  const float e0 = x11 - x10, e1 = y11 - y10, e2 = z11 - z10;
#else
  const float a0 = (float)(c10.x - c00.x), a1 = (float)(c10.y - c00.y), a2 = (float)(c10.z - c00.z);
  const float b0 = (float)(c11.x - c01.x), b1 = (float)(c11.y - c01.y), b2 = (float)(c11.z - c01.z);
  const float d0 = (float)(c01.x - c00.x), d1 = (float)(c01.y - c00.y), d2 = (float)(c01.z - c00.z);
  const float e0 = (float)(c11.x - c10.x), e1 = (float)(c11.y - c10.y), e2 = (float)(c11.z - c10.z);
#endif
  I.du[0] = fmaf(ffv, b0 - a0, a0);
  I.du[1] = fmaf(ffv, b1 - a1, a1);
  I.du[2] = fmaf(ffv, b2 - a2, a2);
  I.dv[0] = fmaf(ffu, e0 - d0, d0);
  I.dv[1] = fmaf(ffu, e1 - d1, d1);
  I.dv[2] = fmaf(ffu, e2 - d2, d2);
  return true;
}

__device__ __forceinline__ bool interp_eval_f(const double4* __restrict__ rays, int W, int H, double u, double v,
                                              InterpF& I) {
  // the LM only evaluates clamped points (the seed and clamp_to_image's
  // trials, camera.cpp:104-107, 124-125): the range test of interpolate_ray
  // always passes there and is not repeated (the API entry keeps it)
  Corners C;
  corners_load(rays, W, H, u, v, C);
  return interp_math_f(C, I);
}

template <class JT>
__device__ __forceinline__ void interp_jac_f(const InterpF& I, JT& J) {
  const float r0 = (float)I.r0, r1 = (float)I.r1, r2 = (float)I.r2, rs = I.rs;
  const float rdu = fmaf(r0, I.du[0], fmaf(r1, I.du[1], r2 * I.du[2]));
  const float rdv = fmaf(r0, I.dv[0], fmaf(r1, I.dv[1], r2 * I.dv[2]));
  J[0] = fmaf(-r0, rdu, I.du[0]) * rs;
  J[1] = fmaf(-r1, rdu, I.du[1]) * rs;
  J[2] = fmaf(-r2, rdu, I.du[2]) * rs;
  J[3] = fmaf(-r0, rdv, I.dv[0]) * rs;
  J[4] = fmaf(-r1, rdv, I.dv[1]) * rs;
  J[5] = fmaf(-r2, rdv, I.dv[2]) * rs;
}

__device__ __forceinline__ void ldlt2_solve_f(float h00, float h01, float h11, float b0, float b1, float* x0,
                                              float* x1) {
  const bool sw = fabsf(h11) > fabsf(h00);
  const float m00 = sw ? h11 : h00;
  float m11 = sw ? h00 : h11;
  if (!(fabsf(m00) > 0.0f)) {
    *x0 = 0.0f;
    *x1 = 0.0f;
    return;
  }
  // approximate reciprocals (MUFU, ~1 ulp): the step only steers the LM
  const float i00 = __fdividef(1.0f, m00);
  const float m10 = h01 * i00;
  m11 -= m10 * (m00 * m10);
  float d0 = sw ? b1 : b0, d1 = sw ? b0 : b1;
  d1 -= m10 * d0;
  d0 = d0 * i00;
  d1 = fabsf(m11) > 1.17549435e-38f ? __fdividef(d1, m11) : 0.0f;
  d0 -= m10 * d1;
  *x0 = sw ? d1 : d0;
  *x1 = sw ? d0 : d1;
}

// 2x2 instance of Eigen's pivoted LDLT solve (camera.cpp:147), same ops as
// ldlt_pivoted_solve(2, ...).
__device__ __forceinline__ void ldlt2_solve(double h00, double h01, double h11, double b0, double b1,
                                            double* x0, double* x1) {
  const bool sw = fabs(h11) > fabs(h00);
  double m00 = sw ? h11 : h00, m11 = sw ? h00 : h11;
  double m10 = h01;
  if (!(fabs(m00) > 0.0)) {
    *x0 = 0.0;
    *x1 = 0.0;
    return;
  }
  // the quotients of Eigen's LDLT as products with reciprocals (within 1-2
  // ulp of the IEEE quotients, like the rsqrt normalisation of interp_eval)
#if PMX_RCP
  const double i00 = rcp64(m00);
  m10 *= i00;
#else
  m10 /= m00;
#endif
  const double temp0 = m00 * m10;
  m11 -= m10 * temp0;
  double d0 = sw ? b1 : b0, d1 = sw ? b0 : b1;
  d1 -= m10 * d0;
  const double tiny = 2.2250738585072014e-308;
#if PMX_RCP
  d0 = fabs(m00) > tiny ? d0 * i00 : 0.0;
  d1 = fabs(m11) > tiny ? d1 * rcp64(m11) : 0.0;
#else
  d0 = fabs(m00) > tiny ? d0 / m00 : 0.0;
  d1 = fabs(m11) > tiny ? d1 / m11 : 0.0;
#endif
  d0 -= m10 * d1;
  *x0 = sw ? d1 : d0;
  *x1 = sw ? d0 : d1;
}

struct ProjOut {
  double pu, pv;
  bool converged;
  int iterations;
};

// iterative_project, camera.cpp:115-174.  SEED_CLAMPED: the caller passes an
// integer seed already clamped into the image (the matcher's pixel seeds), so
// the FP64 clamp of camera.cpp:124-125 is the identity and is skipped.
template <class JT = JReg, bool SEED_CLAMPED = false>
__device__ __forceinline__ ProjOut iterative_project_dev(const double4* __restrict__ rays, int W, int H, double x0,
                                                         double x1, double x2, double pu0, double pv0,
                                                         const LMParams& lp, JT J = JT(),
                                                         const Corners* pre = nullptr) {
  ProjOut res;
  res.converged = false;
  res.iterations = 0;
  const double cu = SEED_CLAMPED ? pu0 : fmin(fmax(pu0, 0.0), (double)(W - 1));
  const double cv = SEED_CLAMPED ? pv0 : fmin(fmax(pv0, 0.0), (double)(H - 1));
#if PMX_LM_RSQRT
  // |x| < 1e-12 as |x|^2 < 1e-24, and x / |x| as x * rsqrt(|x|^2) (~1 ulp)
  const double xx = x0 * x0 + x1 * x1 + x2 * x2;
  if (xx < 1e-24 || !(isfinite(x0) && isfinite(x1) && isfinite(x2))) {
    res.pu = cu;
    res.pv = cv;
    return res;
  }
  const double ixn = lm_rsqrt(xx);
  const double t0 = x0 * ixn, t1 = x1 * ixn, t2 = x2 * ixn;
#else
  const double xn = sqrt(x0 * x0 + x1 * x1 + x2 * x2);
  if (xn < 1e-12 || !(isfinite(x0) && isfinite(x1) && isfinite(x2))) {
    res.pu = cu;
    res.pv = cv;
    return res;
  }
#if PMX_RCP
  const double ixn = rcp64(xn);
  const double t0 = x0 * ixn, t1 = x1 * ixn, t2 = x2 * ixn;
#else
  const double t0 = x0 / xn, t1 = x1 / xn, t2 = x2 / xn;
#endif
#endif
  double pu = cu, pv = cv;
#if PMX_LM_F32 && PMX_EAGER_F32
  InterpF I;
#define PMX_INTERP_EVAL interp_eval_f
#elif PMX_RAY24
  Interp3 I;
#define PMX_INTERP_EVAL interp_eval
#else
  Interp I;
#define PMX_INTERP_EVAL interp_eval
#endif
#if PMX_LM_F32 && PMX_EAGER_F32
  // pre: the seed's supports, loaded by the caller with its own inputs
  const bool first_ok = pre ? interp_math_f(*pre, I) : PMX_INTERP_EVAL(rays, W, H, pu, pv, I);
#else
  (void)pre;
  const bool first_ok = PMX_INTERP_EVAL(rays, W, H, pu, pv, I);
#endif
  if (!first_ok) {
    res.pu = pu;
    res.pv = pv;
    return res;
  }
  double ray0 = I.r0, ray1 = I.r1, ray2 = I.r2;
  double r0 = ray0 - t0, r1 = ray1 - t1, r2 = ray2 - t2;
  double cost = r0 * r0 + r1 * r1 + r2 * r2;
  if (ray0 * t0 + ray1 * t1 + ray2 * t2 >= lp.cos_tol) {
    res.pu = pu;
    res.pv = pv;
    res.converged = true;
    return res;
  }
#if PMX_LM_F32 && PMX_LM_NE_STATE
  // Loop state: the iterate, its FP64 cost, lambda and the fp32 normal
  // equations J^T J, J^T r of the current point - they only change when a
  // step is accepted, so they are formed there once (same fp32 operations on
  // the same values as forming them every iteration).  The FP64 ray is not
  // kept: every decision on it is taken at acceptance.
  (void)J;
  float a00, a01, a11, g0, g1;
  auto normal_eqs = [&](double e0, double e1, double e2) {
    float Jf[6];
    interp_jac_f(I, Jf);
    const float fr0 = (float)e0, fr1 = (float)e1, fr2 = (float)e2;
    a00 = fmaf(Jf[0], Jf[0], fmaf(Jf[1], Jf[1], Jf[2] * Jf[2]));
    a01 = fmaf(Jf[0], Jf[3], fmaf(Jf[1], Jf[4], Jf[2] * Jf[5]));
    a11 = fmaf(Jf[3], Jf[3], fmaf(Jf[4], Jf[4], Jf[5] * Jf[5]));
    g0 = fmaf(Jf[0], fr0, fmaf(Jf[1], fr1, Jf[2] * fr2));
    g1 = fmaf(Jf[3], fr0, fmaf(Jf[4], fr1, Jf[5] * fr2));
  };
  normal_eqs(r0, r1, r2);
  double lambda = lp.lambda_init;
  for (int it = 0; it < lp.max_iterations; ++it) {
    ++res.iterations;
    const float fl = (float)lambda;
    const float h00 = fmaf(fl, fmaxf(a00, 1e-12f), a00);
    const float h11 = fmaf(fl, fmaxf(a11, 1e-12f), a11);
    float fs0, fs1;
    ldlt2_solve_f(h00, a01, h11, g0, g1, &fs0, &fs1);
    if (!isfinite(fs0) || !isfinite(fs1)) break;
    const double d0 = -(double)fs0, d1 = -(double)fs1;
    // clamp_to_image (camera.cpp:104-107); pu + d0 is finite here
    const double xu = pu + d0, xv = pv + d1;
    const double tu = xu < 0.0 ? 0.0 : (xu > (double)(W - 1) ? (double)(W - 1) : xu);
    const double tv = xv < 0.0 ? 0.0 : (xv > (double)(H - 1) ? (double)(H - 1) : xv);
    if (PMX_INTERP_EVAL(rays, W, H, tu, tv, I)) {
      const double e0 = I.r0 - t0, e1 = I.r1 - t1, e2 = I.r2 - t2;
      const double ct = e0 * e0 + e1 * e1 + e2 * e2;
      if (ct < cost) {
        pu = tu;
        pv = tv;
        cost = ct;
        lambda *= lp.lambda_down;
        if (I.r0 * t0 + I.r1 * t1 + I.r2 * t2 >= lp.cos_tol) {
          res.pu = pu;
          res.pv = pv;
          res.converged = true;
          return res;
        }
        normal_eqs(e0, e1, e2);
        continue;
      }
    }
    lambda *= lp.lambda_up;
  }
  res.pu = pu;
  res.pv = pv;
  // the current point failed the convergence test when it was accepted (or
  // at the start): the reference's final test is false here
  res.converged = false;
  return res;
#else
#if PMX_LM_F32
  interp_jac_f(I, J);
#else
  double J[6];
  interp_jac(I, J);
#endif
  double lambda = lp.lambda_init;
  for (int it = 0; it < lp.max_iterations; ++it) {
    ++res.iterations;
    r0 = ray0 - t0;
    r1 = ray1 - t1;
    r2 = ray2 - t2;
#if PMX_LM_F32
    const float fr0 = (float)r0, fr1 = (float)r1, fr2 = (float)r2;
    const float a00 = fmaf(J[0], J[0], fmaf(J[1], J[1], J[2] * J[2]));
    const float a01 = fmaf(J[0], J[3], fmaf(J[1], J[4], J[2] * J[5]));
    const float a11 = fmaf(J[3], J[3], fmaf(J[4], J[4], J[5] * J[5]));
    const float g0 = fmaf(J[0], fr0, fmaf(J[1], fr1, J[2] * fr2));
    const float g1 = fmaf(J[3], fr0, fmaf(J[4], fr1, J[5] * fr2));
    const float fl = (float)lambda;
    const float h00 = fmaf(fl, fmaxf(a00, 1e-12f), a00);
    const float h11 = fmaf(fl, fmaxf(a11, 1e-12f), a11);
    float fs0, fs1;
    ldlt2_solve_f(h00, a01, h11, g0, g1, &fs0, &fs1);
    const double d0 = -(double)fs0, d1 = -(double)fs1;
#else
    const double a00 = J[0] * J[0] + J[1] * J[1] + J[2] * J[2];
    const double a01 = J[0] * J[3] + J[1] * J[4] + J[2] * J[5];
    const double a11 = J[3] * J[3] + J[4] * J[4] + J[5] * J[5];
    const double g0 = J[0] * r0 + J[1] * r1 + J[2] * r2;
    const double g1 = J[3] * r0 + J[4] * r1 + J[5] * r2;
    const double h00 = a00 + lambda * fmax(a00, 1e-12);
    const double h11 = a11 + lambda * fmax(a11, 1e-12);
    double s0, s1;
    ldlt2_solve(h00, a01, h11, g0, g1, &s0, &s1);
    const double d0 = -s0, d1 = -s1;
#endif
    if (!isfinite(d0) || !isfinite(d1)) break;
    // clamp_to_image (camera.cpp:104-107); pu + d0 is finite here
    const double xu = pu + d0, xv = pv + d1;
    const double tu = xu < 0.0 ? 0.0 : (xu > (double)(W - 1) ? (double)(W - 1) : xu);
    const double tv = xv < 0.0 ? 0.0 : (xv > (double)(H - 1) ? (double)(H - 1) : xv);
    if (PMX_INTERP_EVAL(rays, W, H, tu, tv, I)) {
      const double e0 = I.r0 - t0, e1 = I.r1 - t1, e2 = I.r2 - t2;
      const double ct = e0 * e0 + e1 * e1 + e2 * e2;
      if (ct < cost) {
        pu = tu;
        pv = tv;
        ray0 = I.r0;
        ray1 = I.r1;
        ray2 = I.r2;
        cost = ct;
        lambda *= lp.lambda_down;
        if (ray0 * t0 + ray1 * t1 + ray2 * t2 >= lp.cos_tol) {
          res.pu = pu;
          res.pv = pv;
          res.converged = true;
          return res;
        }
#if PMX_LM_F32
        interp_jac_f(I, J);
#else
        interp_jac(I, J);
#endif
        continue;
      }
    }
    lambda *= lp.lambda_up;
  }
  res.pu = pu;
  res.pv = pv;
  res.converged = ray0 * t0 + ray1 * t1 + ray2 * t2 >= lp.cos_tol;
  return res;
#endif
#undef PMX_INTERP_EVAL
}

// ------------------------------------------------------------ refine (K4)
// Exact dot of two fp16 descriptors exactly as the reference evaluates it
// in FP64 (products exact; sequential additions, no FMA).
__device__ __noinline__ double dot_exact(const __half* __restrict__ a, const __half* __restrict__ b,
                                         int dim) {
  double s = 0.0;
  for (int k = 0; k < dim; ++k)
    s = __dadd_rn(s, __dmul_rn((double)__half2float(a[k]), (double)__half2float(b[k])));
  return s;
}

// fp32 dot of a candidate against the register-resident target, with the
// candidate's max |component| (for the rounding-error bound).
template <int DIM>
__device__ __forceinline__ float dot_fast(const __half* __restrict__ a, const float (&bt)[DIM],
                                          float* amax) {
  const uint4* p = reinterpret_cast<const uint4*>(a);
  float s = 0.0f;
  __half2 m2 = __float2half2_rn(0.0f);
#pragma unroll
  for (int q = 0; q < DIM / 8; ++q) {
    const uint4 w = __ldg(p + q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      __half2 v;
      memcpy(&v, &ws[h], 4);
      m2 = __hmax2(m2, __habs2(v));
      const float2 f = __half22float2(v);
      s = fmaf(f.x, bt[8 * q + 2 * h], s);
      s = fmaf(f.y, bt[8 * q + 2 * h + 1], s);
    }
  }
  const float2 mf = __half22float2(m2);
  *amax = fmaxf(mf.x, mf.y);
  return s;
}

// Coarse-to-fine refinement of one match (camera.cpp:239-271) — returns the
// refined a-pixel index.  Candidates inside the previous level's window are
// skipped: they were all scored <= the running best, and only a strict '>'
// can move the best, so skipping them is exact.
template <int DIM>
__device__ __noinline__ int refine_one(const __half* __restrict__ Da, int Wa, int Ha, const __half* __restrict__ bdesc,
                          int pa, const RefineLevels& L) {
  float bt[DIM];
  float bnorm1 = 0.0f;
  {
    const uint4* p = reinterpret_cast<const uint4*>(bdesc);
#pragma unroll
    for (int q = 0; q < DIM / 8; ++q) {
      const uint4 w = __ldg(p + q);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        __half2 v;
        memcpy(&v, &ws[h], 4);
        const float2 f = __half22float2(v);
        bt[8 * q + 2 * h] = f.x;
        bt[8 * q + 2 * h + 1] = f.y;
        bnorm1 += fabsf(f.x) + fabsf(f.y);
      }
    }
  }
  // Error bound of an fp32 FMA chain with exact products:
  // |s - exact| <= DIM * u * sum|a_k b_k| <= DIM * u * max|a| * ||b||_1.
  const float gamma = (float)DIM * 5.9604645e-08f * 1.001f;
  int best_u = pa % Wa, best_v = pa / Wa;
  int prev_cu = 0, prev_cv = 0, prev_s = 0, prev_r = -1;
  for (int l = 0; l < L.n; ++l) {
    const int s = L.stride[l], r = L.radius[l];
    const int cu = best_u, cv = best_v;
    // identical window around the same centre: nothing can win (strict '>')
    if (l > 0 && s == prev_s && r == prev_r && cu == prev_cu && cv == prev_cv) continue;
    const __half* cdesc = Da + (size_t)(cv * Wa + cu) * DIM;
    float am;
    float best_f = dot_fast<DIM>(cdesc, bt, &am);
    float best_b = gamma * am * bnorm1;
    double best_x = 0.0;  // exact score when best_known
    bool best_known = false;
    for (int dv = -r; dv <= r; ++dv) {
      const int v = cv + dv * s;
      if (v < 0 || v >= Ha) continue;
      for (int du = -r; du <= r; ++du) {
        const int u = cu + du * s;
        if (u < 0 || u >= Wa) continue;
        if (du == 0 && dv == 0) continue;  // the centre never beats itself
        if (prev_r >= 0) {  // inside the previous level's (already maximised) window?
          const int eu = u - prev_cu, ev = v - prev_cv;
          if (eu % prev_s == 0 && ev % prev_s == 0 && abs(eu) <= prev_r * prev_s &&
              abs(ev) <= prev_r * prev_s)
            continue;
        }
        const __half* adesc = Da + (size_t)(v * Wa + u) * DIM;
        float amax;
        const float sc = dot_fast<DIM>(adesc, bt, &amax);
        const float sb = gamma * amax * bnorm1;
        bool take;
        if (sc - sb > best_f + best_b) {
          take = true;
        } else if (sc + sb <= best_f - best_b) {
          take = false;
        } else {  // near tie / non-finite: decide in exact arithmetic
          if (!best_known) {
            best_x = dot_exact(Da + (size_t)(best_v * Wa + best_u) * DIM, bdesc, DIM);
            best_known = true;
          }
          const double ex = dot_exact(adesc, bdesc, DIM);
          take = ex > best_x;
          if (take) {
            best_u = u;
            best_v = v;
            best_f = sc;
            best_b = sb;
            best_x = ex;
            continue;
          }
        }
        if (take) {
          best_u = u;
          best_v = v;
          best_f = sc;
          best_b = sb;
          best_known = false;
        }
      }
    }
    prev_cu = cu;
    prev_cv = cv;
    prev_s = s;
    prev_r = r;
  }
  return best_v * Wa + best_u;
}

// Generic-dimension refinement: exact FP64 scores throughout.
__device__ __noinline__ int refine_one_generic(const __half* __restrict__ Da, int Wa, int Ha, int dim,
                                  const __half* __restrict__ bdesc, int pa, const RefineLevels& L) {
  int best_u = pa % Wa, best_v = pa / Wa;
  for (int l = 0; l < L.n; ++l) {
    const int s = L.stride[l], r = L.radius[l];
    const int cu = best_u, cv = best_v;
    double best = dot_exact(Da + (size_t)(cv * Wa + cu) * dim, bdesc, dim);
    for (int dv = -r; dv <= r; ++dv)
      for (int du = -r; du <= r; ++du) {
        const int u = cu + du * s, v = cv + dv * s;
        if (u < 0 || v < 0 || u >= Wa || v >= Ha) continue;
        const double sc = dot_exact(Da + (size_t)(v * Wa + u) * dim, bdesc, dim);
        if (sc > best) {
          best = sc;
          best_u = u;
          best_v = v;
        }
      }
  }
  return best_v * Wa + best_u;
}

// Pruned refinement for 24-dim descriptors (the hot path).  Every candidate
// first costs one 8-dim head dot from the planar head array; by
// Cauchy-Schwarz its exact score is <= head + ||a_t|| ||b_t|| (+ rounding
// bounds), and when that cannot beat the current best (strict '>') the
// candidate is skipped exactly.  Otherwise the full fp32 dot is decided with
// a rigorous error bound, and near-ties in exact FP64 (as the reference).
struct ExactBest {
  float f;    // fp32 score
  float err;  // |f - exact| bound
};

__device__ __forceinline__ bool certainly_gt(float x, float ex, float y, float ey) {
  const float d = (x - ex) - (y + ey);
  return d > 4.0f * kU * (fabsf(x) + ex + fabsf(y) + ey);
}
__device__ __forceinline__ bool certainly_le(float x, float ex, float y, float ey) {
  const float d = (y - ey) - (x + ex);
  return d >= 4.0f * kU * (fabsf(x) + ex + fabsf(y) + ey);
}

// Running best of one refinement level (exact-argmax bookkeeping).
struct BestState {
  int u, v;
  float f, err;   // fp32 score and its rounding bound
  float thr;      // prune threshold: candidates with ub <= thr cannot win
  double x;       // exact score when known
  bool known;
};

__device__ __forceinline__ void best_set(BestState& B, int u, int v, float f, float err) {
  B.u = u;
  B.v = v;
  B.f = f;
  B.err = err;
  B.thr = (f - err) - 4.0f * kU * (fabsf(f) + err);
  B.known = false;
}

// Exact decision for a candidate whose full fp32 dot is within rounding of
// the running best (rare): FP64 replay of the reference's exact sums.
__device__ __noinline__ void refine_exact(const PairDev& P, const __half* __restrict__ bdesc, int u, int v, float sc,
                                          float err, BestState& B) {
  if (!B.known) {
    B.x = dot_exact(P.da + (size_t)(B.v * P.Wa + B.u) * 24, bdesc, 24);
    B.known = true;
  }
  const double ex = dot_exact(P.da + (size_t)(v * P.Wa + u) * 24, bdesc, 24);
  if (ex > B.x) {
    best_set(B, u, v, sc, err);
    B.x = ex;
    B.known = true;
  }
}

// Where the candidates' descriptors and norm bounds come from (global memory:
// standalone refine and the batched path's exact fallback).
struct GlobalAux {
  const uint4* rows;  // 3 uint4 per pixel
  const float4* norms;
  int W;
  __device__ __forceinline__ int at(int u, int v) const { return v * W + u; }
  __device__ __forceinline__ uint4 d0(int i) const { return __ldg(rows + 3 * i); }
  __device__ __forceinline__ uint4 d1(int i) const { return __ldg(rows + 3 * i + 1); }
  __device__ __forceinline__ uint4 d2(int i) const { return __ldg(rows + 3 * i + 2); }
  __device__ __forceinline__ float4 nrm(int i) const { return __ldg(norms + i); }
};
struct BConst {  // register-resident target descriptor and its bound constants
  uint4 b0, b1, b2;
  float c8, t8, c16, t16, c24;
};

// Full decision for one candidate that survived the 8-dim bound against the
// current best: 16-dim bound, then the full fp32 dot with its rounding bound,
// then (near tie) the exact FP64 replay.
template <class Aux>
__device__ __forceinline__ void refine_candidate(const PairDev& P, const Aux& X, const BConst& K,
                                                 const __half* __restrict__ bdesc, int u, int v, int i, float h8,
                                                 float4 nr, BestState& B) {
  const float h16 = dot8(X.d1(i), K.b1, h8);
  const float u16 = fmaf(nr.x, K.c16, fmaf(nr.y, K.t16, h16));
  if (fmaf(8.0f * kU, fabsf(h16) + fabsf(u16), u16) <= B.thr) return;
  const float sc = dot8(X.d2(i), K.b2, h16);
  const float err = K.c24 * nr.x;
  if (certainly_gt(sc, err, B.f, B.err)) {
    best_set(B, u, v, sc, err);
  } else if (!certainly_le(sc, err, B.f, B.err)) {
    refine_exact(P, bdesc, u, v, sc, err, B);
  }
}

__device__ __forceinline__ bool bound8_fails(float h8, float4 nr, const BConst& K, float thr) {
  const float u8 = fmaf(nr.x, K.c8, fmaf(nr.z, K.t8, h8));
  return fmaf(8.0f * kU, fabsf(h8) + fabsf(u8), u8) <= thr;  // cannot beat the best: skip
}

// One refinement level (camera.cpp:247-265) around (cu, cv), general form.
template <bool CHECK_PREV, class Aux>
__device__ __forceinline__ void refine_level(const PairDev& P, const Aux& X, const BConst& K,
                                             const __half* __restrict__ bdesc, int cu, int cv, int s, int r,
                                             int prev_cu, int prev_cv, int prev_s, int prev_r, BestState& B) {
  const int Wa = P.Wa, Ha = P.Ha;
  const int du_lo = -min(r, cu / s), du_hi = min(r, (Wa - 1 - cu) / s);
  const int dv_lo = -min(r, cv / s), dv_hi = min(r, (Ha - 1 - cv) / s);
  const int lim = prev_r * prev_s;
  for (int dv = dv_lo; dv <= dv_hi; ++dv) {
    const int v = cv + dv * s;
    for (int du = du_lo; du <= du_hi; ++du) {
      if (du == 0 && dv == 0) continue;
      const int u = cu + du * s;
      if (CHECK_PREV) {  // already maximised by the previous level: cannot win (strict '>')
        const int eu = u - prev_cu, ev = v - prev_cv;
        if (abs(eu) <= lim && abs(ev) <= lim && (prev_s == 1 || (eu % prev_s == 0 && ev % prev_s == 0))) continue;
      }
      const int i = X.at(u, v);
      const float4 nr = X.nrm(i);
      const float h8 = dot8(X.d0(i), K.b0, 0.0f);
      if (bound8_fails(h8, nr, K, B.thr)) continue;
      refine_candidate(P, X, K, bdesc, u, v, i, h8, nr, B);
    }
  }
}

template <class Aux>
__device__ __forceinline__ int refine_pruned(const PairDev& P, const Aux& X, int pa, const __half* __restrict__ bdesc,
                                             const RefineLevels& L) {
  const int Wa = P.Wa;
  BConst K;
  {
    const uint4* bp = reinterpret_cast<const uint4*>(bdesc);
    K.b0 = __ldg(bp);
    K.b1 = __ldg(bp + 1);
    K.b2 = __ldg(bp + 2);
    const float s0 = dot8(K.b0, K.b0, 0.0f), s1 = dot8(K.b1, K.b1, 0.0f), s2 = dot8(K.b2, K.b2, 0.0f);
    // Three-stage Cauchy-Schwarz pruning: after the first 8 (16) dims,
    //   exact(cand) <= partial + k u ||a|| ||b_head|| + ||a_tail|| ||b_tail||
    K.c8 = 8.01f * kU * norm_ub(s0, 8);
    K.t8 = norm_ub(s1 + s2, 16) * (1.0f + 4.0f * kU);
    K.c16 = 16.01f * kU * norm_ub(s0 + s1, 16);
    K.t16 = norm_ub(s2, 8) * (1.0f + 4.0f * kU);
    K.c24 = 24.01f * kU * norm_ub(s0 + s1 + s2, 24);
  }
  int cu = pa % Wa, cv = pa / Wa;
  int prev_cu = 0, prev_cv = 0, prev_s = 1, prev_r = -1;
  for (int l = 0; l < L.n; ++l) {
    const int s = L.stride[l], r = L.radius[l];
    if (l > 0 && s == prev_s && r == prev_r && cu == prev_cu && cv == prev_cv) continue;
    BestState B;
    {
      const int i = X.at(cu, cv);
      const float f = dot8(X.d2(i), K.b2, dot8(X.d1(i), K.b1, dot8(X.d0(i), K.b0, 0.0f)));
      best_set(B, cu, cv, f, K.c24 * X.nrm(i).x);
      B.x = 0.0;
    }
    if (prev_r < 0) {
      refine_level<false>(P, X, K, bdesc, cu, cv, s, r, 0, 0, 1, -1, B);
    } else {
      refine_level<true>(P, X, K, bdesc, cu, cv, s, r, prev_cu, prev_cv, prev_s, prev_r, B);
    }
    prev_cu = cu;
    prev_cv = cv;
    prev_s = s;
    prev_r = r;
    cu = B.u;
    cv = B.v;
  }
  return cv * Wa + cu;
}

__device__ __forceinline__ int refine_dispatch(const PairDev& P, int pa, int pb, const RefineLevels& L) {
  const __half* bdesc = P.db + (size_t)pb * P.dim;
  if (((uintptr_t)P.da | (uintptr_t)P.db) & 15)  // vector loads need 16-byte rows
    return refine_one_generic(P.da, P.Wa, P.Ha, P.dim, bdesc, pa, L);
  if (P.dnorm && P.dim == 24)
    return refine_pruned(P, GlobalAux{reinterpret_cast<const uint4*>(P.da), P.dnorm, P.Wa}, pa, bdesc, L);
  if (P.dim == 24) return refine_one<24>(P.da, P.Wa, P.Ha, bdesc, pa, L);
  if (P.dim == 16) return refine_one<16>(P.da, P.Wa, P.Ha, bdesc, pa, L);
  if (P.dim == 32) return refine_one<32>(P.da, P.Wa, P.Ha, bdesc, pa, L);
  return refine_one_generic(P.da, P.Wa, P.Ha, P.dim, bdesc, pa, L);
}

// ---------------------------------------------------------------- K3 + K4
// One thread per b-pixel, 32x8 pixel tiles, blockIdx.y = pair.
// match_pointmaps for b-pixel n (camera.cpp:213-236): LM from the seed,
// lround + clamp, validity, q.  Writes the outputs; returns (pa, valid).
// (u, v): the b-pixel's column / row (n = v W_b + u).  Returns {pixel_a,
// valid, column, row of pixel_a} (pixel_a = -1: skipped pixel).
// Post-LM loads of the refinement (PMX_ROW_WITH_GATHERS): the target
// descriptor row and the pair's int8 statistics, fetched with the pixel_a
// gathers (one round trip).
struct RowLoads {
  uint4 d0, d1, d2;
  int qbad, a1max;
};

template <class JT = JReg, bool ROW = false>
__device__ __forceinline__ int4 match_pixel(const PairDev& P, const LMParams& lp, int n, int u, int v, JT J = JT(),
                                            RowLoads* rl = nullptr) {
  if (P.out_pb) P.out_pb[n] = n;
  int32_t pa_out = -1;
  float q_out = 0.0f;
  uint8_t valid_out = 0;
  int cu = 0, cv = 0;
#if PMX_PRELOAD_SEED && PMX_LM_F32 && PMX_EAGER_F32
  // identity seed (camera.cpp:221): its ray-map supports are loaded together
  // with X_b instead of after it (same indices / values as the LM's own load)
  Corners pre;
  const bool have_pre = !P.seed_last && P.Wa == P.Wb && P.Ha >= 1;
  if (have_pre) corners_load(P.rays, P.Wa, P.Ha, (double)u, (double)min(v, P.Ha - 1), pre);
#endif
  const bool vb = P.vb ? P.vb[n] != 0 : true;
  const double x0 = P.xb[3 * n], x1 = P.xb[3 * n + 1], x2 = P.xb[3 * n + 2];
  // camera.cpp:217-219 (norm < 1e-12 skips; a NaN norm does not), as |x|^2 < 1e-24
  const double xx = x0 * x0 + x1 * x1 + x2 * x2;
  if (vb && !(xx < 1e-24)) {
    // seed = pixel n of the a-grid (camera.cpp:221), or the init match
    int su = u, sv = v;
    if (P.Wa != P.Wb) {
      su = n % P.Wa;
      sv = n / P.Wa;
    }
    if (P.seed_last) {
      const int k = P.seed_last[n];
      if (k >= 0) {
        const int s = P.init_pa[k];
        if (s >= 0) {
          su = s % P.Wa;
          sv = s / P.Wa;
        }
      }
    }
#if PMX_PRELOAD_SEED && PMX_LM_F32 && PMX_EAGER_F32
    const ProjOut pr =
        iterative_project_dev(P.rays, P.Wa, P.Ha, x0, x1, x2, (double)su, (double)sv, lp, J, have_pre ? &pre : nullptr);
#else
    // the seed clamped in integers (camera.cpp:124-125 on an integer seed)
    const int csu = min(max(su, 0), P.Wa - 1), csv = min(max(sv, 0), P.Ha - 1);
    const ProjOut pr =
        iterative_project_dev<JT, true>(P.rays, P.Wa, P.Ha, x0, x1, x2, (double)csu, (double)csv, lp, J);
#endif
    cu = min(max((int)round(pr.pu), 0), P.Wa - 1);  // std::lround: half away from zero
    cv = min(max((int)round(pr.pv), 0), P.Ha - 1);
    int pa = cv * P.Wa + cu;
    PMX_CHECK_INDEX(pa, P.Wa * P.Ha);
    // every gather of pa issued at once (one round trip, not one per test)
    const uint8_t vpa = P.va ? __ldg(P.va + pa) : (uint8_t)1;
    const float a0f = __ldg(P.xa + 3 * pa), a1f = __ldg(P.xa + 3 * pa + 1), a2f = __ldg(P.xa + 3 * pa + 2);
    const float qpa = __ldg(P.qa + pa), qn = __ldg(P.qb + n);
    const double thr = P.sel->threshold;
    if (ROW) {
      const uint4* row = reinterpret_cast<const uint4*>(P.db) + 3 * (size_t)n;
      rl->d0 = __ldg(row);
      rl->d1 = __ldg(row + 1);
      rl->d2 = __ldg(row + 2);
      rl->qbad = __ldg(&P.sel->qbad);
      rl->a1max = __ldg(&P.sel->a1max);
    }
    bool valid = pr.converged && vpa != 0;
    if (valid) {
      const double e0 = (double)a0f - x0, e1 = (double)a1f - x1, e2 = (double)a2f - x2;
      const double dist = sqrt(e0 * e0 + e1 * e1 + e2 * e2);
      if (dist > thr) valid = false;
    }
    pa_out = pa;
    q_out = (float)sqrt((double)qpa * (double)qn);
    valid_out = valid ? 1 : 0;
  }
  P.out_pa[n] = pa_out;
  P.out_q[n] = q_out;
  P.out_valid[n] = valid_out;
  return make_int4(pa_out, valid_out, cu, cv);
}

// One thread per b-pixel, 32x8 pixel tiles, blockIdx.y = pair (no refinement).
__global__ void __launch_bounds__(256, 3) k_match(const PairDev* __restrict__ pairs, LMParams lp) {
  const PairDev& P = pairs[blockIdx.z];
  const int u = blockIdx.x * 32 + (threadIdx.x & 31), v = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (u >= P.Wb || v >= P.Hb) return;
  match_pixel(P, lp, v * P.Wb + u, u, v);
}

// K4: feature_refine of the valid matches just written by k_match, in place.
//
// One thread per b-pixel, 32x8 tiles.  k_prep wrote the int8 image q8(a) =
// rne(127 a) of every a-descriptor (24 B/pixel, L2-resident per chunk); the
// windows of a tile overlap, so candidates are read through L1 (an earlier
// shared-memory staging variant with cp.async double buffering was slower:
// its per-tile box reduction and barriers cost more than the L1 misses).
// Every window candidate gets an exact integer score q_c = q8(a_c) . q8(b)
// (6 DP4A).
// With q8(x) = 127 x + e, |e| <= 1/2, the exact score satisfies
//   |127^2 (a_c . b) - q_c| <= E = 0.5 (sum|q8(a)| + sum|q8(b)|) + 6,
// so if the best integer score beats the second best by more than 2E, its
// candidate is the unique exact argmax, whatever the scan order and the tie
// rule.  Otherwise (true near-ties; never on well-separated peaks) the pixel
// is refined by the exact scalar path (refine_dispatch: fp32 + FP64 replay),
// so the result always equals the reference's exact-arithmetic argmax
// (camera.cpp:247-265: strict '>', centre first, raster order).
//
// A later level whose centre moved only needs the candidates outside the
// previous window (those were all strictly below the moved-to centre); a level
// whose window is unchanged is skipped (camera.cpp semantics, strict '>').
struct QB {  // register-resident int8 target descriptor
  uint32_t w[6];  // dims 0-3, 4-7 (head), 8-11, 12-15, 16-19, 20-23 (tail)
  int nt;         // ceil(sqrt(sum of squares of the tail))
};

// Head (dims 0-7) and tail (dims 8-23) partial scores of one candidate.
__device__ __forceinline__ int qdot_head(const uint2 h, const QB& B) {
  return __dp4a((int)h.y, (int)B.w[1], __dp4a((int)h.x, (int)B.w[0], 0));
}
__device__ __forceinline__ int qdot_tail(const uint4 t, const QB& B, int s) {
  s = __dp4a((int)t.x, (int)B.w[2], s);
  s = __dp4a((int)t.y, (int)B.w[3], s);
  s = __dp4a((int)t.z, (int)B.w[4], s);
  return __dp4a((int)t.w, (int)B.w[5], s);
}

// Best and second-best candidate of a scan as packed keys score * 256 + rank
// (|score| <= 24 * 127^2 < 2^19, rank < 256): one max/min pair per candidate.
struct Top2 {
  int b1, b2;
  __device__ __forceinline__ int score1() const { return b1 >> 8; }
  __device__ __forceinline__ int rank1() const { return b1 & 255; }
  // unique exact argmax: the best beats the second by more than 2E
  __device__ __forceinline__ bool decided(int tgap) const { return (b1 >> 8) - (b2 >> 8) > tgap; }
};
__device__ __forceinline__ int qkey(int s, int k) { return s * 256 + k; }
__device__ __forceinline__ void top2_add(Top2& T, int key) {
  T.b2 = max(T.b2, min(T.b1, key));
  T.b1 = max(T.b1, key);
}

// The int8 a-image read in place from the (L2-resident) chunk scratch
// through the L1 cache: no staging, no block barriers.
struct QGlob {
  const uint2* __restrict__ h;     // dims 0-7 (see PairDev::q8h)
  const uint16_t* __restrict__ n;  // tail bound
  const uint4* __restrict__ t;     // dims 8-23
  int bw;                          // row pitch (= W)
  int hw;                          // pixels of the a-image (checked builds)
  __device__ __forceinline__ int at(int u, int v) const { return v * bw + u; }
  __device__ __forceinline__ uint2 head(int i) const {
    PMX_CHECK_INDEX(i, hw);
    return __ldg(h + i);
  }
  __device__ __forceinline__ int nt(int i) const {
    PMX_CHECK_INDEX(i, hw);
    return (int)__ldg(n + i);
  }
  __device__ __forceinline__ uint4 tail(int i) const {
    PMX_CHECK_INDEX(i, hw);
    return __ldg(t + i);
  }
  __device__ __forceinline__ int score(int i, const QB& B) const { return qdot_tail(tail(i), B, qdot_head(head(i), B)); }
};

// First level, compile-time radius / stride, window inside the image,
// unrolled (immediate load offsets).  The centre is scored first; every other
// candidate costs its 8-dim head score plus the Cauchy-Schwarz bound of its
// tail, |tail . b_tail| <= nt_a nt_b, and is skipped when even that upper
// bound stays at or below best - tgap - 1: it can then neither become the
// argmax nor come within the uniqueness gap of the final best (which is >=
// the running best), so skipping it leaves the decision exact.  Survivors
// (the true peak, near ties) get the full score (4 more DP4A).
template <int R, int S, class Tile>
__device__ __forceinline__ Top2 q_level1(const Tile& T, const QB& B, int cu, int cv, int tgap) {
  constexpr int D = 2 * R + 1, C = R * D + R;
  const int base = T.at(cu - R * S, cv - R * S);
  Top2 t{qkey(T.score(base + R * S * T.bw + R * S, B), C), INT_MIN};
  int thr = t.score1() - tgap - 1;
#pragma unroll
  for (int dv = 0; dv < D; ++dv) {
#pragma unroll
    for (int du = 0; du < D; ++du) {
      if (dv * D + du == C) continue;
      const int i = base + dv * S * T.bw + du * S;
      const int s8 = qdot_head(T.head(i), B);
      if (!PMX_PRUNE || s8 + T.nt(i) * B.nt > thr) {
        top2_add(t, qkey(qdot_tail(T.tail(i), B, s8), dv * D + du));
        thr = t.score1() - tgap - 1;
      }
    }
  }
  return t;
}

// 256-bit read-only load of two consecutive tails (dims 8-23 of pixels i, i+1; 32-B aligned).
__device__ __forceinline__ void ld_tail2(const uint4* p, uint4& a, uint4& b) {
  unsigned long long x, y, z, w;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(x), "=l"(y), "=l"(z), "=l"(w) : "l"(p));
  a = make_uint4((uint32_t)x, (uint32_t)(x >> 32), (uint32_t)y, (uint32_t)(y >> 32));
  b = make_uint4((uint32_t)z, (uint32_t)(z >> 32), (uint32_t)w, (uint32_t)(w >> 32));
}

// First level, stride 1, as q_level1<R, 1> but each window row is read as
// the R + 1 aligned pixel pairs (e, e + 1), e = row start & ~1, that cover
// it: one 16-byte head load and one 32-byte tail load per two candidates.
// Neighbouring lanes' windows start one pixel apart, so two lanes share
// every pair and the warp moves ~half the L1 bytes of per-candidate loads.
// The slot outside the window (first or last of the 2R + 2) is masked; the
// centre is scored in its row.  Same top-2 as q_level1 (keys are
// order-independent).  Needs 16-B aligned heads and 32-B aligned tails; the
// last pair may reach one pixel past the image (the chunk scratch continues
// there: q8t is followed by q8h, q8h by q8n).
template <int R, class Tile>
__device__ __forceinline__ Top2 q_level1_pairs(const Tile& T, const QB& B, int cu, int cv) {
  constexpr int D = 2 * R + 1;
  const int s0 = T.at(cu - R, cv - R);
  Top2 t{INT_MIN, INT_MIN};
#pragma unroll
  for (int dv = 0; dv < D; ++dv) {
    const int rs = s0 + dv * T.bw;  // window row start
    const int e = rs & ~1;
    const int sh = rs - e;  // 0 or 1: slot k of the row is window column k - sh
    PMX_CHECK_INDEX(e, T.hw);
    PMX_CHECK_INDEX(e + 2 * R + 1, T.hw + 1);
    const uint4* hp = reinterpret_cast<const uint4*>(T.h + e);
    const uint4* tp = T.t + e;
#pragma unroll
    for (int j = 0; j <= R; ++j) {
      const uint4 h2 = __ldg(hp + j);
      uint4 ta, tb;
      ld_tail2(tp + 2 * j, ta, tb);
      const int sa = qdot_tail(ta, B, qdot_head(make_uint2(h2.x, h2.y), B));
      const int sb = qdot_tail(tb, B, qdot_head(make_uint2(h2.z, h2.w), B));
      const int ka = 2 * j - sh, kb = 2 * j + 1 - sh;
      top2_add(t, ka >= 0 ? qkey(sa, dv * D + ka) : INT_MIN);
      top2_add(t, kb < D ? qkey(sb, dv * D + kb) : INT_MIN);
    }
  }
  return t;
}

// One level at run-time radius / stride for one lane (border windows and
// uncommon level shapes).  Candidates of the previous window (pr >= 0) are
// skipped; the centre enters with score `centre` (its rank r*D+r).
template <class Tile>
__device__ __forceinline__ Top2 q_level_lane(const Tile& T, const QB& B, int cu, int cv, int s, int r, int Wa,
                                             int Ha, int centre, int pcu, int pcv, int ps, int pr) {
  const int D = 2 * r + 1;
  Top2 t{qkey(centre, r * D + r), INT_MIN};
  const int lim = pr * ps;
  for (int dv = -r; dv <= r; ++dv) {
    const int v = cv + dv * s;
    if (v < 0 || v >= Ha) continue;
    for (int du = -r; du <= r; ++du) {
      const int u = cu + du * s;
      if (u < 0 || u >= Wa || (du == 0 && dv == 0)) continue;
      if (pr >= 0) {
        const int eu = u - pcu, ev = v - pcv;
        if (abs(eu) <= lim && abs(ev) <= lim && (ps == 1 || (eu % ps == 0 && ev % ps == 0))) continue;
      }
      top2_add(t, qkey(T.score(T.at(u, v), B), (dv + r) * D + (du + r)));
    }
  }
  return t;
}

// Refinement state of one lane between levels.
struct QState {
  int cu, cv;         // current centre
  int pcu, pcv, ps, pr;  // previous window (pr < 0: none)
  int best;           // integer score of the centre
  int st;             // 0 active, 1 undecided (exact path), 2 no pixel
};

// Level l of one lane from its top-2: move the centre, or mark undecided.
__device__ __forceinline__ void q_advance(QState& q, const Top2& t, int tgap, int s, int r) {
  if (!t.decided(tgap)) {
    q.st = 1;
    return;
  }
  const int D = 2 * r + 1, k = t.rank1();
  q.pcu = q.cu;
  q.pcv = q.cv;
  q.ps = s;
  q.pr = r;
  if (r == 3) {  // BASELINE's window: division by a constant
    const int kv = k / 7;
    q.cu += (k - 7 * kv - 3) * s;
    q.cv += (kv - 3) * s;
  } else {
    const int kv = k / D;
    q.cu += (k - D * kv - r) * s;
    q.cv += (kv - r) * s;
  }
  q.best = t.score1();
}

// All levels of the warp's 32 pixels.  Interior first-level windows of the
// common shapes run per lane, unrolled; every other window (border windows,
// a later level that only some lanes need because their centre moved:
// BASELINE's second level) is evaluated by the whole warp, one such pixel at
// a time, lanes spread over its window - or per lane when more than 8 lanes
// need one.
template <class Tile>
__device__ __forceinline__ void q_refine_warp(const Tile& T, const QB& B, int tgap, int Wa, int Ha,
                                              const RefineLevels& L, QState& q) {
  const int lane = threadIdx.x & 31;
  const bool pair_aligned = ((uintptr_t)T.h & 15) == 0 && ((uintptr_t)T.t & 31) == 0;
  for (int l = 0; l < L.n; ++l) {
    // compile-time indices: the levels stay in the kernel's parameter bank
    // (a dynamic index would copy them to local memory in every thread)
    int s = L.stride[0], r = L.radius[0];
#pragma unroll
    for (int k = 1; k < PMX_MAX_REFINE_LEVELS; ++k)
      if (l == k) {
        s = L.stride[k];
        r = L.radius[k];
      }
    const bool same = q.pr >= 0 && s == q.ps && r == q.pr && q.cu == q.pcu && q.cv == q.pcv;  // identical window
    const bool need = q.st == 0 && !same;
    if (!__any_sync(0xffffffffu, need)) continue;
    // Interior first-level windows of the common shapes: unrolled, per lane.
    const bool interior = q.pr < 0 && q.cu - r * s >= 0 && q.cu + r * s < Wa && q.cv - r * s >= 0 &&
                          q.cv + r * s < Ha;
    const bool fixed = need && interior && ((s == 1 && r == 3) || (s == 2 && r == 2));
    if (__any_sync(0xffffffffu, fixed) && fixed) {
      Top2 t;
      if (s == 1) {
#if PMX_PAIRLD
        if (pair_aligned)
          t = q_level1_pairs<3, Tile>(T, B, q.cu, q.cv);
        else
#endif
          t = q_level1<3, 1, Tile>(T, B, q.cu, q.cv, tgap);
      } else {
        t = q_level1<2, 2, Tile>(T, B, q.cu, q.cv, tgap);
      }
      q_advance(q, t, tgap, s, r);
    }
    // The rest - border windows, moved centres of later levels, uncommon
    // shapes: per lane when many, else by the whole warp one pixel at a time
    // (a warp with one border lane no longer runs the generic window loop
    // for it while 31 lanes wait).
    const unsigned m = __ballot_sync(0xffffffffu, need && !fixed);
    if (!m) continue;
    if (__popc(m) > 8) {  // per lane
      if (need && !fixed) {
        if (q.best == INT_MIN) q.best = T.score(T.at(q.cu, q.cv), B);
        const Top2 t = q_level_lane(T, B, q.cu, q.cv, s, r, Wa, Ha, q.best, q.pcu, q.pcv, q.ps, q.pr);
        q_advance(q, t, tgap, s, r);
      }
    } else {  // warp-cooperative, one pending pixel at a time
      const int D = 2 * r + 1, nc = D * D, lim0 = r * D + r;
      for (unsigned mm = m; mm; mm &= mm - 1) {
        const int src = __ffs(mm) - 1;
        const int cu = __shfl_sync(0xffffffffu, q.cu, src), cv = __shfl_sync(0xffffffffu, q.cv, src);
        const int pcu = __shfl_sync(0xffffffffu, q.pcu, src), pcv = __shfl_sync(0xffffffffu, q.pcv, src);
        const int ps = __shfl_sync(0xffffffffu, q.ps, src), pr = __shfl_sync(0xffffffffu, q.pr, src);
        const int centre = __shfl_sync(0xffffffffu, q.best, src);
        const bool have_centre = centre != INT_MIN;  // not yet scored on a first-level border window
        QB Bs;
#pragma unroll
        for (int w = 0; w < 6; ++w) Bs.w[w] = __shfl_sync(0xffffffffu, B.w[w], src);
#if PMX_PRUNE
        Bs.nt = __shfl_sync(0xffffffffu, B.nt, src);
#else
        Bs.nt = 0;
#endif
        Top2 t{lane == 0 && have_centre ? qkey(centre, lim0) : INT_MIN, INT_MIN};
        const int lim = pr * ps;
        for (int k = lane; k < nc; k += 32) {
          const int kv = r == 3 ? k / 7 : k / D;  // BASELINE's window: a constant divisor
          const int dv = kv - r, du = k - D * kv - r;
          const int u = cu + du * s, v = cv + dv * s;
          if (u < 0 || u >= Wa || v < 0 || v >= Ha || (du == 0 && dv == 0 && have_centre)) continue;
          const int eu = u - pcu, ev = v - pcv;
          if (pr >= 0 && abs(eu) <= lim && abs(ev) <= lim && (ps == 1 || (eu % ps == 0 && ev % ps == 0))) continue;
          top2_add(t, qkey(T.score(T.at(u, v), Bs), k));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // merge the top-2 keys over the warp
          const int ob1 = __shfl_xor_sync(0xffffffffu, t.b1, o);
          const int ob2 = __shfl_xor_sync(0xffffffffu, t.b2, o);
          t.b2 = max(max(t.b2, ob2), min(t.b1, ob1));
          t.b1 = max(t.b1, ob1);
        }
        if (lane == src) q_advance(q, t, tgap, s, r);
      }
    }
  }
}

// Undecided pixels (near ties, unstageable tiles, no int8 image): the
// per-thread exact refinement, kept out of line (rare).
__device__ __noinline__ int refine_exact_path(const PairDev& P, int pa, int n, const RefineLevels L) {
  return refine_dispatch(P, pa, n, L);
}

// K3 + K4 fused: one thread per b-pixel of a 32 x PMX_MR_TY tile (blockIdx.x = tile,
// blockIdx.y = pair) runs the LM, then (warp-collectively) the refinement of
// the valid matches; the int8 a-image (L2-resident chunk scratch) is read
// through L1, where a tile's windows overlap.  Fusing lets the FP64-bound LM
// of some warps overlap the integer-bound refinement of others on every SM.
#ifndef PMX_MR_BLOCKS
#define PMX_MR_BLOCKS 8  // resident CTAs per SM (64 registers at 128 threads)
#endif
#ifndef PMX_MR_TY
#define PMX_MR_TY 4  // tile rows: 32 x PMX_MR_TY b-pixels per CTA (32x4 at 8 CTAs/SM: 1.363 -> 1.347 ms against 32x8 at 4; 32x2 at 16: 1.396)
#endif
__global__ void __launch_bounds__(32 * PMX_MR_TY, PMX_MR_BLOCKS) k_match_refine(const PairDev* __restrict__ pairs, LMParams lp,
                                                         RefineLevels L, unsigned long long* __restrict__ exact_px) {
  const PairDev& P = pairs[blockIdx.z];
  if ((int)blockIdx.x * 32 >= P.Wb || (int)blockIdx.y * PMX_MR_TY >= P.Hb) return;
  const int u = blockIdx.x * 32 + (threadIdx.x & 31), v = blockIdx.y * PMX_MR_TY + (threadIdx.x >> 5);
  const int m = v * P.Wb + u;
  int n = -1, pa = 0, pcu = 0, pcv = 0;
#if PMX_ROW_WITH_GATHERS
  RowLoads rl{};
  rl.qbad = 1;  // pixels outside the image: no fast path
#endif
#if PMX_PREFETCH
  // the descriptor row quantized after the LM: its HBM latency overlaps the LM
  if (u < P.Wb && v < P.Hb && P.q8h != nullptr)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(P.db) + 48 * (size_t)m));
#endif
  if (u < P.Wb && v < P.Hb) {
#if PMX_J_SMEM && PMX_LM_F32
    __shared__ float sJ[6 * 32 * PMX_MR_TY];
    const int4 r = match_pixel(P, lp, m, u, v, JSm<32 * PMX_MR_TY>{sJ + threadIdx.x});
#elif PMX_ROW_WITH_GATHERS
    const int4 r = match_pixel<JReg, true>(P, lp, m, u, v, JReg(), &rl);
#else
    const int4 r = match_pixel(P, lp, m, u, v);
#endif
    pa = r.x;
    pcu = r.z;
    pcv = r.w;
    if (r.y) n = m;
  }
#if PMX_ROW_WITH_GATHERS
  const bool fast_pair = P.q8h != nullptr && rl.qbad == 0;
#else
  const bool fast_pair = P.q8h != nullptr && P.sel->qbad == 0;
#endif
  QB B;
  int tgap = 0;
  bool fast = n >= 0 && fast_pair;
  if (fast) {
#if PMX_ROW_WITH_GATHERS
    const Q8 q = quantize24(rl.d0, rl.d1, rl.d2);
#else
    const uint4* row = reinterpret_cast<const uint4*>(P.db) + 3 * (size_t)n;
    const Q8 q = quantize24(__ldg(row), __ldg(row + 1), __ldg(row + 2));
#endif
    B.w[0] = q.a.x;
    B.w[1] = q.a.y;
    B.w[2] = q.a.z;
    B.w[3] = q.a.w;
    B.w[4] = q.b.x;
    B.w[5] = q.b.y;
    B.nt = q.nt;
#if PMX_ROW_WITH_GATHERS
    tgap = rl.a1max + q.l1 + 12;  // 2E, E = (sum|q8(a)| + sum|q8(b)|) / 2 + 6
#else
    tgap = P.sel->a1max + q.l1 + 12;  // 2E, E = (sum|q8(a)| + sum|q8(b)|) / 2 + 6
#endif
    fast = !q.bad;
  }
  QState q{pcu, pcv, 0, 0, 1, -1, INT_MIN, n < 0 ? 2 : fast ? 0 : 1};
  if (__any_sync(0xffffffffu, fast)) {
    const QGlob T{P.q8h, P.q8n, P.q8t, P.Wa, P.Wa * P.Ha};
    q_refine_warp(T, B, tgap, P.Wa, P.Ha, L, q);
  }
  if (exact_px) {
    const unsigned c = __popc(__ballot_sync(0xffffffffu, q.st == 1));
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(exact_px, (unsigned long long)c);
  }
  if (q.st != 2) {
    int out = q.st == 0 ? q.cv * P.Wa + q.cu : refine_exact_path(P, pa, n, L);
    PMX_CHECK_INDEX(out, P.Wa * P.Ha);
    if (out != pa) {
      P.out_pa[n] = out;
      P.out_q[n] = (float)sqrt((double)__ldg(P.qa + out) * (double)__ldg(P.qb + n));
    }
  }
}

// PMX_SPLIT: the refinement as its own kernel after k_match (each phase with
// its own register budget / occupancy; the fused kernel overlaps them).
#ifndef PMX_RF_TY
#define PMX_RF_TY 4
#endif
#ifndef PMX_RF_BLOCKS
#define PMX_RF_BLOCKS 8  // 64 registers (12 / 16: 40 / 32 registers, heavy spills)
#endif
__global__ void __launch_bounds__(32 * PMX_RF_TY, PMX_RF_BLOCKS) k_refine_tiles(const PairDev* __restrict__ pairs,
                                                                              RefineLevels L) {
  const PairDev& P = pairs[blockIdx.z];
  if ((int)blockIdx.x * 32 >= P.Wb || (int)blockIdx.y * PMX_RF_TY >= P.Hb) return;
  const int u = blockIdx.x * 32 + (threadIdx.x & 31), v = blockIdx.y * PMX_RF_TY + (threadIdx.x >> 5);
  const int m = v * P.Wb + u;
  int n = -1, pa = 0, pcu = 0, pcv = 0;
  if (u < P.Wb && v < P.Hb && P.out_valid[m]) {
    pa = P.out_pa[m];
    pcu = pa % P.Wa;
    pcv = pa / P.Wa;
    n = m;
  }
  const bool fast_pair = P.q8h != nullptr && __ldg(&P.sel->qbad) == 0;
  QB B;
  int tgap = 0;
  bool fast = n >= 0 && fast_pair;
  if (fast) {
    const uint4* row = reinterpret_cast<const uint4*>(P.db) + 3 * (size_t)n;
    const Q8 q = quantize24(__ldg(row), __ldg(row + 1), __ldg(row + 2));
    B.w[0] = q.a.x;
    B.w[1] = q.a.y;
    B.w[2] = q.a.z;
    B.w[3] = q.a.w;
    B.w[4] = q.b.x;
    B.w[5] = q.b.y;
    B.nt = q.nt;
    tgap = __ldg(&P.sel->a1max) + q.l1 + 12;
    fast = !q.bad;
  }
  QState q{pcu, pcv, 0, 0, 1, -1, INT_MIN, n < 0 ? 2 : fast ? 0 : 1};
  if (__any_sync(0xffffffffu, fast)) {
    const QGlob T{P.q8h, P.q8n, P.q8t, P.Wa, P.Wa * P.Ha};
    q_refine_warp(T, B, tgap, P.Wa, P.Ha, L, q);
  }
  if (q.st != 2) {
    int out = q.st == 0 ? q.cv * P.Wa + q.cu : refine_exact_path(P, pa, n, L);
    PMX_CHECK_INDEX(out, P.Wa * P.Ha);
    if (out != pa) {
      P.out_pa[n] = out;
      P.out_q[n] = (float)sqrt((double)__ldg(P.qa + out) * (double)__ldg(P.qb + n));
    }
  }
}

// Standalone feature_refine over an arbitrary MatchSet (camera.cpp:239-271).
__global__ void __launch_bounds__(256) k_refine(PairDev P, int64_t count, const int32_t* __restrict__ in_pa,
                                                const int32_t* __restrict__ in_pb,
                                                const float* __restrict__ in_q,
                                                const uint8_t* __restrict__ in_valid, RefineLevels L,
                                                int32_t* out_pa, int32_t* out_pb, float* out_q,
                                                uint8_t* out_valid) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  int pa = in_pa[k];
  const int pb = in_pb ? in_pb[k] : (int)k;
  float q = in_q ? in_q[k] : 0.0f;
  const uint8_t valid = in_valid ? in_valid[k] : 1;
  if (valid && pa >= 0 && pb >= 0 && pa < P.Ha * P.Wa && pb < P.Hb * P.Wb) {
    pa = refine_dispatch(P, pa, pb, L);
    q = (float)sqrt((double)P.qa[pa] * (double)P.qb[pb]);
  }
  out_pa[k] = pa;
  if (out_pb) out_pb[k] = pb;
  out_q[k] = q;
  out_valid[k] = valid;
}

// Seed map: last valid init match per pixel_b (camera.cpp:202-210, last write wins).
__global__ void k_seed_scatter(int64_t m, const int32_t* __restrict__ pb, const uint8_t* __restrict__ valid,
                               int HWb, int32_t* __restrict__ last) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int b = pb ? pb[k] : (int)k;
  if ((valid ? valid[k] : 1) && b >= 0 && b < HWb) atomicMax(&last[b], (int32_t)k);
}

__global__ void k_project_points(const double4* __restrict__ rays, int W, int H, int64_t n,
                                 const float* __restrict__ x, const double* __restrict__ p0, LMParams lp,
                                 double* pix, uint8_t* conv, int32_t* iters) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const ProjOut r = iterative_project_dev(rays, W, H, x[3 * k], x[3 * k + 1], x[3 * k + 2], p0[2 * k],
                                          p0[2 * k + 1], lp);
  pix[2 * k] = r.pu;
  pix[2 * k + 1] = r.pv;
  conv[k] = r.converged ? 1 : 0;
  iters[k] = r.iterations;
}

__global__ void k_rays_out(const double4* __restrict__ rays, int HW, double* out_rays, double* out_dist,
                           uint8_t* out_valid, const float* __restrict__ xyz) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= HW) return;
  double4 r = rays[i];
  if (r.w == 0.0) r = make_double4(0.0, 0.0, 1.0, 0.0);  // camera.cpp: invalid pixels keep (0, 0, 1)
  out_rays[3 * i] = r.x;
  out_rays[3 * i + 1] = r.y;
  out_rays[3 * i + 2] = r.z;
  out_valid[i] = r.w != 0.0 ? 1 : 0;
  if (r.w != 0.0) {
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    out_dist[i] = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
  } else {
    out_dist[i] = 1.0;
  }
}

// accept_loop_edge's descriptor-agreement gate (retrieval.cpp:238-244): a
// valid match stays valid only if the exact dot of its endpoints'
// descriptors is >= 0.5 (unit-norm descriptors; FP64 sum of the exact fp16
// products, as the reference's double dot).  Counts the surviving matches
// of every pair (valid_fraction, camera.cpp:16-19).
__global__ void __launch_bounds__(256) k_loop_gate(const PairDev* __restrict__ pairs, double min_agreement,
                                                   unsigned long long* __restrict__ valid_count) {
  const PairDev& P = pairs[blockIdx.y];
  const int hwb = P.Hb * P.Wb;
  int cnt = 0;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < hwb; n += gridDim.x * blockDim.x) {
    if (!P.out_valid[n]) continue;
    const int pa = P.out_pa[n];
    const double d = dot_exact(P.da + (size_t)pa * P.dim, P.db + (size_t)n * P.dim, P.dim);
    if (d < min_agreement)
      P.out_valid[n] = 0;
    else
      ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(valid_count + blockIdx.y, (unsigned long long)cnt);
}

// Host path: copies of the small per-pair inputs (valid masks, confidences)
// from pinned, device-mapped host memory, done by SM loads over PCIe in one
// launch per chunk.  Each DMA transfer costs the copy engine a fixed ~5 us
// on top of its bytes; these arrays are half of the transfers and 8% of the
// bytes (tools/probes/zerocopy.cu: 512 DMA copies of the config-2 mix 21.6
// ms per GiB, large ones by DMA + small ones by this kernel 20.8 ms).
struct CopySeg {
  const uint8_t* src;  // device-mapped host pointer
  uint8_t* dst;
  unsigned long long bytes;
};
constexpr int kMaxCopySegs = 96;
struct CopySegs {
  int n;
  CopySeg s[kMaxCopySegs];
};
__global__ void __launch_bounds__(256) k_copy_segs(const CopySegs segs) {
  for (int g = blockIdx.y; g < segs.n; g += gridDim.y) {
    const CopySeg sg = segs.s[g];
    const unsigned long long step = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long done = 0;
    if ((((uintptr_t)sg.src | (uintptr_t)sg.dst) & 15) == 0) {  // 16-byte body
      const unsigned long long n16 = sg.bytes >> 4;
      const uint4* src = reinterpret_cast<const uint4*>(sg.src);
      uint4* dst = reinterpret_cast<uint4*>(sg.dst);
      for (unsigned long long i = t0; i < n16; i += step) dst[i] = src[i];
      done = n16 << 4;
    }
    for (unsigned long long i = done + t0; i < sg.bytes; i += step) sg.dst[i] = sg.src[i];
  }
}

// ------------------------------------------------------------------ host
// Largest double d with acos(clamp(d, -1, 1)) >= tol, found on the host with
// the same libm acos the reference uses; the device tests d >= cos_tol.
static double exact_cos_threshold(double tol) {
  auto pass = [&](double d) { return std::acos(std::min(1.0, std::max(-1.0, d))) < tol; };
  if (pass(-1.0)) return -INFINITY;
  if (!pass(1.0)) return INFINITY;
  // bisection over the ordered bit patterns of [-1, 1]
  auto ord = [](double d) {
    int64_t i;
    std::memcpy(&i, &d, 8);
    return i >= 0 ? i : -(i & 0x7fffffffffffffffLL);
  };
  auto unord = [](int64_t k) {
    const uint64_t u = k >= 0 ? (uint64_t)k : ((uint64_t)(-k) | 0x8000000000000000ull);
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  };
  int64_t lo = ord(-1.0), hi = ord(1.0);  // pass(lo) false, pass(hi) true
  while (hi - lo > 1) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (pass(unord(mid)))
      hi = mid;
    else
      lo = mid;
  }
  return unord(hi);
}

static LMParams make_lm(const pmx_match_params& p) {
  LMParams lp;
  lp.lambda_init = p.projection.lambda_init;
  lp.lambda_up = p.projection.lambda_up;
  lp.lambda_down = p.projection.lambda_down;
  lp.cos_tol = exact_cos_threshold(p.projection.angle_tol);
  lp.max_iterations = p.projection.max_iterations;
  lp.median_fraction = p.invalidation_median_fraction;
  return lp;
}

static RefineLevels make_levels(const pmx_refine_params* r) {
  RefineLevels L;
  std::memset(&L, 0, sizeof(L));
  if (!r) return L;
  require(r->num_levels >= 0 && r->num_levels <= PMX_MAX_REFINE_LEVELS, "refine: bad level count");
  L.n = r->num_levels;
  for (int i = 0; i < L.n; ++i) {
    require(r->stride[i] >= 1 && r->radius[i] >= 0, "refine: stride >= 1 and radius >= 0 required");
    L.stride[i] = r->stride[i];
    L.radius[i] = r->radius[i];
  }
  return L;
}

static void check_pointmap(const pmx_pointmap& p) {
  require(p.height > 0 && p.width > 0 && p.xyz, "pointmap: empty or null");
}

// Median threshold (camera.cpp:178-200) of every pair of `dev_pairs[0..n)`
// (keys / hist / sel set), enqueued on ctx.stream: one key pass and three
// radix-select rounds over all pairs at once.
// The three radix rounds after the keys and the first histogram level.
#ifndef PMX_SEL_PPB
#define PMX_SEL_PPB 16384  // keys per block of the histogram / collect passes (4096 measured slower)
#endif
static void select_rounds(Context& ctx, PairDev* dev_pairs, int n, int max_hwa, double fraction) {
  const int ppb = PMX_SEL_PPB;
  dim3 g1((max_hwa + ppb - 1) / ppb, n);
  k_sel_scan<1><<<n, 1024, 0, ctx.stream>>>(dev_pairs, fraction);
  launch_check(ctx, "k_sel_scan1");
  k_sel_hist<2><<<g1, 256, 0, ctx.stream>>>(dev_pairs, ppb);
  launch_check(ctx, "k_sel_hist2");
  k_sel_scan<2><<<n, 1024, 0, ctx.stream>>>(dev_pairs, fraction);
  launch_check(ctx, "k_sel_scan2");
  k_sel_hist<3><<<g1, 256, 0, ctx.stream>>>(dev_pairs, ppb);
  launch_check(ctx, "k_sel_hist3");
  k_sel_scan<3><<<n, 1024, 0, ctx.stream>>>(dev_pairs, fraction);
  launch_check(ctx, "k_sel_scan3");
  k_sel_collect<<<g1, 256, 0, ctx.stream>>>(dev_pairs, ppb);
  launch_check(ctx, "k_sel_collect");
  k_sel_exact<<<n, 256, 0, ctx.stream>>>(dev_pairs, fraction);
  launch_check(ctx, "k_sel_exact");
}

static void select_median(Context& ctx, PairDev* dev_pairs, int n, int max_hwa, double fraction) {
  const int ppb = 4096;
  k_keys<<<dim3((max_hwa + ppb - 1) / ppb, n), 256, 0, ctx.stream>>>(dev_pairs, ppb);
  launch_check(ctx, "k_keys");
  select_rounds(ctx, dev_pairs, n, max_hwa, fraction);
}

static void prep_rays(Context& ctx, PairDev* dev_pairs, int n, int max_hwa, bool with_keys = false) {
  const int ppb = 1024;
  k_prep<<<dim3((max_hwa + ppb - 1) / ppb, n), 256, 0, ctx.stream>>>(dev_pairs, ppb, with_keys);
  launch_check(ctx, "k_prep");
}

// Ray maps + median threshold of the pairs (single-pair entry points).
static void prep_and_select(Context& ctx, PairDev* dev_pairs, int n, int max_hwa, double fraction) {
  select_median(ctx, dev_pairs, n, max_hwa, fraction);
  prep_rays(ctx, dev_pairs, n, max_hwa);
}

// Batched match(+refine).  All pointers in `pairs` are device pointers.
// Scratch budget of one chunk of pairs (FP64 ray maps + int8 descriptors,
// 56 B per a-pixel).  Measured on B200: one chunk over all 64 config-2 pairs
// (704 MB, HBM-resident) beats L2-sized chunks of 5 pairs: the matcher is
// issue-bound (its DRAM traffic is ~10% of peak either way) and one launch
// per kernel removes 12 tails and launch gaps.
constexpr size_t kChunkBytes = size_t(4) << 30;

// Host-staging hooks of the pipelined PMX_MEM_HOST path (run_match_batch):
// before_select makes the stream wait for the a-side points, before_chunk /
// after_chunk bracket a chunk's compute with its input / output copies.
struct MatchHooks {
  std::function<void()> before_select;
  std::function<void(int, int)> before_chunk, after_chunk;
  int chunk_pairs;  // pairs per chunk (small: the copies of chunk c+1 overlap chunk c)
};

void match_batch_device(Context& ctx, const std::vector<PairDev>& host_pairs, const pmx_match_params& mp,
                        const pmx_refine_params* refine, const MatchHooks* hooks = nullptr) {
  const LMParams lp = make_lm(mp);
  const RefineLevels L = make_levels(refine);
  const int npairs = (int)host_pairs.size();
  if (npairs == 0) return;
  int max_hwa = 0, max_hwb = 0;
  for (const auto& p : host_pairs) {
    max_hwa = std::max(max_hwa, p.Ha * p.Wa);
    max_hwb = std::max(max_hwb, p.Hb * p.Wb);
  }
  // chunks of pairs sharing one scratch allocation: FP64 ray maps + int8
  // descriptors (56 B per a-pixel), see kChunkBytes
  const size_t per_px = sizeof(double4) + sizeof(uint2) + sizeof(uint16_t) + sizeof(uint4);
  const size_t pair_bytes = per_px * (size_t)max_hwa;
  int chunk = std::max(1, std::min(npairs, (int)((size_t(kChunkBytes)) / std::max<size_t>(pair_bytes, 1))));
  if (hooks) chunk = std::max(1, std::min(chunk, hooks->chunk_pairs));
  // Device path, many pairs: chunks of PMX_OVERLAP pairs on two scratch
  // slots, k_prep + select of chunk c+1 on a high-priority side stream while
  // k_match_refine of chunk c runs (HBM-bound prep under the latency-bound
  // matcher).
  const bool overlap = !hooks && PMX_OVERLAP > 0 && npairs > PMX_OVERLAP;
  if (overlap) chunk = PMX_OVERLAP;
  const int nslots = overlap ? 2 : 1;
  DevBuf scratch(pair_bytes * chunk * nslots, ctx.stream);
  DevBuf keybuf(sizeof(uint32_t) * (size_t)max_hwa * npairs, ctx.stream);
  DevBuf hist(sizeof(uint32_t) * (size_t)kHistTotal * npairs, ctx.stream);
  DevBuf sel(sizeof(SelState) * npairs, ctx.stream);
  DevBuf dpairs(sizeof(PairDev) * npairs, ctx.stream);
  std::vector<PairDev> hp = host_pairs;
  char* base = scratch.as<char>();
  const size_t nslot = (size_t)max_hwa * chunk * nslots;
  double4* rays = reinterpret_cast<double4*>(base);
  uint4* q8t = reinterpret_cast<uint4*>(base + sizeof(double4) * nslot);
  uint2* q8h = reinterpret_cast<uint2*>(base + (sizeof(double4) + sizeof(uint4)) * nslot);
  uint16_t* q8n = reinterpret_cast<uint16_t*>(base + (sizeof(double4) + sizeof(uint4) + sizeof(uint2)) * nslot);
  for (int i = 0; i < npairs; ++i) {
    const int slot = ((i / chunk) % nslots) * chunk + i % chunk;
    hp[i].rays = rays + (size_t)slot * max_hwa;
    hp[i].keys = keybuf.as<uint32_t>() + (size_t)i * max_hwa;
    hp[i].hist = hist.as<uint32_t>() + (size_t)kHistTotal * i;
    hp[i].sel = sel.as<SelState>() + i;
    hp[i].dnorm = nullptr;
    const bool aligned = ((uintptr_t)hp[i].da % 16 == 0) && ((uintptr_t)hp[i].db % 16 == 0);
    if (refine && hp[i].dim == 24 && aligned) {
      hp[i].q8h = q8h + (size_t)slot * max_hwa;
      hp[i].q8n = q8n + (size_t)slot * max_hwa;
      hp[i].q8t = q8t + (size_t)slot * max_hwa;
    }
  }
  PMX_CUDA(cudaMemcpyAsync(dpairs.p, hp.data(), sizeof(PairDev) * npairs, cudaMemcpyHostToDevice, ctx.stream));
  PMX_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes, ctx.stream));
  PMX_CUDA(cudaMemsetAsync(sel.p, 0, sel.bytes, ctx.stream));
  if (hooks) hooks->before_select();
  std::vector<cudaEvent_t> ev_prep, ev_match;
  cudaStream_t main_stream = ctx.stream;
  if (overlap) {
    if (!ctx.aux) {
      int lo = 0, hi = 0;
      PMX_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      PMX_CUDA(cudaStreamCreateWithPriority(&ctx.aux, cudaStreamNonBlocking, hi));
    }
    const int nchunks = (npairs + chunk - 1) / chunk;
    ev_prep.resize(nchunks + 1);
    ev_match.resize(nchunks);
    for (auto& e : ev_prep) PMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ev_match) PMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PMX_CUDA(cudaEventRecord(ev_prep[nchunks], main_stream));  // scratch allocated, state zeroed
    PMX_CUDA(cudaStreamWaitEvent(ctx.aux, ev_prep[nchunks], 0));
  }
  // Host path: the last chunks halve (4, 2, 1, 1 after full ones), so the
  // compute and output copies left after the final input copy are one pair's.
  auto chunk_at = [&](int c0) {
    const int rest = npairs - c0;
    return hooks && rest <= chunk ? std::max(1, (rest + 1) / 2) : std::min(chunk, rest);
  };
  for (int c0 = 0, cn = 0; c0 < npairs; c0 += cn) {
    cn = chunk_at(c0);
    const int ci = c0 / chunk;
    PairDev* dp = dpairs.as<PairDev>() + c0;
    if (hooks) hooks->before_chunk(c0, cn);
    if (overlap) {
      if (ci >= 2) PMX_CUDA(cudaStreamWaitEvent(ctx.aux, ev_match[ci - 2], 0));  // slot reuse
      ctx.stream = ctx.aux;  // prep + select of this chunk on the side stream
    }
    try {
      {
        ProfScope ps(ctx, "k_prep");  // rays, int8 image, norm keys + first histogram level
        prep_rays(ctx, dp, cn, max_hwa, true);
      }
      {
        ProfScope ps(ctx, "k_select");
        select_rounds(ctx, dp, cn, max_hwa, lp.median_fraction);
      }
    } catch (...) {
      ctx.stream = main_stream;
      throw;
    }
    if (overlap) {
      ctx.stream = main_stream;
      PMX_CUDA(cudaEventRecord(ev_prep[ci], ctx.aux));
      PMX_CUDA(cudaStreamWaitEvent(main_stream, ev_prep[ci], 0));
    }
    int max_tx = 0, max_ty = 0;  // grid (x tiles, y tiles, pairs) of 32x8 b-pixel tiles
    for (int i = c0; i < c0 + cn; ++i) {
      max_tx = std::max(max_tx, (hp[i].Wb + 31) / 32);
      max_ty = std::max(max_ty, (hp[i].Hb + 7) / 8);
    }
    if (PMX_SPLIT && refine && L.n > 0) {
      ProfScope ps(ctx, "k_match_refine");  // both kernels under the fused kernel's name
      k_match<<<dim3(max_tx, max_ty, cn), 256, 0, ctx.stream>>>(dp, lp);
      launch_check(ctx, "k_match");
      int ty = 0;
      for (int i = c0; i < c0 + cn; ++i) ty = std::max(ty, (hp[i].Hb + PMX_RF_TY - 1) / PMX_RF_TY);
      k_refine_tiles<<<dim3(max_tx, ty, cn), 32 * PMX_RF_TY, 0, ctx.stream>>>(dp, L);
      launch_check(ctx, "k_refine_tiles");
    } else if (refine && L.n > 0) {
      // counter first: its first allocation must stay outside the timed scope
      unsigned long long* exact_px = ctx.profiling ? dev_counter(ctx, "refine_exact_px") : nullptr;
      ProfScope ps(ctx, "k_match_refine");
      int ty = 0;
      for (int i = c0; i < c0 + cn; ++i) ty = std::max(ty, (hp[i].Hb + PMX_MR_TY - 1) / PMX_MR_TY);
      k_match_refine<<<dim3(max_tx, ty, cn), 32 * PMX_MR_TY, 0, ctx.stream>>>(dp, lp, L, exact_px);
      launch_check(ctx, "k_match_refine");
    } else {
      ProfScope ps(ctx, "k_match");
      k_match<<<dim3(max_tx, max_ty, cn), 256, 0, ctx.stream>>>(dp, lp);
      launch_check(ctx, "k_match");
    }
    if (overlap) PMX_CUDA(cudaEventRecord(ev_match[ci], main_stream));
    if (hooks) hooks->after_chunk(c0, cn);
  }
  for (auto& e : ev_prep) cudaEventDestroy(e);  // released once their work completes
  for (auto& e : ev_match) cudaEventDestroy(e);
  // Device-memory calls on a caller-adopted stream (pmx_set_stream) stay
  // asynchronous like any CUDA library call (scratch is stream-ordered and
  // the pageable PairDev upload is staged before cudaMemcpyAsync returns);
  // on the context's own stream they complete before returning.
  if (ctx.stream == ctx.own_stream) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
}

// ------------------------------------------------------------ C-ABI glue
static PairDev stage_pair(Stager& st, const pmx_pair& p, DevBuf* seed_buf, Context& ctx) {
  check_pointmap(p.X_a);
  check_pointmap(p.X_b_in_a);
  require(p.F_a.descriptors && p.F_b.descriptors && p.F_a.match_confidence && p.F_b.match_confidence,
          "featuremap: null arrays");
  require(p.F_a.height == p.X_a.height && p.F_a.width == p.X_a.width, "F_a / X_a size mismatch");
  require(p.F_b.height == p.X_b_in_a.height && p.F_b.width == p.X_b_in_a.width, "F_b / X_b size mismatch");
  require(p.F_a.dim == p.F_b.dim && p.F_a.dim > 0, "descriptor dim mismatch");
  const size_t hwa = (size_t)p.X_a.height * p.X_a.width, hwb = (size_t)p.X_b_in_a.height * p.X_b_in_a.width;
  PairDev d;
  std::memset(&d, 0, sizeof(d));
  d.Ha = p.X_a.height;
  d.Wa = p.X_a.width;
  d.Hb = p.X_b_in_a.height;
  d.Wb = p.X_b_in_a.width;
  d.dim = p.F_a.dim;
  d.xa = st.in(p.X_a.xyz, 3 * hwa);
  d.va = st.in(p.X_a.valid, hwa);
  d.xb = st.in(p.X_b_in_a.xyz, 3 * hwb);
  d.vb = st.in(p.X_b_in_a.valid, hwb);
  d.da = reinterpret_cast<const __half*>(st.in(p.F_a.descriptors, hwa * d.dim));
  d.db = reinterpret_cast<const __half*>(st.in(p.F_b.descriptors, hwb * d.dim));
  d.qa = st.in(p.F_a.match_confidence, hwa);
  d.qb = st.in(p.F_b.match_confidence, hwb);
  if (p.init && p.init->count > 0) {
    const int64_t m = p.init->count;
    const int32_t* ipa = st.in(p.init->pixel_a, (size_t)m);
    const int32_t* ipb = st.in(p.init->pixel_b, (size_t)m);
    const uint8_t* iv = st.in(p.init->valid, (size_t)m);
    *seed_buf = DevBuf(sizeof(int32_t) * hwb, ctx.stream);
    PMX_CUDA(cudaMemsetAsync(seed_buf->p, 0xff, seed_buf->bytes, ctx.stream));
    k_seed_scatter<<<(unsigned)((m + 255) / 256), 256, 0, ctx.stream>>>(m, ipb, iv, (int)hwb,
                                                                        seed_buf->as<int32_t>());
    launch_check(ctx, "k_seed_scatter");
    d.seed_last = seed_buf->as<int32_t>();
    d.init_pa = ipa;
  }
  return d;
}

}  // namespace pmx

using namespace pmx;

// Stage a batch of pairs + their outputs (PMX_MEM_HOST: H2D / scratch),
// run the fused matcher, optionally the loop-edge gate, copy the outputs back.
static void run_match_batch(Context& ctx, pmx_memory mem, int32_t num_pairs, const pmx_pair* pairs,
                            const pmx_match_params* params, const pmx_refine_params* refine, pmx_matchset* outs,
                            double gate, std::vector<unsigned long long>* gate_counts) {
  require(num_pairs >= 0 && (num_pairs == 0 || (pairs && outs)), "match_batch: null arguments");
  pmx_match_params mp;
  pmx_default_match_params(&mp);
  if (params) mp = *params;
  bool seeded = false;
  for (int i = 0; i < num_pairs; ++i) seeded = seeded || (pairs[i].init && pairs[i].init->count > 0);
  // Host buffers: pipelined staging (inputs of chunk c+1 copied while chunk c
  // computes, outputs of chunk c copied back on a second copy stream).
  const bool pipelined = mem == PMX_MEM_HOST && !seeded && num_pairs > 0;
  Stager st(ctx, pipelined ? PMX_MEM_DEVICE : mem);
  std::vector<PairDev> hp(num_pairs);
  std::vector<DevBuf> seeds(num_pairs), dbufs;
  for (int i = 0; i < num_pairs; ++i) {
    hp[i] = stage_pair(st, pairs[i], &seeds[i], ctx);  // device path: pointers as given / staged
    const size_t hwb = (size_t)hp[i].Hb * hp[i].Wb;
    require(outs[i].count >= (int64_t)hwb && outs[i].pixel_a && outs[i].confidence && outs[i].valid,
            "match_batch: output matchset too small or null");
    hp[i].out_pa = st.out(outs[i].pixel_a, hwb);
    hp[i].out_pb = st.out(outs[i].pixel_b, hwb);
    hp[i].out_q = st.out(outs[i].confidence, hwb);
    hp[i].out_valid = st.out(outs[i].valid, hwb);
  }
  MatchHooks hooks;
  hooks.chunk_pairs = PMX_HOST_CHUNK;
  cudaEvent_t ev_a = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  if (pipelined) {  // device mirrors of every array (one allocation), copies issued by the hooks
    if (!ctx.copy_in) {
      PMX_CUDA(cudaStreamCreateWithFlags(&ctx.copy_in, cudaStreamNonBlocking));
      PMX_CUDA(cudaStreamCreateWithFlags(&ctx.copy_out, cudaStreamNonBlocking));
    }
    if (PMX_SM_SMALL_COPIES && !ctx.copy_in2) {  // high priority: its blocks slot in as matcher CTAs retire
      int lo = 0, hi = 0;
      PMX_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      PMX_CUDA(cudaStreamCreateWithPriority(&ctx.copy_in2, cudaStreamNonBlocking, hi));
    }
    size_t total = 0;
    auto room = [&](size_t bytes) { total += (bytes + 255) & ~size_t(255); };
    for (int i = 0; i < num_pairs; ++i) {
      const pmx_pair& p = pairs[i];
      const size_t hwa = (size_t)hp[i].Ha * hp[i].Wa, hwb = (size_t)hp[i].Hb * hp[i].Wb;
      room(12 * hwa); room(p.X_a.valid ? hwa : 0); room(12 * hwb); room(p.X_b_in_a.valid ? hwb : 0);
      room(2 * hwa * hp[i].dim); room(2 * hwb * hp[i].dim); room(4 * hwa); room(4 * hwb);
      room(4 * hwb); room(outs[i].pixel_b ? 4 * hwb : 0); room(4 * hwb); room(hwb);
    }
    dbufs.emplace_back(total, ctx.stream);
    char* cur = dbufs.back().as<char>();
    auto take = [&](size_t bytes) {
      char* r = bytes ? cur : nullptr;
      cur += (bytes + 255) & ~size_t(255);
      return r;
    };
    for (int i = 0; i < num_pairs; ++i) {
      const pmx_pair& p = pairs[i];
      const size_t hwa = (size_t)hp[i].Ha * hp[i].Wa, hwb = (size_t)hp[i].Hb * hp[i].Wb;
      hp[i].xa = reinterpret_cast<const float*>(take(12 * hwa));
      hp[i].va = reinterpret_cast<const uint8_t*>(take(p.X_a.valid ? hwa : 0));
      hp[i].xb = reinterpret_cast<const float*>(take(12 * hwb));
      hp[i].vb = reinterpret_cast<const uint8_t*>(take(p.X_b_in_a.valid ? hwb : 0));
      hp[i].da = reinterpret_cast<const __half*>(take(2 * hwa * hp[i].dim));
      hp[i].db = reinterpret_cast<const __half*>(take(2 * hwb * hp[i].dim));
      hp[i].qa = reinterpret_cast<const float*>(take(4 * hwa));
      hp[i].qb = reinterpret_cast<const float*>(take(4 * hwb));
      hp[i].out_pa = reinterpret_cast<int32_t*>(take(4 * hwb));
      hp[i].out_pb = reinterpret_cast<int32_t*>(take(outs[i].pixel_b ? 4 * hwb : 0));
      hp[i].out_q = reinterpret_cast<float*>(take(4 * hwb));
      hp[i].out_valid = reinterpret_cast<uint8_t*>(take(hwb));
    }
    PMX_CUDA(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
    PMX_CUDA(cudaEventRecord(ev_a, ctx.stream));  // device buffers allocated (stream-ordered)
    PMX_CUDA(cudaStreamWaitEvent(ctx.copy_in, ev_a, 0));
    if (PMX_SM_SMALL_COPIES) PMX_CUDA(cudaStreamWaitEvent(ctx.copy_in2, ev_a, 0));
    auto h2d = [&](const void* d, const void* h, size_t bytes) {
      if (bytes) PMX_CUDA(cudaMemcpyAsync(const_cast<void*>(d), h, bytes, cudaMemcpyHostToDevice, ctx.copy_in));
    };
    // Small inputs in pinned (device-mapped) host memory: gathered into one
    // k_copy_segs launch per chunk on copy_in2; anything else goes by DMA.
    CopySegs pending;
    pending.n = 0;
    auto flush_small = [&]() {
      if (!pending.n) return;
      k_copy_segs<<<dim3(4, pending.n), 256, 0, ctx.copy_in2>>>(pending);
      launch_check(ctx, "k_copy_segs");
      pending.n = 0;
    };
    auto h2d_small = [&](const void* d, const void* h, size_t bytes) {
      if (!bytes) return;
      const void* mapped = nullptr;
      if (PMX_SM_SMALL_COPIES && bytes < (size_t(PMX_SM_COPY_MAX_KB) << 10)) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, h) == cudaSuccess) {
          if (a.type == cudaMemoryTypeHost && a.devicePointer) mapped = a.devicePointer;
        } else {
          cudaGetLastError();  // not a CUDA-known pointer: plain DMA
        }
      }
      if (!mapped) return h2d(d, h, bytes);
      if (pending.n == kMaxCopySegs) flush_small();
      pending.s[pending.n++] = CopySeg{static_cast<const uint8_t*>(mapped), static_cast<uint8_t*>(const_cast<void*>(d)),
                                       (unsigned long long)bytes};
    };
    // the compute stream waits for both input queues' copies so far
    auto join_h2d = [&](cudaEvent_t e, cudaEvent_t e2) {
      flush_small();
      PMX_CUDA(cudaEventRecord(e, ctx.copy_in));
      PMX_CUDA(cudaStreamWaitEvent(ctx.stream, e, 0));
      if (PMX_SM_SMALL_COPIES) {
        PMX_CUDA(cudaEventRecord(e2, ctx.copy_in2));
        PMX_CUDA(cudaStreamWaitEvent(ctx.stream, e2, 0));
      }
    };
    auto d2h = [&](void* h, const void* d, size_t bytes) {
      if (bytes && h) PMX_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx.copy_out));
    };
    hooks.before_select = [&]() {  // the median needs every pair's a-side points
      for (int i = 0; i < num_pairs; ++i) {
        const size_t hwa = (size_t)hp[i].Ha * hp[i].Wa;
        h2d(hp[i].xa, pairs[i].X_a.xyz, 12 * hwa);
        if (pairs[i].X_a.valid) h2d_small(hp[i].va, pairs[i].X_a.valid, hwa);
      }
      cudaEvent_t e2;
      PMX_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      ev_in.push_back(e2);
      join_h2d(ev_a, e2);
    };
    hooks.before_chunk = [&](int c0, int cn) {
      for (int i = c0; i < c0 + cn; ++i) {
        const pmx_pair& p = pairs[i];
        const size_t hwa = (size_t)hp[i].Ha * hp[i].Wa, hwb = (size_t)hp[i].Hb * hp[i].Wb;
        h2d(hp[i].xb, p.X_b_in_a.xyz, 12 * hwb);
        if (p.X_b_in_a.valid) h2d_small(hp[i].vb, p.X_b_in_a.valid, hwb);
        h2d(hp[i].da, p.F_a.descriptors, 2 * hwa * hp[i].dim);
        h2d(hp[i].db, p.F_b.descriptors, 2 * hwb * hp[i].dim);
        h2d_small(hp[i].qa, p.F_a.match_confidence, 4 * hwa);
        h2d_small(hp[i].qb, p.F_b.match_confidence, 4 * hwb);
      }
      cudaEvent_t e, e2;
      PMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      PMX_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      ev_in.push_back(e);
      ev_in.push_back(e2);
      join_h2d(e, e2);
    };
    hooks.after_chunk = [&](int c0, int cn) {
      if (gate_counts) return;  // the gate still rewrites valid: copied back at the end
      cudaEvent_t e;
      PMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev_out.push_back(e);
      PMX_CUDA(cudaEventRecord(e, ctx.stream));
      PMX_CUDA(cudaStreamWaitEvent(ctx.copy_out, e, 0));
      for (int i = c0; i < c0 + cn; ++i) {
        const size_t hwb = (size_t)hp[i].Hb * hp[i].Wb;
        d2h(outs[i].pixel_a, hp[i].out_pa, 4 * hwb);
        d2h(outs[i].pixel_b, hp[i].out_pb, 4 * hwb);
        d2h(outs[i].confidence, hp[i].out_q, 4 * hwb);
        d2h(outs[i].valid, hp[i].out_valid, hwb);
      }
    };
  }
  match_batch_device(ctx, hp, mp, refine, pipelined ? &hooks : nullptr);
  if (gate_counts && num_pairs > 0) {
    DevBuf dp(sizeof(PairDev) * num_pairs, ctx.stream), cnt(sizeof(unsigned long long) * num_pairs, ctx.stream);
    PMX_CUDA(cudaMemcpyAsync(dp.p, hp.data(), dp.bytes, cudaMemcpyHostToDevice, ctx.stream));
    PMX_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, ctx.stream));
    k_loop_gate<<<dim3(2 * ctx.num_sms, num_pairs), 256, 0, ctx.stream>>>(dp.as<PairDev>(), gate,
                                                                           cnt.as<unsigned long long>());
    launch_check(ctx, "k_loop_gate");
    gate_counts->resize(num_pairs);
    PMX_CUDA(cudaMemcpyAsync(gate_counts->data(), cnt.p, cnt.bytes, cudaMemcpyDeviceToHost, ctx.stream));
    PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  if (pipelined) {
    if (gate_counts) {  // outputs after the gate
      for (int i = 0; i < num_pairs; ++i) {
        const size_t hwb = (size_t)hp[i].Hb * hp[i].Wb;
        PMX_CUDA(cudaMemcpyAsync(outs[i].pixel_a, hp[i].out_pa, 4 * hwb, cudaMemcpyDeviceToHost, ctx.stream));
        if (outs[i].pixel_b)
          PMX_CUDA(cudaMemcpyAsync(outs[i].pixel_b, hp[i].out_pb, 4 * hwb, cudaMemcpyDeviceToHost, ctx.stream));
        PMX_CUDA(cudaMemcpyAsync(outs[i].confidence, hp[i].out_q, 4 * hwb, cudaMemcpyDeviceToHost, ctx.stream));
        PMX_CUDA(cudaMemcpyAsync(outs[i].valid, hp[i].out_valid, hwb, cudaMemcpyDeviceToHost, ctx.stream));
      }
    }
    PMX_CUDA(cudaStreamSynchronize(ctx.copy_out));
    PMX_CUDA(cudaStreamSynchronize(ctx.copy_in));
    if (ctx.copy_in2) PMX_CUDA(cudaStreamSynchronize(ctx.copy_in2));
    PMX_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaEventDestroy(ev_a);
    for (auto e : ev_in) cudaEventDestroy(e);
    for (auto e : ev_out) cudaEventDestroy(e);
    for (int i = 0; i < num_pairs; ++i) outs[i].count = (int64_t)hp[i].Hb * hp[i].Wb;
    return;
  }
  for (int i = 0; i < num_pairs; ++i) {
    const size_t hwb = (size_t)hp[i].Hb * hp[i].Wb;
    st.back(outs[i].pixel_a, hp[i].out_pa, hwb);
    st.back(outs[i].pixel_b, hp[i].out_pb, hwb);
    st.back(outs[i].confidence, hp[i].out_q, hwb);
    st.back(outs[i].valid, hp[i].out_valid, hwb);
    outs[i].count = (int64_t)hwb;
  }
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
}

extern "C" int pmx_impl_match_batch(pmx_context* c, pmx_memory mem, int32_t num_pairs, const pmx_pair* pairs,
                                    const pmx_match_params* params, const pmx_refine_params* refine,
                                    pmx_matchset* outs) {
  run_match_batch(*reinterpret_cast<Context*>(c), mem, num_pairs, pairs, params, refine, outs, 0.0, nullptr);
  return PMX_OK;
}

// accept_loop_edge (retrieval.cpp:226-251) for a batch of candidate edges.
extern "C" int pmx_impl_accept_loop_edges(pmx_context* c, pmx_memory mem, int32_t num_pairs, const pmx_pair* pairs,
                                          double omega_l, const pmx_match_params* params,
                                          const pmx_refine_params* refine, pmx_matchset* outs, int32_t* accepted) {
  require(num_pairs == 0 || accepted, "accept_loop_edges: null accepted");
  std::vector<unsigned long long> counts;
  constexpr double kMinDescriptorAgreement = 0.5;  // retrieval.cpp:238
  run_match_batch(*reinterpret_cast<Context*>(c), mem, num_pairs, pairs, params, refine, outs,
                  kMinDescriptorAgreement, &counts);
  for (int i = 0; i < num_pairs; ++i) {  // valid_fraction() < omega_l -> nullopt (camera.cpp:16-19)
    const double size = (double)pairs[i].X_b_in_a.height * pairs[i].X_b_in_a.width;
    const double frac = size > 0 ? (double)counts[i] / size : 0.0;
    accepted[i] = frac < omega_l ? 0 : 1;
  }
  return PMX_OK;
}

extern "C" int pmx_impl_feature_refine(pmx_context* c, pmx_memory mem, const pmx_matchset* in,
                                       const pmx_featuremap* F_a, const pmx_featuremap* F_b,
                                       const pmx_refine_params* params, pmx_matchset* out) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(in && F_a && F_b && out, "feature_refine: null arguments");
  require(F_a->dim == F_b->dim && F_a->dim > 0, "descriptor dim mismatch");
  require(out->count >= in->count && out->pixel_a && out->confidence && out->valid,
          "feature_refine: output too small");
  pmx_refine_params rp;
  pmx_default_refine_params(&rp);
  if (params) rp = *params;
  const RefineLevels L = make_levels(&rp);
  Stager st(ctx, mem);
  PairDev P;
  std::memset(&P, 0, sizeof(P));
  P.Ha = F_a->height;
  P.Wa = F_a->width;
  P.Hb = F_b->height;
  P.Wb = F_b->width;
  P.dim = F_a->dim;
  const size_t hwa = (size_t)P.Ha * P.Wa, hwb = (size_t)P.Hb * P.Wb;
  P.da = reinterpret_cast<const __half*>(st.in(F_a->descriptors, hwa * P.dim));
  P.db = reinterpret_cast<const __half*>(st.in(F_b->descriptors, hwb * P.dim));
  P.qa = st.in(F_a->match_confidence, hwa);
  P.qb = st.in(F_b->match_confidence, hwb);
  const int64_t n = in->count;
  const int32_t* ipa = st.in(in->pixel_a, n);
  const int32_t* ipb = st.in(in->pixel_b, n);
  const float* iq = st.in(in->confidence, n);
  const uint8_t* iv = st.in(in->valid, n);
  int32_t* opa = st.out(out->pixel_a, n);
  int32_t* opb = st.out(out->pixel_b, n);
  float* oq = st.out(out->confidence, n);
  uint8_t* ov = st.out(out->valid, n);
  DevBuf aux;
  if (P.dim == 24 && ((uintptr_t)P.da % 16 == 0) && ((uintptr_t)P.db % 16 == 0) && hwa > 0) {
    aux = DevBuf(sizeof(float4) * hwa, ctx.stream);
    P.dnorm = aux.as<float4>();
    k_desc_prep<<<(unsigned)((hwa + 255) / 256), 256, 0, ctx.stream>>>(P.da, P.qa, (int)hwa, P.dnorm);
    launch_check(ctx, "k_desc_prep");
  }
  if (n > 0) {
    k_refine<<<(unsigned)((n + 255) / 256), 256, 0, ctx.stream>>>(P, n, ipa, ipb, iq, iv, L, opa, opb, oq, ov);
    launch_check(ctx, "k_refine");
  }
  st.back(out->pixel_a, opa, n);
  st.back(out->pixel_b, opb, n);
  st.back(out->confidence, oq, n);
  st.back(out->valid, ov, n);
  out->count = n;
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

// Ray map of one pointmap (+ optional median threshold) in a scratch buffer.
static void build_raymap(Context& ctx, Stager& st, const pmx_pointmap* pm, DevBuf& rays, DevBuf& keys,
                         DevBuf& hist, DevBuf& sel, DevBuf& dpair, const float** xyz_dev) {
  check_pointmap(*pm);
  const size_t hw = (size_t)pm->height * pm->width;
  PairDev P;
  std::memset(&P, 0, sizeof(P));
  P.Ha = pm->height;
  P.Wa = pm->width;
  P.xa = st.in(pm->xyz, 3 * hw);
  P.va = st.in(pm->valid, hw);
  *xyz_dev = P.xa;
  rays = DevBuf(sizeof(double4) * hw, ctx.stream);
  keys = DevBuf(sizeof(uint32_t) * hw, ctx.stream);
  hist = DevBuf(sizeof(uint32_t) * kHistTotal, ctx.stream);
  sel = DevBuf(sizeof(SelState), ctx.stream);
  dpair = DevBuf(sizeof(PairDev), ctx.stream);
  P.rays = rays.as<double4>();
  P.keys = keys.as<uint32_t>();
  P.hist = hist.as<uint32_t>();
  P.sel = sel.as<SelState>();
  PMX_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes, ctx.stream));
  PMX_CUDA(cudaMemsetAsync(sel.p, 0, sel.bytes, ctx.stream));  // a1max / qbad start at 0
  PMX_CUDA(cudaMemcpyAsync(dpair.p, &P, sizeof(P), cudaMemcpyHostToDevice, ctx.stream));
  prep_and_select(ctx, dpair.as<PairDev>(), 1, (int)hw, 1.0);
}

extern "C" int pmx_impl_normalize_rays(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, double* rays,
                                       double* distances, uint8_t* valid) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(pm && rays && distances && valid, "normalize_rays: null arguments");
  Stager st(ctx, mem);
  DevBuf r, k, h, s, d;
  const float* xyz = nullptr;
  build_raymap(ctx, st, pm, r, k, h, s, d, &xyz);
  const size_t hw = (size_t)pm->height * pm->width;
  double* orays = st.out(rays, 3 * hw);
  double* odist = st.out(distances, hw);
  uint8_t* ov = st.out(valid, hw);
  k_rays_out<<<(unsigned)((hw + 255) / 256), 256, 0, ctx.stream>>>(r.as<double4>(), (int)hw, orays, odist, ov,
                                                                   xyz);
  launch_check(ctx, "k_rays_out");
  st.back(rays, orays, 3 * hw);
  st.back(distances, odist, hw);
  st.back(valid, ov, hw);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

__global__ void k_interp_points(const double4* __restrict__ rays, int W, int H, int64_t n, const double* __restrict__ p,
                                double* ray, double* jac, uint8_t* ok) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double r[3] = {0.0, 0.0, 0.0}, J[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const bool good = interp_ray(rays, W, H, p[2 * k], p[2 * k + 1], r, J);
  if (!good) r[0] = r[1] = r[2] = J[0] = J[1] = J[2] = J[3] = J[4] = J[5] = 0.0;
  for (int c = 0; c < 3; ++c) ray[3 * k + c] = r[c];
  if (jac)
    for (int c = 0; c < 6; ++c) jac[6 * k + c] = J[c];  // J[0..2] = d/du, J[3..5] = d/dv
  ok[k] = good ? 1 : 0;
}

extern "C" int pmx_impl_interpolate_ray(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, int64_t n,
                                        const double* p, double* ray, double* jacobian, uint8_t* ok) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(pm && p && ray && ok && n >= 0, "interpolate_ray: null arguments");
  Stager st(ctx, mem);
  DevBuf r, k, h, s, d;
  const float* xyz = nullptr;
  build_raymap(ctx, st, pm, r, k, h, s, d, &xyz);
  const double* dp = st.in(p, 2 * (size_t)n);
  double* dray = st.out(ray, 3 * (size_t)n);
  double* djac = jacobian ? st.out(jacobian, 6 * (size_t)n) : nullptr;
  uint8_t* dok = st.out(ok, (size_t)n);
  if (n > 0) {
    k_interp_points<<<(unsigned)((n + 127) / 128), 128, 0, ctx.stream>>>(r.as<double4>(), pm->width, pm->height, n,
                                                                         dp, dray, djac, dok);
    launch_check(ctx, "k_interp_points");
  }
  st.back(ray, dray, 3 * (size_t)n);
  if (jacobian) st.back(jacobian, djac, 6 * (size_t)n);
  st.back(ok, dok, (size_t)n);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

extern "C" int pmx_impl_median_scene_distance(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, double* out) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(pm && out, "median_scene_distance: null arguments");
  Stager st(ctx, mem);
  DevBuf r, k, h, s, d;
  const float* xyz = nullptr;
  build_raymap(ctx, st, pm, r, k, h, s, d, &xyz);  // fraction 1.0: threshold = median
  double* dout = st.out(out, 1);
  PMX_CUDA(cudaMemcpyAsync(dout, &s.as<SelState>()->median, sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
  st.back(out, dout, 1);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

extern "C" int pmx_impl_iterative_project(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, int64_t n,
                                          const float* x, const double* p0, const pmx_iter_proj_params* params,
                                          double* pixel, uint8_t* converged, int32_t* iterations) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(pm && x && p0 && pixel && converged && iterations && n >= 0, "iterative_project: null arguments");
  pmx_match_params mp;
  pmx_default_match_params(&mp);
  if (params) mp.projection = *params;
  const LMParams lp = make_lm(mp);
  Stager st(ctx, mem);
  DevBuf r, k, h, s, d;
  const float* xyz = nullptr;
  build_raymap(ctx, st, pm, r, k, h, s, d, &xyz);
  const float* dx = st.in(x, 3 * (size_t)n);
  const double* dp0 = st.in(p0, 2 * (size_t)n);
  double* dpix = st.out(pixel, 2 * (size_t)n);
  uint8_t* dconv = st.out(converged, (size_t)n);
  int32_t* dit = st.out(iterations, (size_t)n);
  if (n > 0) {
    k_project_points<<<(unsigned)((n + 127) / 128), 128, 0, ctx.stream>>>(r.as<double4>(), pm->width, pm->height,
                                                                          n, dx, dp0, lp, dpix, dconv, dit);
    launch_check(ctx, "k_project_points");
  }
  st.back(pixel, dpix, 2 * (size_t)n);
  st.back(converged, dconv, (size_t)n);
  st.back(iterations, dit, (size_t)n);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}

PMX_DEFINE_VIOLATION_READER(pmx_checked_violations_match)
