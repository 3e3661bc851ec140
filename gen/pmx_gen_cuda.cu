// Synthetic BASELINE-config generator, device half (bench / test
// infrastructure, not the product): the per-edge pair predictions of the
// many-edge backend configs (3: 400 edges, 4: 5000 edges), generated on the
// GPU so their matches can be built by the matcher "as in config 2"
// (BASELINE.json configs 3/4) without minutes of host-side generation.
//
// Same model as gen/pmx_gen.cpp (gen_express / gen_pair_desc): counter-based
// splitmix64 hashes + explicit Box-Muller, radial point noise along the
// view's own ray, pair-predicted descriptors keyed by the rounded camera-a
// pixel of the surface point.  Values agree with the host generator up to the
// last bits of the FP64 transcendentals (CUDA libdevice vs glibc), so the
// many-edge configs always take their pair predictions from this file.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../include/pmx.h"

namespace {

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hkey(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0, uint64_t d = 0) {
  uint64_t h = mix(seed ^ 0x51ed270b6f1f4f21ull);
  h = mix(h ^ a);
  h = mix(h ^ b);
  h = mix(h ^ c);
  h = mix(h ^ d);
  return h;
}
__device__ __forceinline__ double u01(uint64_t h) { return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
__device__ __forceinline__ double gauss(uint64_t h) {
  const double u1 = u01(h);
  const double u2 = u01(mix(h ^ 0xa0761d6478bd642full));
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
__device__ __forceinline__ void gauss2(uint64_t h, double* z0, double* z1) {
  const double u1 = u01(h);
  const double u2 = u01(mix(h ^ 0xa0761d6478bd642full));
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincos(6.283185307179586 * u2, &s, &c);
  *z0 = r * c;
  *z1 = r * s;
}

enum Stream : uint64_t { kQ = 1, kPointNoise = 2, kDescBase = 3, kDescNoise = 4 };
constexpr int kMaxDim = 32;

struct Scene {
  uint64_t seed;
  double f, cx, cy;
  int H, W, dim;
  double point_sigma, desc_sigma;
  int noise_mode;
};

Scene to_scene(const double* p) {
  Scene s;
  s.seed = (uint64_t)p[0];
  s.f = p[3];
  s.cx = p[4];
  s.cy = p[5];
  s.H = (int)p[6];
  s.W = (int)p[7];
  s.dim = (int)p[8];
  s.point_sigma = p[9];
  s.desc_sigma = p[10];
  s.noise_mode = (int)p[11];
  return s;
}

__device__ __forceinline__ void apply(const pmx_sim3& T, const double x[3], double y[3]) {
  for (int r = 0; r < 3; ++r) y[r] = T.s * (T.R[3 * r] * x[0] + T.R[3 * r + 1] * x[1] + T.R[3 * r + 2] * x[2]) + T.t[r];
}
__device__ __forceinline__ void apply_inv(const pmx_sim3& T, const double x[3], double y[3]) {
  const double d[3] = {x[0] - T.t[0], x[1] - T.t[1], x[2] - T.t[2]};
  for (int r = 0; r < 3; ++r) y[r] = (T.R[r] * d[0] + T.R[3 + r] * d[1] + T.R[6 + r] * d[2]) / T.s;
}

// gen_express: camera k's world points in the frame of T_frame + noise (salt).
__global__ void k_express(Scene s, int64_t image_id, pmx_sim3 Tk, pmx_sim3 Tf, uint64_t salt,
                          const double* __restrict__ P_in, const uint8_t* __restrict__ valid, float* X, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!valid[i]) {
    X[3 * i] = X[3 * i + 1] = X[3 * i + 2] = 0.0f;
    return;
  }
  const double P[3] = {P_in[3 * i], P_in[3 * i + 1], P_in[3 * i + 2]};
  double Xf[3];
  if (s.noise_mode == 0) {  // radial along camera k's own viewing ray (reference synth.cpp:221-226)
    double Xk[3], Pn[3];
    apply_inv(Tk, P, Xk);
    const double dk = sqrt(Xk[0] * Xk[0] + Xk[1] * Xk[1] + Xk[2] * Xk[2]);
    const double f =
        1.0 + s.point_sigma * gauss(hkey(s.seed, kPointNoise + 16 * salt, (uint64_t)image_id, (uint64_t)i, 7)) / dk;
    for (int c = 0; c < 3; ++c) Xk[c] *= f;
    apply(Tk, Xk, Pn);
    apply_inv(Tf, Pn, Xf);
  } else {
    apply_inv(Tf, P, Xf);
    for (int c = 0; c < 3; ++c)
      Xf[c] += s.point_sigma * gauss(hkey(s.seed, kPointNoise + 16 * salt, (uint64_t)image_id, (uint64_t)i, (uint64_t)c));
  }
  for (int c = 0; c < 3; ++c) X[3 * i + c] = (float)Xf[c];
}

__device__ void desc_base(const Scene& s, int64_t id_u, int64_t id_v, double* base) {
  double nrm = 0.0;
  for (int c = 0; c < s.dim; c += 2) {
    gauss2(hkey(s.seed, kDescBase, (uint64_t)id_u, (uint64_t)id_v, (uint64_t)c), &base[c], &base[c + 1]);
    nrm += base[c] * base[c] + base[c + 1] * base[c + 1];
  }
  nrm = sqrt(nrm);
  for (int c = 0; c < s.dim; ++c) base[c] /= nrm;
}

__device__ void desc_finish(const Scene& s, const double* base, uint64_t image, int64_t pixel, uint16_t* out) {
  double v[kMaxDim], n2 = 0.0;
  for (int c = 0; c < s.dim; c += 2) {
    double z0, z1;
    gauss2(hkey(s.seed, kDescNoise, image, (uint64_t)pixel, (uint64_t)c), &z0, &z1);
    v[c] = base[c] + s.desc_sigma * z0;
    v[c + 1] = base[c + 1] + s.desc_sigma * z1;
    n2 += v[c] * v[c] + v[c + 1] * v[c + 1];
  }
  n2 = sqrt(n2);
  for (int c = 0; c < s.dim; ++c) {
    const __half h = __float2half_rn((float)(v[c] / n2));
    out[c] = *reinterpret_cast<const uint16_t*>(&h);
  }
}

// gen_pair_desc: D_a[i] = h(a, pixel i) + noise, D_b[n] = h(a, round(K proj_a(P_b[n]))) + noise.
__global__ void k_pair_desc(Scene s, int64_t image_a, pmx_sim3 Ta, const uint8_t* __restrict__ valid_a, int64_t image_b,
                            const double* __restrict__ P_b, const uint8_t* __restrict__ valid_b, uint16_t* D_a,
                            uint16_t* D_b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t ns = (int64_t)1 << 24;  // id namespace per camera a
  double base[kMaxDim];
  const int u = i % s.W, v = i / s.W;
  if (valid_a[i])
    desc_base(s, u + ns * image_a, v, base);
  else
    desc_base(s, -1000000 - i + ns * image_a, -1000000, base);
  desc_finish(s, base, (uint64_t)image_a, i, D_a + (size_t)i * s.dim);
  int64_t iu = -2000000 - i, iv = -2000000;
  if (valid_b[i]) {
    double Xa[3];
    const double P[3] = {P_b[3 * i], P_b[3 * i + 1], P_b[3 * i + 2]};
    apply_inv(Ta, P, Xa);
    if (Xa[2] > 1e-9) {
      iu = (int64_t)llround(s.f * Xa[0] / Xa[2] + s.cx);
      iv = (int64_t)llround(s.f * Xa[1] / Xa[2] + s.cy);
    }
  }
  desc_base(s, iu + ns * image_a, iv, base);  // in-image ids are camera a's pixel ids
  desc_finish(s, base, (uint64_t)image_b, i, D_b + (size_t)i * s.dim);
}

}  // namespace

extern "C" {

/* Device twins of gen_express / gen_pair_desc (all arrays device memory,
 * enqueued on `stream`).  Returns 0 or the CUDA error code. */
int gen_cuda_express(const double* scene, int64_t image_id, const pmx_sim3* T_wk, const pmx_sim3* T_frame,
                     uint64_t salt, const double* P_in, const uint8_t* valid, float* X, void* stream) {
  const Scene s = to_scene(scene);
  const int n = s.H * s.W;
  k_express<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(s, image_id, *T_wk, *T_frame, salt, P_in, valid, X, n);
  return (int)cudaGetLastError();
}

int gen_cuda_pair_desc(const double* scene, int64_t image_a, const pmx_sim3* T_wa, const uint8_t* valid_a,
                       int64_t image_b, const double* P_b, const uint8_t* valid_b, uint16_t* D_a, uint16_t* D_b,
                       void* stream) {
  const Scene s = to_scene(scene);
  if (s.dim > kMaxDim || (s.dim & 1)) return (int)cudaErrorInvalidValue;
  const int n = s.H * s.W;
  k_pair_desc<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(s, image_a, *T_wa, valid_a, image_b, P_b, valid_b, D_a,
                                                                 D_b, n);
  return (int)cudaGetLastError();
}

}  // extern "C"
