// Synthetic BASELINE-config generator (bench / test infrastructure, not the
// product).  Deterministic and library-independent: every random value is a
// counter-based splitmix64 hash of (seed, stream, indices) followed by an
// explicit Box-Muller, so the same inputs are produced on any host and in any
// thread order.  Outputs are exactly what the reference consumes: fp32
// pointmaps (the PMPAIR01 stream precision, reference src/pipeline.cpp:532-543),
// fp32 confidences and fp16 descriptors.
//
// World: the surface of BASELINE config 0, z(x, y) = 2 + 0.3 sin(3x) cos(2y)
// + a x + b y over the normalised image coordinates (x, y) of a reference
// camera at the world origin; the surface point of parameter (x, y) is
// z(x, y) * (x, y, 1).  Every camera k (Sim(3) pose T_wk, camera -> world)
// ray-casts its pixels into that surface (Newton in FP64).  Descriptor
// identity of a surface point = its rounded reference-camera pixel, so the
// descriptor peak of a correspondence is the nearest ground-truth pixel.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../include/pmx.h"

namespace {

inline uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t hkey(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0, uint64_t d = 0) {
  uint64_t h = mix(seed ^ 0x51ed270b6f1f4f21ull);
  h = mix(h ^ a);
  h = mix(h ^ b);
  h = mix(h ^ c);
  h = mix(h ^ d);
  return h;
}
inline double u01(uint64_t h) { return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
inline double gauss(uint64_t h) {
  const double u1 = u01(h);
  const double u2 = u01(mix(h ^ 0xa0761d6478bd642full));
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

enum Stream : uint64_t {
  kQ = 1,
  kPointNoise = 2,
  kDescBase = 3,
  kDescNoise = 4,
};

uint16_t float_to_half(float f) {  // round to nearest even
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000;
  const int32_t exp = (int32_t)((x >> 23) & 0xff) - 127 + 15;
  uint32_t mant = x & 0x7fffff;
  if (((x >> 23) & 0xff) == 0xff) return (uint16_t)(sign | 0x7c00 | (mant ? 0x200 : 0));
  if (exp >= 31) return (uint16_t)(sign | 0x7c00);
  if (exp <= 0) {
    if (exp < -10) return (uint16_t)sign;
    mant |= 0x800000;
    const int shift = 14 - exp;
    uint32_t h = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) ++h;
    return (uint16_t)(sign | h);
  }
  uint32_t h = ((uint32_t)exp << 10) | (mant >> 13);
  const uint32_t rem = mant & 0x1fff;
  if (rem > 0x1000 || (rem == 0x1000 && (h & 1))) ++h;
  return (uint16_t)(sign | h);
}

struct Scene {
  uint64_t seed;
  double a, b;
  double f, cx, cy;
  int H, W, dim;
  double point_sigma, desc_sigma;
  int noise_mode;  // 0 = radial in the view's own frame (reference synth.cpp:221-226), 1 = isotropic
  int surface;     // 0 = depth map of the reference camera (config 0/1), 1 = world heightfield (configs 2-4)
};

inline double surf(const Scene& s, double x, double y, double* zx, double* zy) {
  const double sx = std::sin(3 * x), cx = std::cos(3 * x);
  const double sy = std::sin(2 * y), cy = std::cos(2 * y);
  if (zx) *zx = 0.9 * cx * cy + s.a;
  if (zy) *zy = -0.6 * sx * sy + s.b;
  return 2.0 + 0.3 * sx * cy + s.a * x + s.b * y;
}

// World heightfield Z = h(X, Y) (configs 2-4): the config-0 relief in
// coordinates normalised at the nominal depth 2, a proper graph everywhere.
inline double height(const Scene& s, double X, double Y, double* hx, double* hy) {
  const double x = 0.5 * X, y = 0.5 * Y;
  const double sx = std::sin(3 * x), cx = std::cos(3 * x), sy = std::sin(2 * y), cy = std::cos(2 * y);
  if (hx) *hx = 0.5 * (0.9 * cx * cy + s.a);
  if (hy) *hy = 0.5 * (-0.6 * sx * sy + s.b);
  return 2.0 + 0.3 * sx * cy + s.a * x + s.b * y;
}

bool cast_heightfield(const Scene& s, const double o[3], const double d[3], double P[3], double* px, double* py) {
  if (!(d[2] > 1e-9)) return false;
  double lam = (2.0 - o[2]) / d[2];
  for (int it = 0; it < 50; ++it) {
    double hx, hy;
    const double X = o[0] + lam * d[0], Y = o[1] + lam * d[1];
    const double F = o[2] + lam * d[2] - height(s, X, Y, &hx, &hy);
    const double dF = d[2] - hx * d[0] - hy * d[1];
    if (std::abs(dF) < 1e-12) return false;
    const double step = F / dF;
    lam -= step;
    if (std::abs(step) < 1e-14 * (1.0 + std::abs(lam))) break;
  }
  P[0] = o[0] + lam * d[0];
  P[1] = o[1] + lam * d[1];
  P[2] = o[2] + lam * d[2];
  const double F = P[2] - height(s, P[0], P[1], nullptr, nullptr);
  if (!(std::abs(F) < 1e-9) || !(lam > 0)) return false;
  *px = P[0] / P[2];
  *py = P[1] / P[2];
  return true;
}

// Ray cast o + lambda d into the surface.  Returns false when Newton fails.
bool cast(const Scene& s, const double o[3], const double d[3], double P[3], double* px, double* py) {
  if (s.surface == 1) return cast_heightfield(s, o, d, P, px, py);
  // Initial guess: plane Z = 2.
  if (std::abs(d[2]) < 1e-9) return false;
  double lam = (2.0 - o[2]) / d[2];
  double X = o[0] + lam * d[0], Y = o[1] + lam * d[1], Z = o[2] + lam * d[2];
  if (Z <= 1e-6) return false;
  double x = X / Z, y = Y / Z;
  for (int it = 0; it < 30; ++it) {
    double zx, zy;
    const double z = surf(s, x, y, &zx, &zy);
    const double F[3] = {z * x - o[0] - lam * d[0], z * y - o[1] - lam * d[1], z - o[2] - lam * d[2]};
    const double err = std::abs(F[0]) + std::abs(F[1]) + std::abs(F[2]);
    // J columns: d/dx, d/dy, d/dlam
    const double J[3][3] = {{zx * x + z, zy * x, -d[0]}, {zx * y, zy * y + z, -d[1]}, {zx, zy, -d[2]}};
    // solve J delta = -F (Cramer)
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (std::abs(det) < 1e-14) return false;
    double dl[3];
    for (int c = 0; c < 3; ++c) {
      double M[3][3];
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) M[r][k] = (k == c) ? -F[r] : J[r][k];
      dl[c] = (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
               M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
               M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0])) / det;
    }
    x += dl[0];
    y += dl[1];
    lam += dl[2];
    if (err < 1e-13 && std::abs(dl[0]) + std::abs(dl[1]) < 1e-14) break;
  }
  const double z = surf(s, x, y, nullptr, nullptr);
  P[0] = z * x;
  P[1] = z * y;
  P[2] = z;
  const double F = std::abs(P[0] - o[0] - lam * d[0]) + std::abs(P[1] - o[1] - lam * d[1]) +
                   std::abs(P[2] - o[2] - lam * d[2]);
  if (!(F < 1e-9) || !(lam > 0)) return false;
  *px = x;
  *py = y;
  return true;
}

inline void apply(const pmx_sim3& T, const double x[3], double y[3]) {
  for (int r = 0; r < 3; ++r)
    y[r] = T.s * (T.R[3 * r] * x[0] + T.R[3 * r + 1] * x[1] + T.R[3 * r + 2] * x[2]) + T.t[r];
}
inline void apply_inv(const pmx_sim3& T, const double x[3], double y[3]) {
  double d[3] = {x[0] - T.t[0], x[1] - T.t[1], x[2] - T.t[2]};
  for (int r = 0; r < 3; ++r)
    y[r] = (T.R[r] * d[0] + T.R[3 + r] * d[1] + T.R[6 + r] * d[2]) / T.s;
}

template <class F>
void parallel_rows(int H, int threads, F&& fn) {
  if (threads <= 1) {
    for (int v = 0; v < H; ++v) fn(v);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (int v = next++; v < H; v = next++) fn(v);
    });
  for (auto& th : pool) th.join();
}

// Two N(0,1) draws from one counter hash (both Box-Muller outputs).
inline void gauss2(uint64_t h, double* z0, double* z1) {
  const double u1 = u01(h);
  const double u2 = u01(mix(h ^ 0xa0761d6478bd642full));
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double t = 6.283185307179586 * u2;
  *z0 = r * std::cos(t);
  *z1 = r * std::sin(t);
}

// Unit base vector h(id) of a descriptor identity (dim even).
void desc_base(const Scene& s, int64_t id_u, int64_t id_v, double* base) {
  double nrm = 0.0;
  for (int c = 0; c < s.dim; c += 2) {
    gauss2(hkey(s.seed, kDescBase, (uint64_t)id_u, (uint64_t)id_v, (uint64_t)c), &base[c], &base[c + 1]);
    nrm += base[c] * base[c] + base[c + 1] * base[c + 1];
  }
  nrm = std::sqrt(nrm);
  for (int c = 0; c < s.dim; ++c) base[c] /= nrm;
}

// normalise(base + N(0, desc_sigma^2)) -> fp16, noise keyed by (image, pixel).
void desc_finish(const Scene& s, const double* base, uint64_t image, int64_t pixel, uint16_t* out) {
  double v[64], n2 = 0.0;
  for (int c = 0; c < s.dim; c += 2) {
    double z0, z1;
    gauss2(hkey(s.seed, kDescNoise, image, (uint64_t)pixel, (uint64_t)c), &z0, &z1);
    v[c] = base[c] + s.desc_sigma * z0;
    v[c + 1] = base[c + 1] + s.desc_sigma * z1;
    n2 += v[c] * v[c] + v[c + 1] * v[c + 1];
  }
  n2 = std::sqrt(n2);
  for (int c = 0; c < s.dim; ++c) out[c] = float_to_half((float)(v[c] / n2));
}

void descriptor(const Scene& s, int64_t id_u, int64_t id_v, uint64_t image, int64_t pixel, uint16_t* out) {
  double base[64];
  desc_base(s, id_u, id_v, base);
  desc_finish(s, base, image, pixel, out);
}

Scene to_scene(const double* p) {
  Scene s;
  s.seed = (uint64_t)p[0];
  s.a = p[1];
  s.b = p[2];
  s.f = p[3];
  s.cx = p[4];
  s.cy = p[5];
  s.H = (int)p[6];
  s.W = (int)p[7];
  s.dim = (int)p[8];
  s.point_sigma = p[9];
  s.desc_sigma = p[10];
  s.noise_mode = (int)p[11];
  s.surface = (int)p[12];
  return s;
}

}  // namespace

extern "C" {

/* Scene parameter vector (doubles): seed, tilt a, tilt b, f, cx, cy, H, W,
 * descriptor dim, point noise sigma, descriptor noise sigma, noise mode. */
#define GEN_SCENE_PARAMS 12

/* Render camera `image_id` with pose T_wk: world points of its pixel rays,
 * expressed in the frame of T_frame (points = T_frame^-1 P), plus N(0,
 * point_sigma^2) noise keyed by (salt, image, pixel).  Any output may be NULL.
 * surface_xy (double[HW*2], nullable) receives the surface parameter. */
int gen_image(const double* scene, int64_t image_id, const pmx_sim3* T_wk,
              const pmx_sim3* T_frame, uint64_t salt, float* X, uint8_t* valid, float* Q,
              uint16_t* D, double* surface_xy, int threads) {
  const Scene s = to_scene(scene);
  const pmx_sim3 Tk = *T_wk, Tf = *T_frame;
  parallel_rows(s.H, threads, [&](int v) {
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      const double dc[3] = {(u - s.cx) / s.f, (v - s.cy) / s.f, 1.0};
      double dw[3];
      for (int r = 0; r < 3; ++r) dw[r] = Tk.R[3 * r] * dc[0] + Tk.R[3 * r + 1] * dc[1] + Tk.R[3 * r + 2] * dc[2];
      double P[3], px = 0, py = 0;
      const bool ok = cast(s, Tk.t, dw, P, &px, &py);
      if (valid) valid[i] = ok ? 1 : 0;
      if (surface_xy) {
        surface_xy[2 * i] = ok ? px : NAN;
        surface_xy[2 * i + 1] = ok ? py : NAN;
      }
      if (X) {
        if (ok) {
          double Xf[3];
          if (s.noise_mode == 0) {
            // Radial: perturb the distance along camera k's own viewing ray by
            // N(0, sigma^2) (absolute), then re-express in the output frame.
            double Xk[3], Pn[3];
            apply_inv(Tk, P, Xk);
            const double dk = std::sqrt(Xk[0] * Xk[0] + Xk[1] * Xk[1] + Xk[2] * Xk[2]);
            const double f = 1.0 + s.point_sigma *
                                       gauss(hkey(s.seed, kPointNoise + 16 * salt, (uint64_t)image_id,
                                                  (uint64_t)i, 7)) / dk;
            for (int c = 0; c < 3; ++c) Xk[c] *= f;
            apply(Tk, Xk, Pn);
            apply_inv(Tf, Pn, Xf);
          } else {
            apply_inv(Tf, P, Xf);
            for (int c = 0; c < 3; ++c)
              Xf[c] += s.point_sigma * gauss(hkey(s.seed, kPointNoise + 16 * salt, (uint64_t)image_id,
                                                  (uint64_t)i, (uint64_t)c));
          }
          for (int c = 0; c < 3; ++c) X[3 * i + c] = (float)Xf[c];
        } else {
          X[3 * i] = X[3 * i + 1] = X[3 * i + 2] = 0.0f;
        }
      }
      if (Q) Q[i] = (float)(1.0 + 9.0 * u01(hkey(s.seed, kQ, (uint64_t)image_id, (uint64_t)i)));
      if (D) {
        int64_t iu = 0, iv = 0;
        if (ok) {
          iu = (int64_t)std::llround(s.f * px + s.cx);
          iv = (int64_t)std::llround(s.f * py + s.cy);
        } else {
          iu = -1000000 - i;
          iv = -1000000;
        }
        descriptor(s, iu, iv, (uint64_t)image_id, i, D + (size_t)i * s.dim);
      }
    }
  });
  return 0;
}

/* Two-step form of gen_image for many edges over few cameras: gen_camera
 * ray-casts camera k once (world points P double[HW*3], valid, Q, D);
 * gen_express re-expresses them in any frame with per-prediction noise (salt).
 * gen_image(...) == gen_camera + gen_express, bit for bit. */
int gen_camera(const double* scene, int64_t image_id, const pmx_sim3* T_wk, double* P_out, uint8_t* valid,
               float* Q, uint16_t* D, int threads) {
  const Scene s = to_scene(scene);
  const pmx_sim3 Tk = *T_wk;
  parallel_rows(s.H, threads, [&](int v) {
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      const double dc[3] = {(u - s.cx) / s.f, (v - s.cy) / s.f, 1.0};
      double dw[3];
      for (int r = 0; r < 3; ++r) dw[r] = Tk.R[3 * r] * dc[0] + Tk.R[3 * r + 1] * dc[1] + Tk.R[3 * r + 2] * dc[2];
      double P[3] = {0, 0, 0}, px = 0, py = 0;
      const bool ok = cast(s, Tk.t, dw, P, &px, &py);
      valid[i] = ok ? 1 : 0;
      for (int c = 0; c < 3; ++c) P_out[3 * i + c] = ok ? P[c] : 0.0;
      if (Q) Q[i] = (float)(1.0 + 9.0 * u01(hkey(s.seed, kQ, (uint64_t)image_id, (uint64_t)i)));
      if (D) {
        int64_t iu, iv;
        if (ok) {
          iu = (int64_t)std::llround(s.f * px + s.cx);
          iv = (int64_t)std::llround(s.f * py + s.cy);
        } else {
          iu = -1000000 - i;
          iv = -1000000;
        }
        descriptor(s, iu, iv, (uint64_t)image_id, i, D + (size_t)i * s.dim);
      }
    }
  });
  return 0;
}

int gen_express(const double* scene, int64_t image_id, const pmx_sim3* T_wk, const pmx_sim3* T_frame,
                uint64_t salt, const double* P_in, const uint8_t* valid, float* X, int threads) {
  const Scene s = to_scene(scene);
  const pmx_sim3 Tk = *T_wk, Tf = *T_frame;
  parallel_rows(s.H, threads, [&](int v) {
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      if (!valid[i]) {
        X[3 * i] = X[3 * i + 1] = X[3 * i + 2] = 0.0f;
        continue;
      }
      const double* P = P_in + 3 * i;
      double Xf[3];
      if (s.noise_mode == 0) {
        double Xk[3], Pn[3];
        apply_inv(Tk, P, Xk);
        const double dk = std::sqrt(Xk[0] * Xk[0] + Xk[1] * Xk[1] + Xk[2] * Xk[2]);
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
  });
  return 0;
}

/* Pair-predicted descriptors of edge (a, b) (MASt3R predicts D_i, D_j per
 * pair): the identity of a surface point is its rounded pixel in camera a's
 * grid (config 0: camera i), so the descriptor peak of a correspondence is
 * the nearest camera-a pixel.  D_a[i] = h(a, u_i, v_i) + noise; D_b[n] =
 * h(a, round(K proj_a(P_b[n]))) + noise; h = hash-seeded unit vector. */
int gen_pair_desc(const double* scene, int64_t image_a, const pmx_sim3* T_wa, const uint8_t* valid_a,
                  int64_t image_b, const double* P_b, const uint8_t* valid_b, uint16_t* D_a, uint16_t* D_b,
                  int threads) {
  const Scene s = to_scene(scene);
  const pmx_sim3 Ta = *T_wa;
  const int64_t ns = (int64_t)1 << 24;  // id namespace per camera a
  // base vectors of camera a's pixel grid, shared by D_a and the in-image ids of D_b
  std::vector<double> grid((size_t)s.H * s.W * s.dim);
  parallel_rows(s.H, threads, [&](int v) {
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      desc_base(s, u + ns * image_a, v, grid.data() + (size_t)i * s.dim);
    }
  });
  parallel_rows(s.H, threads, [&](int v) {
    double base[64];
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      if (valid_a[i]) {
        desc_finish(s, grid.data() + (size_t)i * s.dim, (uint64_t)image_a, i, D_a + (size_t)i * s.dim);
      } else {
        desc_base(s, -1000000 - i + ns * image_a, -1000000, base);
        desc_finish(s, base, (uint64_t)image_a, i, D_a + (size_t)i * s.dim);
      }
      int64_t iu = -2000000 - i, iv = -2000000;
      if (valid_b[i]) {
        double Xa[3];
        apply_inv(Ta, P_b + 3 * i, Xa);
        if (Xa[2] > 1e-9) {
          iu = (int64_t)std::llround(s.f * Xa[0] / Xa[2] + s.cx);
          iv = (int64_t)std::llround(s.f * Xa[1] / Xa[2] + s.cy);
        }
      }
      const double* b;
      if (iu >= 0 && iv >= 0 && iu < s.W && iv < s.H) {
        b = grid.data() + (size_t)(iv * s.W + iu) * s.dim;
      } else {
        desc_base(s, iu + ns * image_a, iv, base);
        b = base;
      }
      desc_finish(s, b, (uint64_t)image_b, i, D_b + (size_t)i * s.dim);
    }
  });
  return 0;
}

/* Ground-truth matches of edge (a, b) from cached world points of camera b:
 * pixel_a = rounded projection into camera a (-1 outside / behind),
 * q = sqrt(Q_a[pixel_a] Q_b[n]). */
int gen_gt_from_points(const double* scene, const pmx_sim3* T_wa, const double* P_b, const uint8_t* valid_b,
                       const float* Q_a, const float* Q_b, int32_t* pixel_a, float* confidence, uint8_t* valid,
                       int threads) {
  const Scene s = to_scene(scene);
  const pmx_sim3 Ta = *T_wa;
  parallel_rows(s.H, threads, [&](int v) {
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      int32_t pa = -1;
      if (valid_b[i]) {
        double Xa[3];
        apply_inv(Ta, P_b + 3 * i, Xa);
        if (Xa[2] > 1e-9) {
          const long ru = std::lround(s.f * Xa[0] / Xa[2] + s.cx), rv = std::lround(s.f * Xa[1] / Xa[2] + s.cy);
          if (ru >= 0 && rv >= 0 && ru < s.W && rv < s.H) pa = (int32_t)(rv * s.W + ru);
        }
      }
      pixel_a[i] = pa;
      valid[i] = pa >= 0 ? 1 : 0;
      confidence[i] = pa >= 0 ? (float)std::sqrt((double)Q_a[pa] * (double)Q_b[i]) : 0.0f;
    }
  });
  return 0;
}

/* Ground-truth correspondences of edge (a, b): for every pixel n of camera b,
 * its surface point projected into camera a, rounded (pixel_a, -1 when it
 * falls outside the image or behind the camera).  q = sqrt(Q_a Q_b). */
int gen_gt_matches(const double* scene, int64_t image_a, const pmx_sim3* T_wa, int64_t image_b,
                   const pmx_sim3* T_wb, int32_t* pixel_a, float* confidence, uint8_t* valid,
                   double* subpixel, int threads) {
  const Scene s = to_scene(scene);
  const pmx_sim3 Ta = *T_wa, Tb = *T_wb;
  parallel_rows(s.H, threads, [&](int v) {
    for (int u = 0; u < s.W; ++u) {
      const int64_t i = (int64_t)v * s.W + u;
      const double dc[3] = {(u - s.cx) / s.f, (v - s.cy) / s.f, 1.0};
      double dw[3];
      for (int r = 0; r < 3; ++r) dw[r] = Tb.R[3 * r] * dc[0] + Tb.R[3 * r + 1] * dc[1] + Tb.R[3 * r + 2] * dc[2];
      double P[3], px, py;
      bool ok = cast(s, Tb.t, dw, P, &px, &py);
      int32_t pa = -1;
      double fu = NAN, fv = NAN;
      if (ok) {
        double Xa[3];
        apply_inv(Ta, P, Xa);
        if (Xa[2] > 1e-9) {
          fu = s.f * Xa[0] / Xa[2] + s.cx;
          fv = s.f * Xa[1] / Xa[2] + s.cy;
          const long ru = std::lround(fu), rv = std::lround(fv);
          if (ru >= 0 && rv >= 0 && ru < s.W && rv < s.H) pa = (int32_t)(rv * s.W + ru);
        }
      }
      pixel_a[i] = pa;
      if (subpixel) {
        subpixel[2 * i] = fu;
        subpixel[2 * i + 1] = fv;
      }
      if (valid) valid[i] = pa >= 0 ? 1 : 0;
      if (confidence) {
        if (pa >= 0) {
          const double qa = (float)(1.0 + 9.0 * u01(hkey(s.seed, kQ, (uint64_t)image_a, (uint64_t)pa)));
          const double qb = (float)(1.0 + 9.0 * u01(hkey(s.seed, kQ, (uint64_t)image_b, (uint64_t)i)));
          confidence[i] = (float)std::sqrt(qa * qb);
        } else {
          confidence[i] = 0.0f;
        }
      }
    }
  });
  return 0;
}

/* Counter-based uniforms / gaussians for Python-side draws (poses, outliers). */
void gen_uniform(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = u01(hkey(seed, 1000 + stream, (uint64_t)i));
}
void gen_gauss(uint64_t seed, uint64_t stream, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = gauss(hkey(seed, 1000 + stream, (uint64_t)i));
}
void gen_float_to_half(const float* in, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = float_to_half(in[i]);
}

}  // extern "C"
