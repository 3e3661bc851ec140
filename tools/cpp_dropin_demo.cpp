// C++ drop-in demo: the reference-shaped API of include/pmslam_b200.hpp used
// exactly as pmslam's own tests use theirs (test_camera.cpp:119-132 self-pair
// identity, test_tracking.cpp:200-223 exact Sim(3) recovery,
// test_backend.cpp:241-264 consistent-graph fixed point).  Exit code = number
// of failed checks.  Build: see tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "pmslam_b200.hpp"

using namespace pmslam_b200;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static uint16_t to_half(float f) {  // round-to-nearest (test data only)
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t s = (x >> 16) & 0x8000;
  const int e = (int)((x >> 23) & 0xff) - 112;
  if (e <= 0) return (uint16_t)s;
  return (uint16_t)(s | (e << 10) | ((x >> 13) & 0x3ff));
}

static Pointmap plane(int h, int w) {  // wavy surface seen by a pinhole camera
  Pointmap pm(h, w);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const double x = (u - 0.5 * w) / (0.8 * w), y = (v - 0.5 * h) / (0.8 * w);
      const double z = 2.0 + 0.2 * std::sin(3 * x) * std::cos(2 * y);
      float* p = &pm.xyz[3 * (size_t)pm.index(u, v)];
      p[0] = (float)(z * x);
      p[1] = (float)(z * y);
      p[2] = (float)z;
    }
  return pm;
}

static FeatureMap features(int h, int w, int dim, unsigned seed) {
  FeatureMap f;
  f.height = h;
  f.width = w;
  f.dim = dim;
  f.descriptors.resize((size_t)h * w * dim);
  f.match_confidence.assign((size_t)h * w, 1.0f);
  std::mt19937 rng(seed);
  std::normal_distribution<float> n(0.f, 1.f);
  for (int i = 0; i < h * w; ++i) {
    std::vector<float> d(dim);
    float s = 0;
    for (auto& x : d) {
      x = n(rng);
      s += x * x;
    }
    for (int k = 0; k < dim; ++k) f.descriptors[(size_t)i * dim + k] = to_half(d[k] / std::sqrt(s));
  }
  return f;
}

static Sim3Pose make_pose(double ax, double ay, double az, double tx, double ty, double tz, double s) {
  const double th = std::sqrt(ax * ax + ay * ay + az * az);
  const double kx = ax / th, ky = ay / th, kz = az / th, c = std::cos(th), sn = std::sin(th), C = 1 - c;
  Sim3Pose T;
  const double R[9] = {c + kx * kx * C,      kx * ky * C - kz * sn, kx * kz * C + ky * sn,
                       ky * kx * C + kz * sn, c + ky * ky * C,      ky * kz * C - kx * sn,
                       kz * kx * C - ky * sn, kz * ky * C + kx * sn, c + kz * kz * C};
  for (int i = 0; i < 9; ++i) T.R[i] = R[i];
  T.t[0] = tx;
  T.t[1] = ty;
  T.t[2] = tz;
  T.s = s;
  return T;
}

static void apply_inv(const Sim3Pose& T, const float* x, float* y) {
  const double d[3] = {x[0] - T.t[0], x[1] - T.t[1], x[2] - T.t[2]};
  for (int r = 0; r < 3; ++r) y[r] = (float)((T.R[r] * d[0] + T.R[3 + r] * d[1] + T.R[6 + r] * d[2]) / T.s);
}

int main() {
  const int h = 48, w = 64, n = h * w;
  Context ctx(0);
  // camera.hpp: self pair with identity init is the identity (test_camera.cpp:119-132)
  const Pointmap X = plane(h, w);
  const FeatureMap F = features(h, w, 24, 1);
  MatchSet m = match_pointmaps(ctx, X, X, F, F);
  int ident = 0;
  for (const auto& mm : m.matches) ident += (mm.valid && mm.pixel_a == mm.pixel_b);
  CHECK(ident == n);
  MatchSet r = feature_refine(ctx, m, F, F);
  int moved = 0;
  for (int k = 0; k < n; ++k) moved += r.matches[k].pixel_a != m.matches[k].pixel_a;
  CHECK(moved == 0);
  // contract violation -> std::invalid_argument, as in the reference
  bool threw = false;
  try {
    FeatureMap bad = F;
    bad.dim = 16;
    match_pointmaps(ctx, X, X, F, bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // retrieval.hpp: a self pair agrees in appearance everywhere -> accepted,
  // all matches kept; omega_l above 1 can never be met -> nullopt
  const auto edge = accept_loop_edge(ctx, 3, 7, X, X, F, F, 0.9);
  CHECK(edge.has_value() && edge->i == 3 && edge->j == 7 && edge->matches.valid_count() == n);
  CHECK(!accept_loop_edge(ctx, 3, 7, X, X, F, F, 1.01).has_value());
  // pipeline.cpp: constrain_to_rays puts points back on their pixel rays
  Pointmap Xc = X;
  const pmx_intrinsics Kc{50.0, 50.0, 32.0, 24.0};
  constrain_to_rays(ctx, Xc, Kc);
  const int pc = Xc.index(10, 20);
  CHECK(std::fabs(Xc.xyz[3 * pc] - (float)(Xc.xyz[3 * pc + 2] * ((10 - 32.0) / 50.0))) < 1e-6f);

  // tracking.hpp: exact Sim(3) recovery with scale (test_tracking.cpp:200-223)
  const Sim3Pose T_true = make_pose(0.1, -0.08, 0.12, 0.08, -0.12, 0.05, 1.3);
  Keyframe kf;
  kf.canonical = X;
  kf.canonical_confidence.assign(n, 1.0f);
  FramePrediction pred;
  pred.X_f_f = Pointmap(h, w);
  for (int i = 0; i < n; ++i) apply_inv(T_true, &X.xyz[3 * (size_t)i], &pred.X_f_f.xyz[3 * (size_t)i]);
  pred.X_k_f = pred.X_f_f;
  pred.F_f = F;
  pred.F_k = F;
  const TrackResult tr = solve_pose(ctx, kf, pred, identity_pose(), PMX_TRACK_RAY);
  CHECK(!tr.lost);
  double et = 0;
  for (int i = 0; i < 3; ++i) et = std::max(et, std::fabs(tr.T_kf.t[i] - T_true.t[i]));
  CHECK(et < 1e-4);
  CHECK(std::fabs(tr.T_kf.s / T_true.s - 1) < 1e-5);
  for (size_t i = 1; i < tr.cost_trace.size(); ++i)
    CHECK(tr.cost_trace[i] <= tr.cost_trace[i - 1] * (1 + 1e-12) + 1e-300);
  // fusion: first observation is exact
  Keyframe fk;
  fk.canonical = Pointmap(h, w);
  fk.canonical.valid.assign(n, 0);
  fk.canonical_confidence.assign(n, 0.0f);
  fuse_canonical(ctx, fk, X, std::vector<float>(n, 1.0f), identity_pose());
  double fe = 0;
  for (size_t i = 0; i < X.xyz.size(); ++i) fe = std::max(fe, (double)std::fabs(fk.canonical.xyz[i] - X.xyz[i]));
  CHECK(fe == 0.0);

  // backend.hpp: consistent graph is a fixed point, anchor bit-identical (test_backend.cpp:241-264)
  Graph g;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<float> world(3 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    world[3 * i] = (float)(2 * U(rng));
    world[3 * i + 1] = (float)(2 * U(rng));
    world[3 * i + 2] = (float)(4 + 1.5 * U(rng));
  }
  for (int k = 0; k < 4; ++k) {
    Keyframe K;
    K.T_WC = make_pose(0.01, 0.05 * k + 0.01, 0.02 * k, 0.1 * k, 0.0, 0.02 * k, 1.0);
    K.canonical = Pointmap(h, w);
    for (int i = 0; i < n; ++i) apply_inv(K.T_WC, &world[3 * (size_t)i], &K.canonical.xyz[3 * (size_t)i]);
    K.canonical_confidence.assign(n, 1.0f);
    g.keyframes.push_back(K);
    if (k > 0) {
      Edge e;
      e.i = k - 1;
      e.j = k;
      for (int i = 0; i < n; ++i) e.matches.matches.push_back({i, i, 1.0, true});
      g.edges.push_back(e);
    }
  }
  g.anchor = 0;
  const Sim3Pose anchor = g.keyframes[0].T_WC;
  std::vector<Sim3Pose> before;
  for (const auto& k : g.keyframes) before.push_back(k.T_WC);
  const OptimizeResult res = global_optimize(ctx, g);
  CHECK(res.converged);
  CHECK(std::memcmp(&anchor, &g.keyframes[0].T_WC, sizeof(Sim3Pose)) == 0);
  for (size_t k = 0; k < before.size(); ++k)
    for (int i = 0; i < 3; ++i) CHECK(std::fabs(g.keyframes[k].T_WC.t[i] - before[k].t[i]) < 1e-5);
  std::printf("%s (%d failed checks)\n", failures ? "FAILED" : "PASSED", failures);
  return failures;
}
