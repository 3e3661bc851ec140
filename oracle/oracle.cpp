// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).  FP64 restatement of
// /root/reference/proj/src/{lie,camera,tracking,backend}.cpp; each function
// cites the reference line range it follows.
#include "oracle.hpp"

#include <algorithm>
#include <cfloat>
#include <limits>
#include <map>
#include <stdexcept>
#include <unordered_set>

namespace orc {

// ------------------------------------------------------------ linear algebra
Mat3 operator*(const Mat3& a, const Mat3& b) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(i, 0) * b(0, j) + a(i, 1) * b(1, j) + a(i, 2) * b(2, j);
  return r;
}
Vec3 operator*(const Mat3& a, const Vec3& x) {
  return {a(0, 0) * x[0] + a(0, 1) * x[1] + a(0, 2) * x[2],
          a(1, 0) * x[0] + a(1, 1) * x[1] + a(1, 2) * x[2],
          a(2, 0) * x[0] + a(2, 1) * x[1] + a(2, 2) * x[2]};
}
Mat3 operator+(const Mat3& a, const Mat3& b) {
  Mat3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = a.m[i] + b.m[i];
  return r;
}
Mat3 operator*(double s, const Mat3& a) {
  Mat3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = s * a.m[i];
  return r;
}
Mat3 transpose(const Mat3& a) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(j, i);
  return r;
}

// Eigen's LDLT<Matrix, Lower>: unblocked LDL^T with symmetric pivoting on the
// largest remaining |diagonal|; solve with the pseudo-inverse of D
// (|D_i| <= numeric_limits<double>::min() -> 0).  Restated from the published
// algorithm (Eigen/src/Cholesky/LDLT.h); used by camera.cpp:147 (2x2) and
// tracking.cpp:203 (7x7).
void ldlt_pivoted_solve(int n, const double* A_in, const double* b, double* x) {
  double mat[49];
  for (int i = 0; i < n * n; ++i) mat[i] = A_in[i];
  auto M = [&](int r, int c) -> double& { return mat[r * n + c]; };
  int transp[7];
  double temp[7];
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bigv = std::abs(M(k, k));
    for (int i = k + 1; i < n; ++i) {
      if (std::abs(M(i, i)) > bigv) {
        bigv = std::abs(M(i, i));
        big = i;
      }
    }
    transp[k] = big;
    if (k != big) {
      // swap within the lower triangle only
      for (int c = 0; c < k; ++c) std::swap(M(k, c), M(big, c));
      for (int r = big + 1; r < n; ++r) std::swap(M(r, k), M(r, big));
      std::swap(M(k, k), M(big, big));
      for (int i = k + 1; i < big; ++i) {
        double tmp = M(i, k);
        M(i, k) = M(big, i);
        M(big, i) = tmp;
      }
    }
    const int rs = n - k - 1;
    if (k > 0) {
      for (int c = 0; c < k; ++c) temp[c] = M(c, c) * M(k, c);
      double acc = 0.0;
      for (int c = 0; c < k; ++c) acc += M(k, c) * temp[c];
      M(k, k) -= acc;
      for (int r = k + 1; r < n; ++r) {
        double a = 0.0;
        for (int c = 0; c < k; ++c) a += M(r, c) * temp[c];
        M(r, k) -= a;
      }
    }
    const double akk = M(k, k);
    const bool pivot_ok = std::abs(akk) > 0.0;
    if (k == 0 && !pivot_ok) {
      for (int i = 0; i < n; ++i) x[i] = 0.0;  // entire diagonal zero: D = 0
      return;
    }
    if (rs > 0 && pivot_ok)
      for (int r = k + 1; r < n; ++r) M(r, k) /= akk;
  }
  // dst = P b
  double d[7];
  for (int i = 0; i < n; ++i) d[i] = b[i];
  for (int k = 0; k < n; ++k) std::swap(d[k], d[transp[k]]);
  // L^-1 (unit lower)
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < i; ++c) d[i] -= M(i, c) * d[c];
  const double tol = std::numeric_limits<double>::min();
  for (int i = 0; i < n; ++i) {
    if (std::abs(M(i, i)) > tol)
      d[i] /= M(i, i);
    else
      d[i] = 0.0;
  }
  // L^-T
  for (int i = n - 1; i >= 0; --i)
    for (int r = i + 1; r < n; ++r) d[i] -= M(r, i) * d[r];
  // P^T
  for (int k = n - 1; k >= 0; --k) std::swap(d[k], d[transp[k]]);
  for (int i = 0; i < n; ++i) x[i] = d[i];
}

// ------------------------------------------------------------------- lie.cpp
Mat3 skew(const Vec3& v) {  // lie.cpp:13-21
  Mat3 s;
  s(0, 1) = -v[2];
  s(0, 2) = v[1];
  s(1, 0) = v[2];
  s(1, 2) = -v[0];
  s(2, 0) = -v[1];
  s(2, 1) = v[0];
  return s;
}

Mat3 so3_exp(const Vec3& omega) {  // lie.cpp:23-32
  const double theta = norm(omega);
  const Mat3 O = skew(omega);
  const Mat3 O2 = O * O;
  if (theta < kSmallAngle) return Mat3::identity() + O + 0.5 * O2;
  const double theta_sq = theta * theta;
  return Mat3::identity() + (std::sin(theta) / theta) * O + ((1.0 - std::cos(theta)) / theta_sq) * O2;
}

Vec3 so3_log(const Mat3& R) {  // lie.cpp:34-49
  const double tr = R(0, 0) + R(1, 1) + R(2, 2);
  const double cos_angle = std::clamp(0.5 * (tr - 1.0), -1.0, 1.0);
  const double angle = std::acos(cos_angle);
  const Vec3 axis(R(2, 1) - R(1, 2), R(0, 2) - R(2, 0), R(1, 0) - R(0, 1));
  if (angle < kSmallAngle) return 0.5 * axis;
  if (angle > M_PI - 1e-6) throw std::domain_error("so3_log: rotation angle at pi is degenerate");
  return (0.5 * angle / std::sin(angle)) * axis;
}

Mat3 sim3_w_matrix(const Vec3& omega, double sigma) {  // lie.cpp:51-90
  const double theta = norm(omega);
  const double scale = std::exp(sigma);
  const Mat3 O = skew(omega);
  double A, B, C;
  if (std::abs(sigma) < kSmallAngle) {
    C = 1.0 + 0.5 * sigma + sigma * sigma / 6.0;
    if (theta < kSmallAngle) {
      A = 0.5 + sigma / 3.0;
      B = 1.0 / 6.0 + sigma / 8.0;
    } else {
      const double theta_sq = theta * theta;
      const double denom = sigma * sigma + theta_sq;
      A = (scale * (sigma * std::sin(theta) - theta * std::cos(theta)) + theta) / (theta * denom);
      B = (C - (scale * (sigma * std::cos(theta) + theta * std::sin(theta)) - sigma) / denom) / theta_sq;
    }
  } else {
    C = (scale - 1.0) / sigma;
    if (theta < kSmallAngle) {
      const double sigma_sq = sigma * sigma;
      A = (scale * (sigma - 1.0) + 1.0) / sigma_sq;
      B = (scale * (sigma_sq - 2.0 * sigma + 2.0) - 2.0) / (2.0 * sigma_sq * sigma);
    } else {
      const double theta_sq = theta * theta;
      const double denom = sigma * sigma + theta_sq;
      A = (scale * (sigma * std::sin(theta) - theta * std::cos(theta)) + theta) / (theta * denom);
      B = (C - (scale * (sigma * std::cos(theta) + theta * std::sin(theta)) - sigma) / denom) / theta_sq;
    }
  }
  return C * Mat3::identity() + A * O + B * (O * O);
}

Sim3 Sim3::exp(const Vec7& tau) {  // lie.cpp:99-108
  const Vec3 rho(tau[0], tau[1], tau[2]);
  const Vec3 omega(tau[3], tau[4], tau[5]);
  const double sigma = tau[6];
  Sim3 r;
  r.R = so3_exp(omega);
  r.s = std::exp(sigma);
  r.t = sim3_w_matrix(omega, sigma) * rho;
  return r;
}

static Vec3 solve3(const Mat3& W, const Vec3& b) {
  // partial-pivot LU (lie.cpp:115 uses partialPivLu)
  double a[3][4];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) a[i][j] = W(i, j);
    a[i][3] = b[i];
  }
  for (int k = 0; k < 3; ++k) {
    int p = k;
    for (int i = k + 1; i < 3; ++i)
      if (std::abs(a[i][k]) > std::abs(a[p][k])) p = i;
    for (int j = 0; j < 4; ++j) std::swap(a[k][j], a[p][j]);
    for (int i = k + 1; i < 3; ++i) {
      const double f = a[i][k] / a[k][k];
      for (int j = k; j < 4; ++j) a[i][j] -= f * a[k][j];
    }
  }
  Vec3 x;
  for (int i = 2; i >= 0; --i) {
    double s = a[i][3];
    for (int j = i + 1; j < 3; ++j) s -= a[i][j] * x[j];
    x[i] = s / a[i][i];
  }
  return x;
}

Vec7 Sim3::log() const {  // lie.cpp:110-119
  const Vec3 omega = so3_log(R);
  const double sigma = std::log(s);
  const Mat3 W = sim3_w_matrix(omega, sigma);
  const Vec3 rho = solve3(W, t);
  return {rho[0], rho[1], rho[2], omega[0], omega[1], omega[2], sigma};
}

Sim3 Sim3::inverse() const {  // lie.cpp:121-129
  Sim3 r;
  r.R = transpose(R);
  r.s = 1.0 / s;
  r.t = -r.s * (r.R * t);
  r.ops_since_renorm = ops_since_renorm + 1;
  r.renormalize_if_needed();
  return r;
}

Sim3 Sim3::operator*(const Sim3& o) const {  // lie.cpp:131-140
  Sim3 r;
  r.R = R * o.R;
  r.s = s * o.s;
  r.t = s * (R * o.t) + t;
  r.ops_since_renorm = std::max(ops_since_renorm, o.ops_since_renorm) + 1;
  r.renormalize_if_needed();
  return r;
}

void Sim3::renormalize_if_needed() {  // lie.cpp:142-153
  if (ops_since_renorm < 100) return;
  // Polar factor U V^T of R via Newton iteration X <- (X + X^-T)/2 (equal to
  // the JacobiSVD construction for det > 0, which holds for rotations).
  Mat3 X = R;
  for (int it = 0; it < 30; ++it) {
    const Mat3& a = X;
    const double det = a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) -
                       a(0, 1) * (a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) +
                       a(0, 2) * (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0));
    Mat3 cof;  // inverse transpose = cofactor / det
    cof(0, 0) = (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) / det;
    cof(0, 1) = -(a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) / det;
    cof(0, 2) = (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0)) / det;
    cof(1, 0) = -(a(0, 1) * a(2, 2) - a(0, 2) * a(2, 1)) / det;
    cof(1, 1) = (a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0)) / det;
    cof(1, 2) = -(a(0, 0) * a(2, 1) - a(0, 1) * a(2, 0)) / det;
    cof(2, 0) = (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1)) / det;
    cof(2, 1) = -(a(0, 0) * a(1, 2) - a(0, 2) * a(1, 0)) / det;
    cof(2, 2) = (a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0)) / det;
    X = 0.5 * (X + cof);
  }
  R = X;
  ops_since_renorm = 0;
}

Mat7 Sim3::adjoint() const {  // lie.cpp:155-163
  Mat7 ad{};
  const Mat3 tR = skew(t) * R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      ad[r * 7 + c] = s * R(r, c);
      ad[r * 7 + 3 + c] = tR(r, c);
      ad[(3 + r) * 7 + 3 + c] = R(r, c);
    }
  for (int r = 0; r < 3; ++r) ad[r * 7 + 6] = -t[r];
  ad[6 * 7 + 6] = 1.0;
  return ad;
}

Sim3 relative_pose(const Sim3& T_wi, const Sim3& T_wj) { return T_wi.inverse() * T_wj; }

// ---------------------------------------------------------------- camera.cpp
int MatchSet::valid_count() const {  // camera.cpp:10-14
  int n = 0;
  for (const auto& m : matches) n += m.valid ? 1 : 0;
  return n;
}
double MatchSet::valid_fraction() const {  // camera.cpp:16-19
  if (matches.empty()) return 0.0;
  return (double)valid_count() / (double)matches.size();
}
double MatchSet::unique_pixel_fraction(int num_pixels_a) const {  // camera.cpp:21-28
  if (num_pixels_a <= 0) return 0.0;
  std::unordered_set<int> hit;
  for (const auto& m : matches)
    if (m.valid) hit.insert(m.pixel_a);
  return (double)hit.size() / (double)num_pixels_a;
}
MatchSet MatchSet::identity(int n, double confidence) {  // camera.cpp:30-37
  MatchSet s;
  s.matches.resize(n);
  for (int i = 0; i < n; ++i) s.matches[i] = {i, i, confidence, true};
  return s;
}

RayMap normalize_rays(const Pointmap& pm) {  // camera.cpp:39-56
  RayMap rm;
  rm.height = pm.height;
  rm.width = pm.width;
  const int n = pm.size();
  rm.rays.assign(n, Vec3(0, 0, 1));
  rm.distances.assign(n, 1.0);
  rm.valid.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    if (!pm.valid[i]) continue;
    const double nrm = norm(pm.points[i]);
    if (nrm < 1e-12 || !std::isfinite(nrm)) continue;
    rm.rays[i] = pm.points[i] / nrm;
    rm.distances[i] = nrm;
    rm.valid[i] = 1;
  }
  return rm;
}

bool interpolate_ray(const RayMap& rays, double u, double v, Vec3* ray_out, double* J) {
  // camera.cpp:58-100
  if (u < 0.0 || v < 0.0 || u > rays.width - 1 || v > rays.height - 1) return false;
  int u0 = (int)std::floor(u);
  int v0 = (int)std::floor(v);
  u0 = std::min(u0, rays.width - 2 >= 0 ? rays.width - 2 : 0);
  v0 = std::min(v0, rays.height - 2 >= 0 ? rays.height - 2 : 0);
  const int u1 = std::min(u0 + 1, rays.width - 1);
  const int v1 = std::min(v0 + 1, rays.height - 1);
  const double fu = u - u0;
  const double fv = v - v0;
  const int i00 = rays.index(u0, v0), i10 = rays.index(u1, v0);
  const int i01 = rays.index(u0, v1), i11 = rays.index(u1, v1);
  if (!rays.valid[i00] || !rays.valid[i10] || !rays.valid[i01] || !rays.valid[i11]) return false;
  const Vec3& r00 = rays.rays[i00];
  const Vec3& r10 = rays.rays[i10];
  const Vec3& r01 = rays.rays[i01];
  const Vec3& r11 = rays.rays[i11];
  const Vec3 g = (1 - fu) * (1 - fv) * r00 + fu * (1 - fv) * r10 + (1 - fu) * fv * r01 + fu * fv * r11;
  const double gn = norm(g);
  if (gn < 1e-12) return false;
  const Vec3 ray = g / gn;
  if (J) {
    const Vec3 dg_du = (1 - fv) * (r10 - r00) + fv * (r11 - r01);
    const Vec3 dg_dv = (1 - fu) * (r01 - r00) + fu * (r11 - r10);
    // proj = (I - r r^T) / gn
    for (int c = 0; c < 2; ++c) {
      const Vec3& d = c == 0 ? dg_du : dg_dv;
      const double rd = dot(ray, d);
      for (int r = 0; r < 3; ++r) J[c * 3 + r] = (d[r] - ray[r] * rd) / gn;
    }
  }
  *ray_out = ray;
  return true;
}

namespace {
Vec2 clamp_to_image(const Vec2& p, int width, int height) {  // camera.cpp:104-107
  return {std::clamp(p.x, 0.0, (double)(width - 1)), std::clamp(p.y, 0.0, (double)(height - 1))};
}
double angular_error(const Vec3& a, const Vec3& b) {  // camera.cpp:109-111
  return std::acos(std::clamp(dot(a, b), -1.0, 1.0));
}
}  // namespace

ProjectResult iterative_project(const RayMap& rays, const Vec3& x, const Vec2& p0,
                                const IterProjParams& params) {  // camera.cpp:115-174
  ProjectResult result;
  const double xn = norm(x);
  if (xn < 1e-12 || !finite(x)) {
    result.pixel = clamp_to_image(p0, rays.width, rays.height);
    return result;
  }
  const Vec3 target = x / xn;
  Vec2 p = clamp_to_image(p0, rays.width, rays.height);
  double J[6];
  Vec3 ray;
  if (!interpolate_ray(rays, p.x, p.y, &ray, J)) {
    result.pixel = p;
    return result;
  }
  double cost = sqnorm(ray - target);
  if (angular_error(ray, target) < params.angle_tol) {
    result.pixel = p;
    result.converged = true;
    return result;
  }
  double lambda = params.lambda_init;
  for (int iter = 0; iter < params.max_iterations; ++iter) {
    ++result.iterations;
    const Vec3 r = ray - target;
    const Vec3 j0(J[0], J[1], J[2]), j1(J[3], J[4], J[5]);
    double JtJ[4] = {dot(j0, j0), dot(j0, j1), dot(j1, j0), dot(j1, j1)};
    const double g[2] = {dot(j0, r), dot(j1, r)};
    double H[4] = {JtJ[0], JtJ[1], JtJ[2], JtJ[3]};
    H[0] += lambda * std::max(JtJ[0], 1e-12);
    H[3] += lambda * std::max(JtJ[3], 1e-12);
    double sol[2];
    ldlt_pivoted_solve(2, H, g, sol);
    const Vec2 delta{-sol[0], -sol[1]};
    if (!std::isfinite(delta.x) || !std::isfinite(delta.y)) break;
    const Vec2 p_trial = clamp_to_image({p.x + delta.x, p.y + delta.y}, rays.width, rays.height);
    double J_trial[6];
    Vec3 ray_trial;
    if (interpolate_ray(rays, p_trial.x, p_trial.y, &ray_trial, J_trial)) {
      const double cost_trial = sqnorm(ray_trial - target);
      if (cost_trial < cost) {
        p = p_trial;
        ray = ray_trial;
        for (int k = 0; k < 6; ++k) J[k] = J_trial[k];
        cost = cost_trial;
        lambda *= params.lambda_down;
        if (angular_error(ray, target) < params.angle_tol) {
          result.pixel = p;
          result.converged = true;
          return result;
        }
        continue;
      }
    }
    lambda *= params.lambda_up;
  }
  result.pixel = p;
  result.converged = angular_error(ray, target) < params.angle_tol;
  return result;
}

double median_scene_distance(const Pointmap& pm) {  // camera.cpp:178-191
  std::vector<double> norms;
  norms.reserve(pm.size());
  for (int i = 0; i < pm.size(); ++i) {
    if (pm.valid[i]) {
      const double n = norm(pm.points[i]);
      if (n > 1e-12) norms.push_back(n);
    }
  }
  if (norms.empty()) return 0.0;
  const size_t mid = norms.size() / 2;
  std::nth_element(norms.begin(), norms.begin() + mid, norms.end());
  return norms[mid];
}

MatchSet match_pointmaps(const Pointmap& X_a, const Pointmap& X_b_in_a, const FeatureMap& F_a,
                         const FeatureMap& F_b, const MatchSet* init,
                         const MatchParams& params) {  // camera.cpp:195-237
  const RayMap rays_a = normalize_rays(X_a);
  const double dist_threshold = params.invalidation_median_fraction * median_scene_distance(X_a);
  std::vector<int> seed(X_b_in_a.size(), -1);
  if (init) {
    for (const auto& m : init->matches)
      if (m.valid && m.pixel_b >= 0 && m.pixel_b < X_b_in_a.size()) seed[m.pixel_b] = m.pixel_a;
  }
  MatchSet out;
  out.matches.resize(X_b_in_a.size());
  for (int n = 0; n < X_b_in_a.size(); ++n) {
    Match& m = out.matches[n];
    m.pixel_b = n;
    if (!X_b_in_a.valid[n]) continue;
    const Vec3& x = X_b_in_a.points[n];
    if (norm(x) < 1e-12) continue;
    const int seed_pixel = seed[n] >= 0 ? seed[n] : n;
    const Vec2 p0{(double)(seed_pixel % X_a.width), (double)(seed_pixel / X_a.width)};
    const ProjectResult proj = iterative_project(rays_a, x, p0, params.projection);
    const int pu = (int)std::lround(proj.pixel.x);
    const int pv = (int)std::lround(proj.pixel.y);
    const int pa = std::clamp(pv, 0, X_a.height - 1) * X_a.width + std::clamp(pu, 0, X_a.width - 1);
    m.pixel_a = pa;
    m.confidence = std::sqrt(F_a.match_confidence[pa] * F_b.match_confidence[n]);
    if (!proj.converged || !X_a.valid[pa]) continue;
    if (norm(X_a.points[pa] - x) > dist_threshold) continue;
    m.valid = true;
  }
  return out;
}

static double dotd(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) s += a[k] * b[k];
  return s;
}

MatchSet feature_refine(const MatchSet& matches, const FeatureMap& F_a, const FeatureMap& F_b,
                        const RefineParams& params) {  // camera.cpp:239-271
  MatchSet out = matches;
  const int d = F_a.dim;
  for (auto& m : out.matches) {
    if (!m.valid || m.pixel_a < 0 || m.pixel_b < 0) continue;
    int best_u = m.pixel_a % F_a.width;
    int best_v = m.pixel_a / F_a.width;
    const double* target = F_b.col(m.pixel_b);
    for (const auto& [stride, radius] : params.levels) {
      const int cu = best_u, cv = best_v;
      double best_score = dotd(F_a.col(F_a.index(best_u, best_v)), target, d);
      for (int dv = -radius; dv <= radius; ++dv) {
        for (int du = -radius; du <= radius; ++du) {
          const int u = cu + du * stride;
          const int v = cv + dv * stride;
          if (u < 0 || v < 0 || u >= F_a.width || v >= F_a.height) continue;
          const double score = dotd(F_a.col(F_a.index(u, v)), target, d);
          if (score > best_score) {
            best_score = score;
            best_u = u;
            best_v = v;
          }
        }
      }
    }
    m.pixel_a = F_a.index(best_u, best_v);
    m.confidence = std::sqrt(F_a.match_confidence[m.pixel_a] * F_b.match_confidence[m.pixel_b]);
  }
  return out;
}

PinholeProjection pinhole_project(const Vec3& x, const PinholeIntrinsics& K) {  // camera.cpp:293-303
  const double z = x[2];
  if (!(z > 0.0)) throw std::domain_error("pinhole_project: point behind camera");
  PinholeProjection out;
  out.pixel = {K.fx * x[0] / z + K.cx, K.fy * x[1] / z + K.cy};
  out.J[0] = K.fx / z;
  out.J[1] = 0.0;
  out.J[2] = -K.fx * x[0] / (z * z);
  out.J[3] = 0.0;
  out.J[4] = K.fy / z;
  out.J[5] = -K.fy * x[1] / (z * z);
  return out;
}

// -------------------------------------------------------------- tracking.cpp
double robust_weight(double q, double sigma2, double q_min) {  // tracking.cpp:10-13
  if (q > q_min) return sigma2 / q;
  return std::numeric_limits<double>::infinity();
}
double huber_cost(double e, double delta) {  // tracking.cpp:24-26
  return e <= delta ? 0.5 * e * e : delta * (e - 0.5 * delta);
}
double huber_factor(double e, double delta) {  // tracking.cpp:28-30
  return e <= delta ? 1.0 : delta / e;
}
double median_confidence(const MatchSet& matches) {  // tracking.cpp:32-42
  std::vector<double> q;
  q.reserve(matches.matches.size());
  for (const auto& m : matches.matches)
    if (m.valid) q.push_back(m.confidence);
  if (q.empty()) return 0.0;
  const size_t mid = q.size() / 2;
  std::nth_element(q.begin(), q.begin() + mid, q.end());
  return q[mid];
}

std::vector<ResidualBlock> residual_blocks(const Sim3& T, const MatchSet& matches,
                                           const Pointmap& X_ref, const Pointmap& X_src,
                                           TrackMode mode, const RobustWeightParams& params,
                                           const PinholeIntrinsics* K) {  // tracking.cpp:46-132
  if (mode == TrackMode::kPixel && K == nullptr)
    throw std::invalid_argument("residual_blocks: pixel mode requires intrinsics");
  const double sigma2 = mode == TrackMode::kRay     ? params.sigma2_ray
                        : mode == TrackMode::kPoint ? params.sigma2_point
                                                    : params.sigma2_pixel;
  std::vector<ResidualBlock> blocks(matches.matches.size());
  for (size_t k = 0; k < matches.matches.size(); ++k) {
    const Match& match = matches.matches[k];
    ResidualBlock& b = blocks[k];
    if (!match.valid || match.pixel_a < 0 || match.pixel_b < 0) continue;
    if (!X_ref.valid[match.pixel_b] || !X_src.valid[match.pixel_a]) continue;
    const double denom = robust_weight(match.confidence, sigma2, params.q_min);
    if (!std::isfinite(denom)) continue;
    const double info = 1.0 / denom;
    const Vec3& ref = X_ref.points[match.pixel_b];
    const Vec3 x = T.act(X_src.points[match.pixel_a]);
    const double d = norm(x);
    if (d < 1e-12) continue;
    int main_rows = 3;
    bool has_distance = true;
    double* J = b.jacobian;
    switch (mode) {
      case TrackMode::kRay: {
        const double d_ref = norm(ref);
        if (d_ref < 1e-12) continue;
        const Vec3 xn = x / d;
        const Vec3 rr = ref / d_ref - xn;
        b.residual[0] = rr[0];
        b.residual[1] = rr[1];
        b.residual[2] = rr[2];
        b.residual[3] = d_ref - d;
        const Mat3 S = skew(x);
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 3; ++c) {
            const double P = ((r == c ? 1.0 : 0.0) - xn[r] * xn[c]) / d;
            J[r * 7 + c] = -P;
            J[r * 7 + 3 + c] = S(r, c) / d;
          }
          J[r * 7 + 6] = 0.0;
        }
        for (int c = 0; c < 3; ++c) J[3 * 7 + c] = -xn[c];
        J[3 * 7 + 6] = -d;
        break;
      }
      case TrackMode::kPoint: {
        const Vec3 rr = ref - x;
        b.residual[0] = rr[0];
        b.residual[1] = rr[1];
        b.residual[2] = rr[2];
        const Mat3 S = skew(x);
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 3; ++c) {
            J[r * 7 + c] = r == c ? -1.0 : 0.0;
            J[r * 7 + 3 + c] = S(r, c);
          }
          J[r * 7 + 6] = -x[r];
        }
        has_distance = false;
        break;
      }
      case TrackMode::kPixel: {
        if (x[2] <= 1e-12 || ref[2] <= 1e-12) continue;
        const int u = match.pixel_b % X_ref.width;
        const int v = match.pixel_b / X_ref.width;
        const PinholeProjection proj = pinhole_project(x, *K);
        b.residual[0] = u - proj.pixel.x;
        b.residual[1] = v - proj.pixel.y;
        double pj[21];  // 3x7: [I, -[x]x, x]
        const Mat3 S = skew(x);
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 3; ++c) {
            pj[r * 7 + c] = r == c ? 1.0 : 0.0;
            pj[r * 7 + 3 + c] = -S(r, c);
          }
          pj[r * 7 + 6] = x[r];
        }
        for (int r = 0; r < 2; ++r)
          for (int c = 0; c < 7; ++c) {
            double s = 0.0;
            for (int k2 = 0; k2 < 3; ++k2) s += proj.J[r * 3 + k2] * pj[k2 * 7 + c];
            J[r * 7 + c] = -s;
          }
        b.residual[3] = ref[2] - x[2];
        for (int c = 0; c < 7; ++c) J[3 * 7 + c] = -pj[2 * 7 + c];
        main_rows = 2;
        break;
      }
    }
    double sq = 0.0;
    for (int r = 0; r < main_rows; ++r) sq += b.residual[r] * b.residual[r];
    const double e = std::sqrt(info) * std::sqrt(sq);
    const double w = info * huber_factor(e, params.huber_delta);
    for (int r = 0; r < main_rows; ++r) b.weight[r] = w;
    if (has_distance) {
      const double info_d = params.distance_weight * info;
      const double e_d = std::sqrt(info_d) * std::abs(b.residual[3]);
      b.weight[3] = info_d * huber_factor(e_d, params.huber_delta);
    }
    b.info = info;
    b.used = true;
  }
  return blocks;
}

double block_cost(const std::vector<ResidualBlock>& blocks, const RobustWeightParams& params,
                  TrackMode mode) {  // tracking.cpp:134-147
  double cost = 0.0;
  const int main_rows = mode == TrackMode::kPixel ? 2 : 3;
  for (const auto& b : blocks) {
    if (!b.used) continue;
    double sq = 0.0;
    for (int r = 0; r < main_rows; ++r) sq += b.residual[r] * b.residual[r];
    const double e = std::sqrt(b.info) * std::sqrt(sq);
    cost += huber_cost(e, params.huber_delta);
    const double e_d = std::sqrt(params.distance_weight * b.info) * std::abs(b.residual[3]);
    cost += huber_cost(e_d, params.huber_delta);
  }
  return cost;
}

static void accumulate_normal(const std::vector<ResidualBlock>& blocks, Mat7& H, Vec7& g) {
  // tracking.cpp:188-198
  H.fill(0.0);
  g.fill(0.0);
  for (const auto& b : blocks) {
    if (!b.used) continue;
    for (int r = 0; r < 4; ++r) {
      const double w = b.weight[r];
      if (w <= 0.0) continue;
      const double* j = b.jacobian + r * 7;
      for (int a = 0; a < 7; ++a) {
        for (int c = 0; c < 7; ++c) H[a * 7 + c] += w * j[a] * j[c];
        g[a] += w * j[a] * b.residual[r];
      }
    }
  }
}

TrackResult track_given_matches(const Pointmap& canonical, const Pointmap& X_f_f,
                                const MatchSet& matches, const Sim3& init, TrackMode mode,
                                const SolvePoseParams& params) {  // tracking.cpp:165-225
  TrackResult result;
  result.T_kf = init;
  result.matches = matches;
  if (matches.valid_count() < params.min_valid_matches) {
    result.lost = true;
    return result;
  }
  RobustWeightParams weights = params.weights;
  weights.q_min = weights.q_min_fraction * median_confidence(matches);
  const PinholeIntrinsics* K = params.intrinsics ? &*params.intrinsics : nullptr;
  auto evaluate = [&](const Sim3& T) {
    return residual_blocks(T, matches, canonical, X_f_f, mode, weights, K);
  };
  auto blocks = evaluate(result.T_kf);
  double cost = block_cost(blocks, weights, mode);
  result.cost_trace.push_back(cost);
  double lambda = 1e-8;
  for (int iter = 0; iter < params.max_iterations; ++iter) {
    Mat7 H;
    Vec7 g;
    accumulate_normal(blocks, H, g);
    ++result.iterations;
    Mat7 Hd = H;
    for (int k = 0; k < 7; ++k) Hd[k * 8] += lambda * std::max(H[k * 8], 1e-12);
    Vec7 mg;
    for (int k = 0; k < 7; ++k) mg[k] = -g[k];
    Vec7 tau;
    ldlt_pivoted_solve(7, Hd.data(), mg.data(), tau.data());
    bool accepted = false;
    bool fin = true;
    double inf = 0.0, nrm2 = 0.0;
    for (int k = 0; k < 7; ++k) {
      fin = fin && std::isfinite(tau[k]);
      inf = std::max(inf, std::abs(tau[k]));
      nrm2 += tau[k] * tau[k];
    }
    if (fin && inf < 1e3) {
      const Sim3 T_new = result.T_kf.retract(tau);
      auto blocks_new = evaluate(T_new);
      const double cost_new = block_cost(blocks_new, weights, mode);
      if (cost_new <= cost * (1.0 + 1e-12) + 1e-300) {
        result.T_kf = T_new;
        blocks = std::move(blocks_new);
        cost = cost_new;
        result.cost_trace.push_back(cost);
        lambda = std::max(lambda * 0.3, 1e-10);
        accepted = true;
        if (std::sqrt(nrm2) < params.update_tol) break;
      }
    }
    if (!accepted) {
      lambda *= 10.0;
      if (lambda > 1e8) break;
    }
  }
  return result;
}

TrackResult solve_pose(const Pointmap& canonical, const Pointmap& X_f_f, const Pointmap& X_k_f,
                       const FeatureMap& F_f, const FeatureMap& F_k, const Sim3& init,
                       TrackMode mode, const SolvePoseParams& params,
                       const MatchSet* match_seed) {  // tracking.cpp:149-226
  MatchSet matches = match_pointmaps(X_f_f, X_k_f, F_f, F_k, match_seed, params.matching);
  if (params.refine_features) matches = feature_refine(matches, F_f, F_k, params.refinement);
  if (mode == TrackMode::kPixel && !params.intrinsics) {
    // residual_blocks throws on the first evaluation (tracking.cpp:50-52)
    if (matches.valid_count() >= params.min_valid_matches)
      throw std::invalid_argument("residual_blocks: pixel mode requires intrinsics");
  }
  return track_given_matches(canonical, X_f_f, matches, init, mode, params);
}

void fuse_canonical(Pointmap& canonical, std::vector<double>& canonical_conf, const Pointmap& X_k_f,
                    const std::vector<double>& confidence, const Sim3& T_kf) {  // tracking.cpp:228-247
  for (int i = 0; i < canonical.size(); ++i) {
    if (!X_k_f.valid[i]) continue;
    const double c = confidence[i];
    const double c_prev = canonical_conf[i];
    if (c_prev + c <= 0.0) continue;
    const Vec3 observed = T_kf.act(X_k_f.points[i]);
    if (c_prev <= 0.0 || !canonical.valid[i]) {
      canonical.points[i] = observed;
    } else {
      canonical.points[i] = (c_prev * canonical.points[i] + c * observed) / (c_prev + c);
    }
    canonical.valid[i] = 1;
    canonical_conf[i] = c_prev + c;
  }
}

bool keyframe_decision(const MatchSet& matches, int height, int width, double omega_k) {
  // tracking.cpp:249-257
  const int total = height * width;
  if (total <= 0) return true;
  const double valid_fraction = (double)matches.valid_count() / total;
  const double unique_fraction = matches.unique_pixel_fraction(total);
  return valid_fraction < omega_k || unique_fraction < omega_k;
}

// --------------------------------------------------------------- backend.cpp
namespace {
MatchSet swapped(const MatchSet& m) {  // backend.cpp:31-35
  MatchSet out = m;
  for (auto& x : out.matches) std::swap(x.pixel_a, x.pixel_b);
  return out;
}
double median_edge_confidence(const MatchSet& m) {  // backend.cpp:37-46
  return median_confidence(m);
}
struct DirectedConstraint {  // backend.cpp:48-53
  int ref_index, src_index;
  MatchSet matches;
  double q_min;
};
std::vector<DirectedConstraint> directed_constraints(const Graph& g, const BackendParams& p) {
  // backend.cpp:55-69
  std::vector<DirectedConstraint> out;
  const int n = (int)g.poses.size();
  for (const auto& e : g.edges) {
    if (e.i < 0 || e.j < 0 || e.i >= n || e.j >= n) continue;
    const double q_min = p.weights.q_min_fraction * median_edge_confidence(e.matches);
    out.push_back({e.i, e.j, swapped(e.matches), q_min});
    out.push_back({e.j, e.i, e.matches, q_min});
  }
  return out;
}
void accumulate_directed(const Graph& g, const BackendParams& p, const DirectedConstraint& con,
                         Mat7& Hrel, Vec7& grel, double& cost) {
  const Sim3 T_rel = relative_pose(g.poses[con.ref_index], g.poses[con.src_index]);
  RobustWeightParams w = p.weights;
  w.q_min = con.q_min;
  const PinholeIntrinsics* K = p.intrinsics ? &*p.intrinsics : nullptr;
  const auto res = residual_blocks(T_rel, con.matches, g.canonicals[con.ref_index],
                                   g.canonicals[con.src_index], p.mode, w, K);
  accumulate_normal(res, Hrel, grel);
  cost = block_cost(res, w, p.mode);
}
}  // namespace

AssembledSystem assemble_system(const Graph& g, const BackendParams& p) {  // backend.cpp:91-173
  const int n = (int)g.poses.size();
  const int dim = 7 * n;
  const int anchor = g.anchor;
  const PinholeIntrinsics* K = p.intrinsics ? &*p.intrinsics : nullptr;
  std::map<std::pair<int, int>, Mat7> blocks;
  std::vector<double> gradient(dim, 0.0);
  auto accumulate = [&blocks](int r, int c, const Mat7& v) {
    auto [it, ins] = blocks.try_emplace({r, c}, Mat7{});
    for (int k = 0; k < 49; ++k) it->second[k] += v[k];
  };
  for (const auto& con : directed_constraints(g, p)) {
    const Sim3 T_rel = relative_pose(g.poses[con.ref_index], g.poses[con.src_index]);
    RobustWeightParams w = p.weights;
    w.q_min = con.q_min;
    const auto res = residual_blocks(T_rel, con.matches, g.canonicals[con.ref_index],
                                     g.canonicals[con.src_index], p.mode, w, K);
    const Mat7 adj = g.poses[con.ref_index].inverse().adjoint();
    Mat7 H_rr{}, H_rs{}, H_ss{};
    Vec7 g_ref{}, g_src{};
    for (const auto& b : res) {
      if (!b.used) continue;
      for (int r = 0; r < 4; ++r) {
        const double wr = b.weight[r];
        if (wr <= 0.0) continue;
        const double* jr = b.jacobian + r * 7;
        double j_ref[7], j_src[7];
        for (int c = 0; c < 7; ++c) {
          double s = 0.0;
          for (int k = 0; k < 7; ++k) s += jr[k] * adj[k * 7 + c];
          j_src[c] = s;
          j_ref[c] = -s;
        }
        for (int a = 0; a < 7; ++a) {
          for (int c = 0; c < 7; ++c) {
            H_rr[a * 7 + c] += wr * j_ref[a] * j_ref[c];
            H_rs[a * 7 + c] += wr * j_ref[a] * j_src[c];
            H_ss[a * 7 + c] += wr * j_src[a] * j_src[c];
          }
          g_ref[a] += wr * j_ref[a] * b.residual[r];
          g_src[a] += wr * j_src[a] * b.residual[r];
        }
      }
    }
    Mat7 H_sr;
    for (int a = 0; a < 7; ++a)
      for (int c = 0; c < 7; ++c) H_sr[a * 7 + c] = H_rs[c * 7 + a];
    accumulate(con.ref_index, con.ref_index, H_rr);
    accumulate(con.ref_index, con.src_index, H_rs);
    accumulate(con.src_index, con.ref_index, H_sr);
    accumulate(con.src_index, con.src_index, H_ss);
    for (int a = 0; a < 7; ++a) {
      gradient[7 * con.ref_index + a] += g_ref[a];
      gradient[7 * con.src_index + a] += g_src[a];
    }
  }
  if (anchor >= 0) {  // backend.cpp:144-155
    for (auto it = blocks.begin(); it != blocks.end();) {
      if (it->first.first == anchor || it->first.second == anchor)
        it = blocks.erase(it);
      else
        ++it;
    }
    Mat7 I{};
    for (int k = 0; k < 7; ++k) I[k * 8] = 1.0;
    blocks[{anchor, anchor}] = I;
    for (int a = 0; a < 7; ++a) gradient[7 * anchor + a] = 0.0;
  }
  AssembledSystem sys;
  sys.dim = dim;
  sys.hessian.assign((size_t)dim * dim, 0.0);
  for (const auto& [key, blk] : blocks)
    for (int r = 0; r < 7; ++r)
      for (int c = 0; c < 7; ++c)
        sys.hessian[(size_t)(7 * key.first + r) * dim + 7 * key.second + c] += blk[r * 7 + c];
  sys.gradient = std::move(gradient);
  return sys;
}

double backend_cost(const Graph& g, const BackendParams& p) {  // backend.cpp:175-190
  double cost = 0.0;
  const PinholeIntrinsics* K = p.intrinsics ? &*p.intrinsics : nullptr;
  for (const auto& con : directed_constraints(g, p)) {
    const Sim3 T_rel = relative_pose(g.poses[con.ref_index], g.poses[con.src_index]);
    RobustWeightParams w = p.weights;
    w.q_min = con.q_min;
    const auto res = residual_blocks(T_rel, con.matches, g.canonicals[con.ref_index],
                                     g.canonicals[con.src_index], p.mode, w, K);
    cost += block_cost(res, w, p.mode);
  }
  return cost;
}

bool sparse_ldlt_solve(int n, const std::vector<double>& A, const std::vector<double>& b,
                       std::vector<double>* x) {
  // SimplicialLDLT restatement (backend.cpp:216-218): envelope LDL^T in natural
  // order, no pivoting, failure iff a pivot is exactly zero.  L is stored in
  // the envelope of the lower triangle; entries outside it stay zero.
  std::vector<int> first(n);
  for (int i = 0; i < n; ++i) {
    int f = i;
    for (int j = 0; j < i; ++j)
      if (A[(size_t)i * n + j] != 0.0) {
        f = j;
        break;
      }
    first[i] = f;
  }
  std::vector<double> L((size_t)n * n, 0.0);
  std::vector<double> D(n, 0.0);
  for (int i = 0; i < n; ++i) {
    for (int j = first[i]; j < i; ++j) {
      // L_ij D_j = A_ij - sum_{k<j} L_ik D_k L_jk
      double s = A[(size_t)i * n + j];
      const int k0 = std::max(first[i], first[j]);
      for (int k = k0; k < j; ++k) s -= L[(size_t)i * n + k] * D[k] * L[(size_t)j * n + k];
      L[(size_t)i * n + j] = s / D[j];
    }
    double s = A[(size_t)i * n + i];
    for (int k = first[i]; k < i; ++k) s -= L[(size_t)i * n + k] * L[(size_t)i * n + k] * D[k];
    if (s == 0.0 || !std::isfinite(s)) return false;
    D[i] = s;
  }
  std::vector<double> y(b);
  for (int i = 0; i < n; ++i)
    for (int k = first[i]; k < i; ++k) y[i] -= L[(size_t)i * n + k] * y[k];
  for (int i = 0; i < n; ++i) y[i] /= D[i];
  for (int i = n - 1; i >= 0; --i)
    for (int k = first[i]; k < i; ++k) y[k] -= L[(size_t)i * n + k] * y[i];
  *x = std::move(y);
  return true;
}

OptimizeResult global_optimize(Graph& g, const BackendParams& p,
                               std::vector<std::vector<Sim3>>* pose_trace) {
  // backend.cpp:192-256
  OptimizeResult result;
  const int n = (int)g.poses.size();
  if (n < 2 || g.edges.empty()) {
    result.converged = true;
    return result;
  }
  const int anchor = g.anchor;
  double cost = backend_cost(g, p);
  result.cost_trace.push_back(cost);
  for (int iter = 0; iter < p.max_iterations; ++iter) {
    ++result.iterations;
    AssembledSystem sys = assemble_system(g, p);
    std::vector<double> tau;
    bool solved = false;
    double lambda = 0.0;
    std::vector<double> rhs(sys.dim);
    for (int k = 0; k < sys.dim; ++k) rhs[k] = -sys.gradient[k];
    for (int attempt = 0; attempt <= p.damping_retries; ++attempt) {
      std::vector<double> H = sys.hessian;
      if (lambda > 0.0)
        for (int k = 0; k < sys.dim; ++k) H[(size_t)k * sys.dim + k] += lambda;
      if (sparse_ldlt_solve(sys.dim, H, rhs, &tau)) {
        bool fin = true;
        double inf = 0.0;
        for (double v : tau) {
          fin = fin && std::isfinite(v);
          inf = std::max(inf, std::abs(v));
        }
        if (fin && inf < 1e3) {
          solved = true;
          break;
        }
      }
      lambda = lambda == 0.0 ? p.damping_init : lambda * 10.0;
    }
    if (!solved) return result;
    std::vector<Sim3> previous = g.poses;
    for (int k = 0; k < n; ++k) {
      if (k == anchor) continue;
      Vec7 t7;
      for (int a = 0; a < 7; ++a) t7[a] = tau[7 * k + a];
      g.poses[k] = g.poses[k].retract(t7);
    }
    if (pose_trace) pose_trace->push_back(g.poses);
    const double cost_new = backend_cost(g, p);
    if (cost_new > cost * (1.0 + 1e-12) + 1e-300) {
      g.poses = previous;
      if (pose_trace) pose_trace->back() = previous;
      result.converged = true;
      return result;
    }
    cost = cost_new;
    result.cost_trace.push_back(cost);
    double nrm2 = 0.0;
    for (double v : tau) nrm2 += v * v;
    if (std::sqrt(nrm2) < p.update_tol) {
      result.converged = true;
      return result;
    }
  }
  result.converged = true;
  return result;
}

void backend_edge_terms(const Graph& g, const BackendParams& p, int e, double* out72) {
  const Edge& edge = g.edges[e];
  const double q_min = p.weights.q_min_fraction * median_edge_confidence(edge.matches);
  const DirectedConstraint d1{edge.i, edge.j, swapped(edge.matches), q_min};
  const DirectedConstraint d2{edge.j, edge.i, edge.matches, q_min};
  const DirectedConstraint* dirs[2] = {&d1, &d2};
  for (int k = 0; k < 2; ++k) {
    Mat7 H;
    Vec7 gg;
    double c;
    accumulate_directed(g, p, *dirs[k], H, gg, c);
    double* o = out72 + 36 * k;
    int idx = 0;
    for (int a = 0; a < 7; ++a)
      for (int b = a; b < 7; ++b) o[idx++] = H[a * 7 + b];
    for (int a = 0; a < 7; ++a) o[28 + a] = gg[a];
    o[35] = c;
  }
}

}  // namespace orc
