// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A single-threaded FP64 C++ restatement of the CPU reference "pmslam"
// hot path (MASt3R-SLAM, arXiv 2412.12392): /root/reference/proj/src/
// {lie,camera,tracking,backend}.cpp.  Every function cites the reference
// file:line it follows.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load this library; the product
// (paper_2412_12392_b200, libpmx_cuda.so) never links or calls it.
//
// The reference itself cannot be compiled here or on the GPU box (it needs
// Eigen3, which is absent from the image), so the Eigen arithmetic it calls is
// restated from Eigen's published algorithms (version unpinned by the
// reference, proj/CMakeLists.txt:11):
//   * Matrix::ldlt()            — LDL^T with symmetric diagonal pivoting
//                                 (largest remaining |diagonal| first) and a
//                                 pseudo-inverse of D at solve time
//                                 (|D_i| <= DBL_MIN -> component 0).
//   * SimplicialLDLT            — sparse LDL^T without pivoting; fails iff a
//                                 pivot is exactly 0.  Restated as an envelope
//                                 (skyline) LDL^T in natural ordering: same
//                                 factorisation semantics, ordering differs
//                                 from Eigen's AMD only in rounding.
//   * JacobiSVD (renormalise)   — restated as the polar factor U V^T
//                                 (Newton iteration), identical in exact math.
// Parity pinning: see oracle/README.md and tests/test_oracle_pins.py (the
// reference's known-answer and property tests, ported).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <optional>
#include <utility>
#include <vector>

namespace orc {

// ----------------------------------------------------------------- small LA
struct Vec2 {
  double x = 0, y = 0;
};
struct Vec3 {
  double v[3] = {0, 0, 0};
  Vec3() = default;
  Vec3(double a, double b, double c) : v{a, b, c} {}
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};
inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a[0] / s, a[1] / s, a[2] / s}; }
inline double dot(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double sqnorm(const Vec3& a) { return dot(a, a); }
inline double norm(const Vec3& a) { return std::sqrt(sqnorm(a)); }
inline bool finite(const Vec3& a) {
  return std::isfinite(a[0]) && std::isfinite(a[1]) && std::isfinite(a[2]);
}

struct Mat3 {
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // row-major
  double& operator()(int r, int c) { return m[3 * r + c]; }
  double operator()(int r, int c) const { return m[3 * r + c]; }
  static Mat3 identity() {
    Mat3 I;
    I.m[0] = I.m[4] = I.m[8] = 1.0;
    return I;
  }
};
Mat3 operator*(const Mat3& a, const Mat3& b);
Vec3 operator*(const Mat3& a, const Vec3& x);
Mat3 operator+(const Mat3& a, const Mat3& b);
Mat3 operator*(double s, const Mat3& a);
Mat3 transpose(const Mat3& a);

using Vec7 = std::array<double, 7>;
using Mat7 = std::array<double, 49>;  // row-major

// Eigen LDLT (pivoted, pseudo-inverse D) restatement for small dense SPD/SPSD
// systems: solves A x = b, n <= 7.
void ldlt_pivoted_solve(int n, const double* A, const double* b, double* x);

// ----------------------------------------------------------------- lie.cpp
constexpr double kSmallAngle = 1e-8;  // lie.hpp:21
Mat3 skew(const Vec3& v);                             // lie.cpp:13-21
Mat3 so3_exp(const Vec3& omega);                      // lie.cpp:23-32
Vec3 so3_log(const Mat3& R);                          // lie.cpp:34-49
Mat3 sim3_w_matrix(const Vec3& omega, double sigma);  // lie.cpp:51-90

struct Sim3 {  // lie.hpp:36-70
  Mat3 R = Mat3::identity();
  Vec3 t;
  double s = 1.0;
  int ops_since_renorm = 0;

  static Sim3 exp(const Vec7& tau);  // lie.cpp:99-108
  Vec7 log() const;                  // lie.cpp:110-119
  Sim3 inverse() const;              // lie.cpp:121-129
  Sim3 operator*(const Sim3& o) const;  // lie.cpp:131-140
  Vec3 act(const Vec3& x) const { return s * (R * x) + t; }  // lie.hpp:48
  Mat7 adjoint() const;                                     // lie.cpp:155-163
  Sim3 retract(const Vec7& tau) const { return exp(tau) * *this; }  // lie.hpp:54
  void renormalize_if_needed();                             // lie.cpp:142-153
};
Sim3 relative_pose(const Sim3& T_wi, const Sim3& T_wj);  // lie.cpp:171-173

// -------------------------------------------------------------- camera.cpp
struct Pointmap {  // camera.hpp:17-31
  int height = 0, width = 0;
  std::vector<Vec3> points;
  std::vector<uint8_t> valid;
  int size() const { return height * width; }
  int index(int u, int v) const { return v * width + u; }
};

struct RayMap {  // camera.hpp:44-52
  int height = 0, width = 0;
  std::vector<Vec3> rays;
  std::vector<double> distances;
  std::vector<uint8_t> valid;
  int index(int u, int v) const { return v * width + u; }
};

struct FeatureMap {  // camera.hpp:55-71 (descriptors pixel-major: dim per pixel)
  int height = 0, width = 0, dim = 0;
  std::vector<double> descriptors;  // HW * dim
  std::vector<double> match_confidence;
  int index(int u, int v) const { return v * width + u; }
  const double* col(int pixel) const { return descriptors.data() + (size_t)pixel * dim; }
};

struct Match {  // camera.hpp:73-78
  int pixel_a = -1;
  int pixel_b = -1;
  double confidence = 0.0;
  bool valid = false;
};

struct MatchSet {  // camera.hpp:80-89
  std::vector<Match> matches;
  int valid_count() const;                                 // camera.cpp:10-14
  double valid_fraction() const;                           // camera.cpp:16-19
  double unique_pixel_fraction(int num_pixels_a) const;    // camera.cpp:21-28
  static MatchSet identity(int n, double confidence = 1.0);  // camera.cpp:30-37
};

struct IterProjParams {  // camera.hpp:102-108
  double lambda_init = 1e-4;
  double lambda_up = 10.0;
  double lambda_down = 0.3;
  double angle_tol = 1e-5;
  int max_iterations = 10;
};

struct ProjectResult {  // camera.hpp:110-114
  Vec2 pixel;
  bool converged = false;
  int iterations = 0;
};

struct MatchParams {  // camera.hpp:126-131
  IterProjParams projection;
  double invalidation_median_fraction = 0.1;
};

struct RefineParams {  // camera.hpp:140-143
  std::vector<std::pair<int, int>> levels = {{2, 2}, {1, 2}};
};

struct PinholeIntrinsics {  // camera.hpp:91-96
  double fx = 0, fy = 0, cx = 0, cy = 0;
};

RayMap normalize_rays(const Pointmap& pm);  // camera.cpp:39-56
// camera.cpp:58-100; J is 3x2 column-major {col0 xyz, col1 xyz}
bool interpolate_ray(const RayMap& rays, double u, double v, Vec3* ray, double* J);
ProjectResult iterative_project(const RayMap& rays, const Vec3& x, const Vec2& p0,
                                const IterProjParams& params);  // camera.cpp:115-174
double median_scene_distance(const Pointmap& pm);               // camera.cpp:178-191
MatchSet match_pointmaps(const Pointmap& X_a, const Pointmap& X_b_in_a,
                         const FeatureMap& F_a, const FeatureMap& F_b,
                         const MatchSet* init, const MatchParams& params);  // camera.cpp:195-237
MatchSet feature_refine(const MatchSet& matches, const FeatureMap& F_a,
                        const FeatureMap& F_b, const RefineParams& params);  // camera.cpp:239-271
struct PinholeProjection {
  Vec2 pixel;
  double J[6];  // 2x3 row-major
};
// camera.cpp:293-303; throws std::domain_error for z <= 0
PinholeProjection pinhole_project(const Vec3& x, const PinholeIntrinsics& K);

// ------------------------------------------------------------ tracking.cpp
struct RobustWeightParams {  // tracking.hpp:26-34
  double sigma2_point = 1e-2;
  double sigma2_ray = 1e-3;
  double sigma2_pixel = 4.0;
  double q_min = 0.0;
  double q_min_fraction = 0.1;
  double huber_delta = 1.345;
  double distance_weight = 0.01;
};

enum class TrackMode { kRay = 0, kPoint = 1, kPixel = 2 };  // tracking.hpp:40

struct ResidualBlock {  // tracking.hpp:46-52
  double residual[4] = {0, 0, 0, 0};
  double jacobian[28] = {0};  // 4x7 row-major
  double weight[4] = {0, 0, 0, 0};
  double info = 0.0;
  bool used = false;
};

double robust_weight(double q, double sigma2, double q_min);  // tracking.cpp:10-13
double huber_cost(double e, double delta);                    // tracking.cpp:24-26
double huber_factor(double e, double delta);                  // tracking.cpp:28-30
double median_confidence(const MatchSet& m);                  // tracking.cpp:32-42
std::vector<ResidualBlock> residual_blocks(const Sim3& T, const MatchSet& matches,
                                           const Pointmap& X_ref, const Pointmap& X_src,
                                           TrackMode mode, const RobustWeightParams& params,
                                           const PinholeIntrinsics* K);  // tracking.cpp:46-132
double block_cost(const std::vector<ResidualBlock>& blocks, const RobustWeightParams& params,
                  TrackMode mode);  // tracking.cpp:134-147

struct SolvePoseParams {  // tracking.hpp:82-91
  RobustWeightParams weights;
  MatchParams matching;
  RefineParams refinement;
  bool refine_features = true;
  int max_iterations = 20;
  double update_tol = 1e-6;
  int min_valid_matches = 12;
  std::optional<PinholeIntrinsics> intrinsics;
};

struct TrackResult {  // tracking.hpp:93-99
  Sim3 T_kf;
  MatchSet matches;
  std::vector<double> cost_trace;
  int iterations = 0;
  bool lost = false;
};

// The GN loop of solve_pose (tracking.cpp:165-225) on given matches.
TrackResult track_given_matches(const Pointmap& canonical, const Pointmap& X_f_f,
                                const MatchSet& matches, const Sim3& init, TrackMode mode,
                                const SolvePoseParams& params);
// solve_pose, tracking.cpp:149-226
TrackResult solve_pose(const Pointmap& canonical, const Pointmap& X_f_f,
                       const Pointmap& X_k_f, const FeatureMap& F_f, const FeatureMap& F_k,
                       const Sim3& init, TrackMode mode, const SolvePoseParams& params,
                       const MatchSet* match_seed);
// fuse_canonical, tracking.cpp:228-247
void fuse_canonical(Pointmap& canonical, std::vector<double>& canonical_conf,
                    const Pointmap& X_k_f, const std::vector<double>& confidence,
                    const Sim3& T_kf);
// keyframe_decision, tracking.cpp:249-257
bool keyframe_decision(const MatchSet& matches, int height, int width, double omega_k);

// ------------------------------------------------------------- backend.cpp
struct Edge {  // backend.hpp:18-22 (keyframes by index)
  int i = -1, j = -1;
  MatchSet matches;
};
struct Graph {  // backend.hpp:24-32
  std::vector<Pointmap> canonicals;
  std::vector<Sim3> poses;
  std::vector<Edge> edges;
  int anchor = -1;  // index_of(anchor_id)
};
struct BackendParams {  // backend.hpp:38-46
  RobustWeightParams weights;
  TrackMode mode = TrackMode::kRay;
  std::optional<PinholeIntrinsics> intrinsics;
  int max_iterations = 10;
  double update_tol = 1e-6;
  double damping_init = 1e-6;
  int damping_retries = 3;
};
struct AssembledSystem {  // backend.hpp:48-51, dense 7N x 7N row-major
  int dim = 0;
  std::vector<double> hessian;
  std::vector<double> gradient;
};
struct OptimizeResult {  // backend.hpp:59-63
  int iterations = 0;
  std::vector<double> cost_trace;
  bool converged = false;
};

AssembledSystem assemble_system(const Graph& g, const BackendParams& p);  // backend.cpp:91-173
double backend_cost(const Graph& g, const BackendParams& p);             // backend.cpp:175-190
// backend.cpp:192-256; pose_trace receives the poses after each iteration.
OptimizeResult global_optimize(Graph& g, const BackendParams& p,
                               std::vector<std::vector<Sim3>>* pose_trace);
// SimplicialLDLT factor+solve restatement (envelope LDL^T, natural order).
bool sparse_ldlt_solve(int n, const std::vector<double>& A, const std::vector<double>& b,
                       std::vector<double>* x);

// Per-edge relative-frame normal equations of both directions (for the
// edge-sharded backend's parity tests): 72 doubles per edge.
void backend_edge_terms(const Graph& g, const BackendParams& p, int e, double* out72);

}  // namespace orc
