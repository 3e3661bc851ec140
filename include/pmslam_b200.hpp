// pmslam_b200.hpp — header-only C++17 host mirror of the reference's
// matching / tracking / optimiser API (/root/reference/proj/include/pmslam/
// {camera,tracking,backend}.hpp) over the C ABI of pmx.h.
//
// Same function names, argument meaning and error behaviour as the reference:
// contract violations throw std::invalid_argument / std::domain_error,
// algorithmic outcomes are result fields.  Types are Eigen-free (the reference's
// are Eigen-typed; INTEGRATION.md shows the thin Eigen adapter a pmslam
// maintainer adds on top).  Link: -L<repo>/paper_2412_12392_b200/csrc -lpmx_cuda
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pmx.h"

namespace pmslam_b200 {

// ------------------------------------------------------------------ errors
inline void check(pmx_context* ctx, int status) {
  if (status == PMX_OK) return;
  const std::string msg = ctx ? pmx_last_error(ctx) : "pmx error";
  if (status == PMX_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (status == PMX_ERR_DOMAIN) throw std::domain_error(msg);
  throw std::runtime_error("pmx status " + std::to_string(status) + ": " + msg);
}

// One device + stream; all calls below take host data (PMX_MEM_HOST).
class Context {
 public:
  explicit Context(int device = 0) {
    pmx_context* c = nullptr;
    const int s = pmx_create(device, &c);
    if (s != PMX_OK) throw std::runtime_error("pmx_create failed (no sm_100 device?)");
    ctx_.reset(c);
  }
  pmx_context* get() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(pmx_context* c) const { pmx_destroy(c); }
  };
  std::unique_ptr<pmx_context, Del> ctx_;
};

// ------------------------------------------------------------------- types
struct Pointmap {  // camera.hpp:17-31 (fp32 storage, as the PMPAIR01 stream)
  int height = 0, width = 0;
  std::vector<float> xyz;      // H*W*3
  std::vector<uint8_t> valid;  // H*W (empty = all valid)
  Pointmap() = default;
  Pointmap(int h, int w) : height(h), width(w), xyz((size_t)h * w * 3, 0.0f), valid((size_t)h * w, 1) {}
  int size() const { return height * width; }
  int index(int u, int v) const { return v * width + u; }
  pmx_pointmap view() const { return {height, width, xyz.data(), valid.empty() ? nullptr : valid.data()}; }
};

struct FeatureMap {  // camera.hpp:55-71 (fp16 descriptors, pixel-major)
  int height = 0, width = 0, dim = 0;
  std::vector<uint16_t> descriptors;    // H*W*dim IEEE fp16 bits
  std::vector<float> match_confidence;  // H*W
  pmx_featuremap view() const { return {height, width, dim, descriptors.data(), match_confidence.data()}; }
};

struct Match {  // camera.hpp:73-78
  int pixel_a = -1, pixel_b = -1;
  double confidence = 0.0;
  bool valid = false;
};

struct MatchSet {  // camera.hpp:80-89
  std::vector<Match> matches;
  int valid_count() const {
    int n = 0;
    for (const auto& m : matches) n += m.valid;
    return n;
  }
};

using Sim3Pose = pmx_sim3;  // R (row-major), t, s
inline Sim3Pose identity_pose() {
  Sim3Pose T;
  pmx_sim3_identity(&T);
  return T;
}

struct TrackResult {  // tracking.hpp:93-99
  Sim3Pose T_kf;
  MatchSet matches;
  std::vector<double> cost_trace;
  int iterations = 0;
  bool lost = false;
};

struct Keyframe {  // tracking.hpp:16-24 (the fields the hot path touches)
  Pointmap canonical;
  std::vector<float> canonical_confidence;
  Sim3Pose T_WC = identity_pose();
};

struct FramePrediction {  // tracking.hpp:73-80
  Pointmap X_f_f, X_k_f;
  std::vector<float> C_f, C_k;
  FeatureMap F_f, F_k;
};

struct Edge {  // backend.hpp:18-22 (keyframe indices)
  int i = -1, j = -1;
  MatchSet matches;
};

struct Graph {  // backend.hpp:24-32
  std::vector<Keyframe> keyframes;
  std::vector<Edge> edges;
  int anchor = -1;
};

struct OptimizeResult {  // backend.hpp:59-63
  int iterations = 0;
  std::vector<double> cost_trace;
  bool converged = false;
};

struct AssembledSystem {  // backend.hpp:48-51 (dense row-major)
  int dim = 0;
  std::vector<double> hessian, gradient;
};

inline pmx_match_params default_match_params() {
  pmx_match_params p;
  pmx_default_match_params(&p);
  return p;
}
inline pmx_refine_params default_refine_params() {
  pmx_refine_params p;
  pmx_default_refine_params(&p);
  return p;
}
inline pmx_solve_pose_params default_solve_pose_params() {
  pmx_solve_pose_params p;
  pmx_default_solve_pose_params(&p);
  return p;
}
inline pmx_backend_params default_backend_params() {
  pmx_backend_params p;
  pmx_default_backend_params(&p);
  return p;
}

namespace detail {
struct SoA {
  std::vector<int32_t> pa, pb;
  std::vector<float> q;
  std::vector<uint8_t> v;
  explicit SoA(size_t n) : pa(n), pb(n), q(n), v(n) {}
  explicit SoA(const MatchSet& m) : SoA(m.matches.size()) {
    for (size_t k = 0; k < m.matches.size(); ++k) {
      pa[k] = m.matches[k].pixel_a;
      pb[k] = m.matches[k].pixel_b;
      q[k] = (float)m.matches[k].confidence;
      v[k] = m.matches[k].valid;
    }
  }
  pmx_matchset view() { return {(int64_t)pa.size(), pa.data(), pb.data(), q.data(), v.data()}; }
  MatchSet to_matchset() const {
    MatchSet m;
    m.matches.resize(pa.size());
    for (size_t k = 0; k < pa.size(); ++k) m.matches[k] = {pa[k], pb[k], (double)q[k], v[k] != 0};
    return m;
  }
};
}  // namespace detail

// --------------------------------------------------------- camera.hpp API
inline MatchSet match_pointmaps(Context& c, const Pointmap& X_a, const Pointmap& X_b_in_a, const FeatureMap& F_a,
                                const FeatureMap& F_b, const MatchSet* init = nullptr,
                                const pmx_match_params& params = default_match_params()) {
  detail::SoA out((size_t)X_b_in_a.size());
  auto o = out.view();
  std::unique_ptr<detail::SoA> seed;
  pmx_matchset sv{};
  if (init) {
    seed.reset(new detail::SoA(*init));
    sv = seed->view();
  }
  const auto a = X_a.view(), b = X_b_in_a.view();
  const auto fa = F_a.view(), fb = F_b.view();
  check(c.get(), pmx_match_pointmaps(c.get(), PMX_MEM_HOST, &a, &b, &fa, &fb, init ? &sv : nullptr, &params, &o));
  return out.to_matchset();
}

inline MatchSet feature_refine(Context& c, const MatchSet& matches, const FeatureMap& F_a, const FeatureMap& F_b,
                               const pmx_refine_params& params = default_refine_params()) {
  detail::SoA in(matches), out(matches.matches.size());
  auto i = in.view(), o = out.view();
  const auto fa = F_a.view(), fb = F_b.view();
  check(c.get(), pmx_feature_refine(c.get(), PMX_MEM_HOST, &i, &fa, &fb, &params, &o));
  return out.to_matchset();
}

// ------------------------------------------------------ retrieval.hpp API
// accept_loop_edge, retrieval.cpp:226-251 (std::optional<Edge> as in the reference).
inline std::optional<Edge> accept_loop_edge(Context& c, int kf_i, int kf_j, const Pointmap& X_i_i,
                                            const Pointmap& X_j_in_i, const FeatureMap& F_i, const FeatureMap& F_j,
                                            double omega_l, const pmx_match_params& match_params = default_match_params(),
                                            const pmx_refine_params& refine_params = default_refine_params()) {
  detail::SoA out((size_t)X_j_in_i.size());
  auto o = out.view();
  const pmx_pair p{X_i_i.view(), X_j_in_i.view(), F_i.view(), F_j.view(), nullptr};
  int32_t accepted = 0;
  check(c.get(), pmx_accept_loop_edges(c.get(), PMX_MEM_HOST, 1, &p, omega_l, &match_params, &refine_params, &o,
                                       &accepted));
  if (!accepted) return std::nullopt;
  Edge e;
  e.i = kf_i;
  e.j = kf_j;
  e.matches = out.to_matchset();
  return e;
}

// ------------------------------------------------------- pipeline.cpp API
// constrain_to_rays, pipeline.cpp:32-46 (calibrated mode), in place.
inline void constrain_to_rays(Context& c, Pointmap& pm, const pmx_intrinsics& K) {
  if (pm.valid.empty()) pm.valid.assign((size_t)pm.size(), 1);
  check(c.get(), pmx_constrain_to_rays(c.get(), PMX_MEM_HOST, pm.height, pm.width, pm.xyz.data(), pm.valid.data(),
                                       &K));
}

// ------------------------------------------------------- tracking.hpp API
inline TrackResult solve_pose(Context& c, const Keyframe& keyframe, const FramePrediction& pred,
                              const Sim3Pose& init, pmx_track_mode mode,
                              const pmx_solve_pose_params& params = default_solve_pose_params(),
                              const MatchSet* match_seed = nullptr) {
  detail::SoA out((size_t)pred.X_k_f.size());
  auto o = out.view();
  std::unique_ptr<detail::SoA> seed;
  pmx_matchset sv{};
  if (match_seed) {
    seed.reset(new detail::SoA(*match_seed));
    sv = seed->view();
  }
  const auto can = keyframe.canonical.view(), xf = pred.X_f_f.view(), xk = pred.X_k_f.view();
  const auto ff = pred.F_f.view(), fk = pred.F_k.view();
  pmx_track_result r;
  check(c.get(), pmx_solve_pose(c.get(), PMX_MEM_HOST, &can, &xf, &xk, &ff, &fk, &init, mode, &params,
                                match_seed ? &sv : nullptr, &r, &o));
  TrackResult t;
  t.T_kf = r.T_kf;
  t.iterations = r.iterations;
  t.lost = r.lost != 0;
  t.cost_trace.assign(r.cost_trace, r.cost_trace + r.cost_trace_len);
  t.matches = out.to_matchset();
  return t;
}

inline void fuse_canonical(Context& c, Keyframe& keyframe, const Pointmap& X_k_f, const std::vector<float>& confidence,
                           const Sim3Pose& T_kf) {
  Pointmap& can = keyframe.canonical;
  if (can.valid.empty()) can.valid.assign((size_t)can.size(), 1);
  if (keyframe.canonical_confidence.size() != (size_t)can.size())
    throw std::invalid_argument("fuse_canonical: confidence size mismatch");
  const auto xk = X_k_f.view();
  check(c.get(), pmx_fuse_canonical(c.get(), PMX_MEM_HOST, can.height, can.width, can.xyz.data(), can.valid.data(),
                                    keyframe.canonical_confidence.data(), &xk, confidence.data(), &T_kf));
}

// -------------------------------------------------------- backend.hpp API
namespace detail {
struct GraphView {
  std::vector<pmx_pointmap> cans;
  std::vector<pmx_sim3> poses;
  std::vector<int32_t> ei, ej;
  std::vector<SoA> soa;
  std::vector<pmx_matchset> ms;
  pmx_graph g{};
  explicit GraphView(const Graph& G) {
    for (const auto& kf : G.keyframes) {
      cans.push_back(kf.canonical.view());
      poses.push_back(kf.T_WC);
    }
    soa.reserve(G.edges.size());
    for (const auto& e : G.edges) {
      ei.push_back(e.i);
      ej.push_back(e.j);
      soa.emplace_back(e.matches);
    }
    for (auto& s : soa) ms.push_back(s.view());
    g = {(int32_t)cans.size(), cans.data(), poses.data(), G.anchor, (int32_t)ei.size(), ei.data(), ej.data(),
         ms.data()};
  }
};
}  // namespace detail

inline AssembledSystem assemble_system(Context& c, const Graph& G,
                                       const pmx_backend_params& params = default_backend_params()) {
  detail::GraphView v(G);
  AssembledSystem s;
  s.dim = 7 * (int)G.keyframes.size();
  s.hessian.assign((size_t)s.dim * s.dim, 0.0);
  s.gradient.assign((size_t)s.dim, 0.0);
  check(c.get(), pmx_assemble_system(c.get(), PMX_MEM_HOST, &v.g, &params, s.hessian.data(), s.gradient.data()));
  return s;
}

inline double backend_cost(Context& c, const Graph& G, const pmx_backend_params& params = default_backend_params()) {
  detail::GraphView v(G);
  double cost = 0.0;
  check(c.get(), pmx_backend_cost(c.get(), PMX_MEM_HOST, &v.g, &params, &cost));
  return cost;
}

inline OptimizeResult global_optimize(Context& c, Graph& G,
                                      const pmx_backend_params& params = default_backend_params()) {
  detail::GraphView v(G);
  pmx_optimize_result r;
  check(c.get(), pmx_global_optimize(c.get(), PMX_MEM_HOST, &v.g, &params, &r, nullptr));
  for (size_t k = 0; k < G.keyframes.size(); ++k) G.keyframes[k].T_WC = v.poses[k];
  OptimizeResult o;
  o.iterations = r.iterations;
  o.converged = r.converged != 0;
  o.cost_trace.assign(r.cost_trace, r.cost_trace + r.cost_trace_len);
  return o;
}

}  // namespace pmslam_b200
