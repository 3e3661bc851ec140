// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// The same flat C ABI as oracle_capi.h (orc_* symbols), implemented by the
// GENUINE reference sources /root/reference/proj/src/{lie,camera,tracking,
// backend}.cpp, compiled unmodified against the Eigen-API shim in
// eigen_shim/ (recipe: oracle/Makefile target `ref`, output
// oracle/_ref/libpmslam_ref.so).  tests/ load it next to liborc.so to pin the
// restatement (oracle.cpp) to the reference itself.
//
// Entry points the reference does not have (track_given_matches,
// normal_equations, backend_edge_terms, median_scene_distance, ldlt_solve,
// huber_*) are deliberately absent: the restatement's versions of those are
// pinned through the reference functions that contain them (solve_pose,
// match_pointmaps, assemble_system / backend_cost, global_optimize).
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oracle_capi.h"
#include "pmslam/backend.hpp"
#include "pmslam/camera.hpp"
#include "pmslam/lie.hpp"
#include "pmslam/tracking.hpp"

using namespace pmslam;

namespace {

thread_local std::string g_err;

double half_to_double(uint16_t h) {
  const int sign = h >> 15, exp = (h >> 10) & 0x1f, mant = h & 0x3ff;
  double v;
  if (exp == 0)
    v = std::ldexp((double)mant, -24);
  else if (exp == 31)
    v = mant ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
  else
    v = std::ldexp((double)(mant | 0x400), exp - 25);
  return sign ? -v : v;
}

Pointmap to_pointmap(const pmx_pointmap* p) {
  Pointmap pm(p->height, p->width);
  for (int i = 0; i < pm.size(); ++i) {
    pm.points[i] = Vec3(p->xyz[3 * i], p->xyz[3 * i + 1], p->xyz[3 * i + 2]);
    pm.valid[i] = p->valid ? (p->valid[i] ? 1 : 0) : 1;
  }
  return pm;
}

FeatureMap to_featuremap(const pmx_featuremap* f) {
  FeatureMap fm(f->height, f->width, f->dim);
  const int n = f->height * f->width;
  for (int i = 0; i < n; ++i) {
    for (int d = 0; d < f->dim; ++d) fm.descriptors(d, i) = half_to_double(f->descriptors[(size_t)i * f->dim + d]);
    fm.match_confidence[i] = f->match_confidence[i];
  }
  return fm;
}

MatchSet to_matchset(const orc_matchset* m) {
  MatchSet s;
  s.matches.resize(m->count);
  for (int64_t k = 0; k < m->count; ++k) {
    Match& x = s.matches[k];
    x.pixel_a = m->pixel_a[k];
    x.pixel_b = m->pixel_b ? m->pixel_b[k] : (int)k;
    x.confidence = m->confidence ? m->confidence[k] : 1.0;
    x.valid = m->valid ? m->valid[k] != 0 : true;
  }
  return s;
}

void from_matchset(const MatchSet& s, orc_matchset* m) {
  if ((int64_t)s.matches.size() > m->count) throw std::invalid_argument("output matchset too small");
  m->count = (int64_t)s.matches.size();
  for (size_t k = 0; k < s.matches.size(); ++k) {
    const Match& x = s.matches[k];
    m->pixel_a[k] = x.pixel_a;
    if (m->pixel_b) m->pixel_b[k] = x.pixel_b;
    m->confidence[k] = x.confidence;
    m->valid[k] = x.valid ? 1 : 0;
  }
}

Sim3Pose to_sim3(const pmx_sim3* T) {
  Mat3 R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R(r, c) = T->R[3 * r + c];
  return Sim3Pose(R, Vec3(T->t[0], T->t[1], T->t[2]), T->s);  // throws on s <= 0 (lie.cpp:94-96)
}

void from_sim3(const Sim3Pose& s, pmx_sim3* T) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) T->R[3 * r + c] = s.rotation()(r, c);
  for (int i = 0; i < 3; ++i) T->t[i] = s.translation()(i);
  T->s = s.scale();
}

IterProjParams to_iter(const pmx_iter_proj_params* p) {
  IterProjParams q;
  if (p) {
    q.lambda_init = p->lambda_init;
    q.lambda_up = p->lambda_up;
    q.lambda_down = p->lambda_down;
    q.angle_tol = p->angle_tol;
    q.max_iterations = p->max_iterations;
  }
  return q;
}

MatchParams to_match(const pmx_match_params* p) {
  MatchParams q;
  if (p) {
    q.projection = to_iter(&p->projection);
    q.invalidation_median_fraction = p->invalidation_median_fraction;
  }
  return q;
}

RefineParams to_refine(const pmx_refine_params* p) {
  RefineParams q;
  if (p) {
    q.levels.clear();
    for (int i = 0; i < p->num_levels; ++i) q.levels.push_back({p->stride[i], p->radius[i]});
  }
  return q;
}

RobustWeightParams to_weights(const pmx_robust_weight_params* p) {
  RobustWeightParams q;
  if (p) {
    q.sigma2_point = p->sigma2_point;
    q.sigma2_ray = p->sigma2_ray;
    q.sigma2_pixel = p->sigma2_pixel;
    q.q_min = p->q_min;
    q.q_min_fraction = p->q_min_fraction;
    q.huber_delta = p->huber_delta;
    q.distance_weight = p->distance_weight;
  }
  return q;
}

std::optional<PinholeIntrinsics> to_K(int32_t has, const pmx_intrinsics& k) {
  if (!has) return std::nullopt;
  PinholeIntrinsics K;
  K.fx = k.fx;
  K.fy = k.fy;
  K.cx = k.cx;
  K.cy = k.cy;
  return K;
}

SolvePoseParams to_solve(const pmx_solve_pose_params* p) {
  SolvePoseParams q;
  if (p) {
    q.weights = to_weights(&p->weights);
    q.matching = to_match(&p->matching);
    q.refinement = to_refine(&p->refinement);
    q.refine_features = p->refine_features != 0;
    q.max_iterations = p->max_iterations;
    q.update_tol = p->update_tol;
    q.min_valid_matches = p->min_valid_matches;
    q.intrinsics = to_K(p->has_intrinsics, p->intrinsics);
  }
  return q;
}

BackendParams to_backend(const pmx_backend_params* p) {
  BackendParams q;
  if (p) {
    q.weights = to_weights(&p->weights);
    q.mode = (TrackMode)p->mode;
    q.intrinsics = to_K(p->has_intrinsics, p->intrinsics);
    q.max_iterations = p->max_iterations;
    q.update_tol = p->update_tol;
    q.damping_init = p->damping_init;
    q.damping_retries = p->damping_retries;
  }
  return q;
}

// Keyframes by index: id = index, anchor_id = anchor_index (backend.hpp:18-32).
Graph to_graph(const orc_graph* g) {
  Graph G;
  for (int k = 0; k < g->num_keyframes; ++k) {
    Keyframe kf;
    kf.id = k;
    kf.canonical = to_pointmap(&g->canonicals[k]);
    kf.T_WC = to_sim3(&g->poses[k]);
    G.keyframes.push_back(std::move(kf));
  }
  G.anchor_id = g->anchor_index;
  for (int e = 0; e < g->num_edges; ++e) {
    Edge E;
    E.i = g->edge_i[e];
    E.j = g->edge_j[e];
    E.matches = to_matchset(&g->edge_matches[e]);
    G.edges.push_back(std::move(E));
  }
  return G;
}

void fill_track_result(const TrackResult& r, pmx_track_result* out) {
  from_sim3(r.T_kf, &out->T_kf);
  out->iterations = r.iterations;
  out->lost = r.lost ? 1 : 0;
  out->cost_trace_len = (int)std::min<size_t>(r.cost_trace.size(), PMX_MAX_TRACE);
  for (int i = 0; i < out->cost_trace_len; ++i) out->cost_trace[i] = r.cost_trace[i];
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return PMX_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PMX_ERR_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return PMX_ERR_DOMAIN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PMX_ERR_INVALID_ARGUMENT;
  }
}

template <class W>
void parallel_for(int begin, int end, int threads, W&& work) {
  if (threads <= 1) {
    for (int e = begin; e < end; ++e) work(e);
    return;
  }
  std::vector<std::thread> pool;
  std::atomic<int> next{begin};
  std::string err;
  std::mutex mu;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (int e = next++; e < end; e = next++) {
        try {
          work(e);
        } catch (const std::exception& ex) {
          std::lock_guard<std::mutex> lk(mu);
          err = ex.what();
        }
      }
    });
  for (auto& th : pool) th.join();
  if (!err.empty()) throw std::invalid_argument(err);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// Identifies this build: the genuine reference sources (1) vs the restatement.
int orc_is_reference(void) { return 1; }

int orc_normalize_rays(const pmx_pointmap* pm, double* rays, double* distances, uint8_t* valid) {
  return guard([&] {
    const RayMap rm = normalize_rays(to_pointmap(pm));
    for (size_t i = 0; i < rm.rays.size(); ++i) {
      for (int c = 0; c < 3; ++c) rays[3 * i + c] = rm.rays[i](c);
      distances[i] = rm.distances[i];
      valid[i] = rm.valid[i];
    }
  });
}

int orc_interpolate_ray(const pmx_pointmap* pm, int64_t n, const double* p, double* ray, double* J,
                        uint8_t* ok) {
  return guard([&] {
    const RayMap rm = normalize_rays(to_pointmap(pm));
    for (int64_t k = 0; k < n; ++k) {
      Eigen::Matrix<double, 3, 2> j = Eigen::Matrix<double, 3, 2>::Zero();
      const auto r = interpolate_ray(rm, Vec2(p[2 * k], p[2 * k + 1]), &j);
      ok[k] = r ? 1 : 0;
      for (int c = 0; c < 3; ++c) ray[3 * k + c] = r ? (*r)(c) : 0.0;
      if (J)  // column-major 3x2 (J[3 c + r]), as oracle_capi
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 2; ++b) J[6 * k + 3 * b + a] = r ? j(a, b) : 0.0;
    }
  });
}

int orc_iterative_project(const pmx_pointmap* pm, int64_t n, const float* x, const double* p0,
                          const pmx_iter_proj_params* params, double* pixel, uint8_t* converged,
                          int32_t* iterations) {
  return guard([&] {
    const RayMap rm = normalize_rays(to_pointmap(pm));
    const IterProjParams ip = to_iter(params);
    for (int64_t k = 0; k < n; ++k) {
      const ProjectResult r =
          iterative_project(rm, Vec3(x[3 * k], x[3 * k + 1], x[3 * k + 2]), Vec2(p0[2 * k], p0[2 * k + 1]), ip);
      pixel[2 * k] = r.pixel.x();
      pixel[2 * k + 1] = r.pixel.y();
      converged[k] = r.converged ? 1 : 0;
      iterations[k] = r.iterations;
    }
  });
}

int orc_match_pointmaps(const pmx_pointmap* X_a, const pmx_pointmap* X_b_in_a, const pmx_featuremap* F_a,
                        const pmx_featuremap* F_b, const orc_matchset* init, const pmx_match_params* params,
                        orc_matchset* out) {
  return guard([&] {
    MatchSet seed;
    if (init) seed = to_matchset(init);
    const MatchSet m = match_pointmaps(to_pointmap(X_a), to_pointmap(X_b_in_a), to_featuremap(F_a),
                                       to_featuremap(F_b), init ? &seed : nullptr, to_match(params));
    from_matchset(m, out);
  });
}

int orc_feature_refine(const orc_matchset* in, const pmx_featuremap* F_a, const pmx_featuremap* F_b,
                       const pmx_refine_params* params, orc_matchset* out) {
  return guard([&] {
    const MatchSet m = feature_refine(to_matchset(in), to_featuremap(F_a), to_featuremap(F_b), to_refine(params));
    from_matchset(m, out);
  });
}

int orc_match_batch(int32_t num_pairs, const pmx_pair* pairs, const orc_matchset* const* inits,
                    const pmx_match_params* params, const pmx_refine_params* refine, orc_matchset* outs,
                    int32_t threads) {
  return guard([&] {
    const MatchParams mp = to_match(params);
    const RefineParams rp = to_refine(refine);
    parallel_for(0, num_pairs, threads, [&](int e) {
      const pmx_pair& P = pairs[e];
      const FeatureMap Fa = to_featuremap(&P.F_a), Fb = to_featuremap(&P.F_b);
      MatchSet seed;
      const bool has_seed = inits && inits[e];
      if (has_seed) seed = to_matchset(inits[e]);
      MatchSet m =
          match_pointmaps(to_pointmap(&P.X_a), to_pointmap(&P.X_b_in_a), Fa, Fb, has_seed ? &seed : nullptr, mp);
      if (refine) m = feature_refine(m, Fa, Fb, rp);
      from_matchset(m, &outs[e]);
    });
  });
}

int orc_match_stats(const orc_matchset* m, int32_t num_pixels_a, int64_t* valid_count, double* unique_fraction) {
  return guard([&] {
    const MatchSet s = to_matchset(m);
    *valid_count = s.valid_count();
    *unique_fraction = s.unique_pixel_fraction(num_pixels_a);
  });
}

int orc_keyframe_decision(const orc_matchset* m, int32_t height, int32_t width, double omega_k, int32_t* out) {
  return guard([&] { *out = keyframe_decision(to_matchset(m), height, width, omega_k) ? 1 : 0; });
}

int orc_residual_blocks(const pmx_sim3* T, const orc_matchset* matches, const pmx_pointmap* X_ref,
                        const pmx_pointmap* X_src, pmx_track_mode mode, const pmx_robust_weight_params* params,
                        const pmx_intrinsics* K, double* residual, double* jacobian, double* weight, double* info,
                        uint8_t* used) {
  return guard([&] {
    std::optional<PinholeIntrinsics> Ki;
    if (K) Ki = to_K(1, *K);
    const auto blocks = residual_blocks(to_sim3(T), to_matchset(matches), to_pointmap(X_ref), to_pointmap(X_src),
                                        (TrackMode)mode, to_weights(params), Ki ? &*Ki : nullptr);
    for (size_t k = 0; k < blocks.size(); ++k) {
      const auto& b = blocks[k];
      for (int r = 0; r < 4; ++r) {
        residual[4 * k + r] = b.residual(r);
        weight[4 * k + r] = b.weight(r);
        for (int c = 0; c < 7; ++c) jacobian[28 * k + 7 * r + c] = b.jacobian(r, c);  // row-major 4x7
      }
      info[k] = b.info;
      used[k] = b.used ? 1 : 0;
    }
  });
}

int orc_solve_pose(const pmx_pointmap* canonical, const pmx_pointmap* X_f_f, const pmx_pointmap* X_k_f,
                   const pmx_featuremap* F_f, const pmx_featuremap* F_k, const pmx_sim3* init, pmx_track_mode mode,
                   const pmx_solve_pose_params* params, const orc_matchset* match_seed, pmx_track_result* result,
                   orc_matchset* matches_out) {
  return guard([&] {
    Keyframe kf;
    kf.canonical = to_pointmap(canonical);
    FramePrediction pred;
    pred.X_f_f = to_pointmap(X_f_f);
    pred.X_k_f = to_pointmap(X_k_f);
    pred.F_f = to_featuremap(F_f);
    pred.F_k = to_featuremap(F_k);
    MatchSet seed;
    if (match_seed) seed = to_matchset(match_seed);
    const TrackResult r =
        solve_pose(kf, pred, to_sim3(init), (TrackMode)mode, to_solve(params), match_seed ? &seed : nullptr);
    fill_track_result(r, result);
    if (matches_out) from_matchset(r.matches, matches_out);
  });
}

int orc_fuse_canonical(int32_t height, int32_t width, double* canonical_xyz, uint8_t* canonical_valid,
                       double* canonical_confidence, const pmx_pointmap* X_k_f, const float* confidence,
                       const pmx_sim3* T_kf) {
  return guard([&] {
    Keyframe kf;
    kf.canonical = Pointmap(height, width);
    kf.canonical_confidence = ConfidenceMap(height, width);
    const int n = height * width;
    ConfidenceMap c(height, width);
    for (int i = 0; i < n; ++i) {
      kf.canonical.points[i] = Vec3(canonical_xyz[3 * i], canonical_xyz[3 * i + 1], canonical_xyz[3 * i + 2]);
      kf.canonical.valid[i] = canonical_valid[i];
      kf.canonical_confidence.values[i] = canonical_confidence[i];
      c.values[i] = confidence[i];
    }
    fuse_canonical(kf, to_pointmap(X_k_f), c, to_sim3(T_kf));
    for (int i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) canonical_xyz[3 * i + k] = kf.canonical.points[i](k);
      canonical_valid[i] = kf.canonical.valid[i];
      canonical_confidence[i] = kf.canonical_confidence.values[i];
    }
  });
}

// Dense row-major 7N x 7N Hessian (the SparseMatrix's entries) and gradient.
int orc_assemble_system(const orc_graph* g, const pmx_backend_params* p, double* H, double* grad) {
  return guard([&] {
    const Graph G = to_graph(g);
    const AssembledSystem sys = assemble_system(G, to_backend(p));
    const Eigen::Index n = sys.hessian.rows();
    std::memset(H, 0, sizeof(double) * n * n);
    for (Eigen::Index c = 0; c < sys.hessian.outerSize(); ++c)
      for (Eigen::SparseMatrix<double>::InnerIterator it(sys.hessian, c); it; ++it) H[it.row() * n + it.col()] = it.value();
    for (Eigen::Index i = 0; i < n; ++i) grad[i] = sys.gradient(i);
  });
}

int orc_backend_cost(const orc_graph* g, const pmx_backend_params* p, double* cost) {
  return guard([&] { *cost = backend_cost(to_graph(g), to_backend(p)); });
}

// pose_trace (nullable): the poses after each iteration it = 0 .. iterations-1,
// obtained by re-running global_optimize from the initial graph with
// max_iterations = it + 1 (the reference records no trace; its loop is
// deterministic, so the first it + 1 iterations are those of the full run).
int orc_global_optimize(orc_graph* g, const pmx_backend_params* p, pmx_optimize_result* result, pmx_sim3* pose_trace) {
  return guard([&] {
    const Graph G0 = to_graph(g);
    const BackendParams bp = to_backend(p);
    Graph G = G0;
    const OptimizeResult r = global_optimize(G, bp);
    const int n = g->num_keyframes;
    if (pose_trace) {
      const int rows = r.converged ? r.iterations : std::max(0, r.iterations - 1);
      for (int it = 0; it < rows; ++it) {
        Graph Gi = G0;
        BackendParams bi = bp;
        bi.max_iterations = it + 1;
        global_optimize(Gi, bi);
        for (int k = 0; k < n; ++k) from_sim3(Gi.keyframes[k].T_WC, &pose_trace[(size_t)it * n + k]);
      }
    }
    for (int k = 0; k < n; ++k) from_sim3(G.keyframes[k].T_WC, &g->poses[k]);
    result->iterations = r.iterations;
    result->converged = r.converged ? 1 : 0;
    result->cost_trace_len = (int)std::min<size_t>(r.cost_trace.size(), PMX_MAX_TRACE);
    for (int i = 0; i < result->cost_trace_len; ++i) result->cost_trace[i] = r.cost_trace[i];
  });
}

double orc_robust_weight(double q, double sigma2, double q_min) { return robust_weight(q, sigma2, q_min); }

int orc_sim3_exp(const double* tau7, pmx_sim3* out) {
  return guard([&] {
    Tangent7 t;
    for (int i = 0; i < 7; ++i) t(i) = tau7[i];
    from_sim3(Sim3Pose::exp(t), out);
  });
}
int orc_sim3_log(const pmx_sim3* T, double* tau7) {
  return guard([&] {
    const Tangent7 t = to_sim3(T).log();
    for (int i = 0; i < 7; ++i) tau7[i] = t(i);
  });
}
int orc_sim3_compose(const pmx_sim3* a, const pmx_sim3* b, pmx_sim3* out) {
  return guard([&] { from_sim3(to_sim3(a) * to_sim3(b), out); });
}
int orc_sim3_inverse(const pmx_sim3* a, pmx_sim3* out) {
  return guard([&] { from_sim3(to_sim3(a).inverse(), out); });
}
int orc_sim3_adjoint(const pmx_sim3* a, double* ad49) {
  return guard([&] {
    const Mat7 m = to_sim3(a).adjoint();
    for (int r = 0; r < 7; ++r)
      for (int c = 0; c < 7; ++c) ad49[7 * r + c] = m(r, c);
  });
}

}  // extern "C"
