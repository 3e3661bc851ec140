// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).  Flat-array C ABI over
// the FP64 restatement; converts fp32 / fp16 inputs to double exactly.
#include "oracle_capi.h"

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <mutex>
#include <limits>
#include <cmath>
#include <algorithm>

#include "oracle.hpp"

using namespace orc;

namespace {

thread_local std::string g_err;

double half_to_double(uint16_t h) {
  const int sign = h >> 15;
  const int exp = (h >> 10) & 0x1f;
  const int mant = h & 0x3ff;
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
  Pointmap pm;
  pm.height = p->height;
  pm.width = p->width;
  const int n = pm.size();
  pm.points.resize(n);
  pm.valid.assign(n, 1);
  for (int i = 0; i < n; ++i) {
    pm.points[i] = Vec3(p->xyz[3 * i], p->xyz[3 * i + 1], p->xyz[3 * i + 2]);
    if (p->valid) pm.valid[i] = p->valid[i] ? 1 : 0;
  }
  return pm;
}

FeatureMap to_featuremap(const pmx_featuremap* f) {
  FeatureMap fm;
  fm.height = f->height;
  fm.width = f->width;
  fm.dim = f->dim;
  const size_t n = (size_t)f->height * f->width;
  fm.descriptors.resize(n * f->dim);
  for (size_t i = 0; i < n * f->dim; ++i) fm.descriptors[i] = half_to_double(f->descriptors[i]);
  fm.match_confidence.resize(n);
  for (size_t i = 0; i < n; ++i) fm.match_confidence[i] = f->match_confidence[i];
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

Sim3 to_sim3(const pmx_sim3* T) {
  Sim3 s;
  for (int i = 0; i < 9; ++i) s.R.m[i] = T->R[i];
  s.t = Vec3(T->t[0], T->t[1], T->t[2]);
  s.s = T->s;
  if (!(s.s > 0.0)) throw std::invalid_argument("Sim3Pose: scale must be positive");
  return s;
}

void from_sim3(const Sim3& s, pmx_sim3* T) {
  for (int i = 0; i < 9; ++i) T->R[i] = s.R.m[i];
  for (int i = 0; i < 3; ++i) T->t[i] = s.t[i];
  T->s = s.s;
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
    if (p->has_intrinsics)
      q.intrinsics = PinholeIntrinsics{p->intrinsics.fx, p->intrinsics.fy, p->intrinsics.cx,
                                       p->intrinsics.cy};
  }
  return q;
}

BackendParams to_backend(const pmx_backend_params* p) {
  BackendParams q;
  if (p) {
    q.weights = to_weights(&p->weights);
    q.mode = (TrackMode)p->mode;
    if (p->has_intrinsics)
      q.intrinsics = PinholeIntrinsics{p->intrinsics.fx, p->intrinsics.fy, p->intrinsics.cx,
                                       p->intrinsics.cy};
    q.max_iterations = p->max_iterations;
    q.update_tol = p->update_tol;
    q.damping_init = p->damping_init;
    q.damping_retries = p->damping_retries;
  }
  return q;
}

Graph to_graph(const orc_graph* g) {
  Graph G;
  for (int k = 0; k < g->num_keyframes; ++k) {
    G.canonicals.push_back(to_pointmap(&g->canonicals[k]));
    G.poses.push_back(to_sim3(&g->poses[k]));
  }
  G.anchor = g->anchor_index;
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

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_normalize_rays(const pmx_pointmap* pm, double* rays, double* distances, uint8_t* valid) {
  return guard([&] {
    const RayMap rm = normalize_rays(to_pointmap(pm));
    for (size_t i = 0; i < rm.rays.size(); ++i) {
      for (int c = 0; c < 3; ++c) rays[3 * i + c] = rm.rays[i][c];
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
      Vec3 r;
      double j[6] = {0, 0, 0, 0, 0, 0};
      ok[k] = interpolate_ray(rm, p[2 * k], p[2 * k + 1], &r, j) ? 1 : 0;
      for (int c = 0; c < 3; ++c) ray[3 * k + c] = ok[k] ? r[c] : 0.0;
      if (J)
        for (int c = 0; c < 6; ++c) J[6 * k + c] = j[c];
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
      const ProjectResult r = iterative_project(rm, Vec3(x[3 * k], x[3 * k + 1], x[3 * k + 2]),
                                                Vec2{p0[2 * k], p0[2 * k + 1]}, ip);
      pixel[2 * k] = r.pixel.x;
      pixel[2 * k + 1] = r.pixel.y;
      converged[k] = r.converged ? 1 : 0;
      iterations[k] = r.iterations;
    }
  });
}

int orc_median_scene_distance(const pmx_pointmap* pm, double* out) {
  return guard([&] { *out = median_scene_distance(to_pointmap(pm)); });
}

int orc_match_pointmaps(const pmx_pointmap* X_a, const pmx_pointmap* X_b_in_a,
                        const pmx_featuremap* F_a, const pmx_featuremap* F_b,
                        const orc_matchset* init, const pmx_match_params* params,
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
    const MatchSet m =
        feature_refine(to_matchset(in), to_featuremap(F_a), to_featuremap(F_b), to_refine(params));
    from_matchset(m, out);
  });
}

int orc_match_batch(int32_t num_pairs, const pmx_pair* pairs, const orc_matchset* const* inits,
                    const pmx_match_params* params, const pmx_refine_params* refine,
                    orc_matchset* outs, int32_t threads) {
  return guard([&] {
    const MatchParams mp = to_match(params);
    const RefineParams rp = to_refine(refine);
    auto work = [&](int e) {
      const pmx_pair& P = pairs[e];
      const FeatureMap Fa = to_featuremap(&P.F_a), Fb = to_featuremap(&P.F_b);
      MatchSet seed;
      const bool has_seed = inits && inits[e];
      if (has_seed) seed = to_matchset(inits[e]);
      MatchSet m = match_pointmaps(to_pointmap(&P.X_a), to_pointmap(&P.X_b_in_a), Fa, Fb,
                                   has_seed ? &seed : nullptr, mp);
      if (refine) m = feature_refine(m, Fa, Fb, rp);
      from_matchset(m, &outs[e]);
    };
    if (threads <= 1) {
      for (int e = 0; e < num_pairs; ++e) work(e);
      return;
    }
    std::vector<std::thread> pool;
    std::atomic<int> next{0};
    std::string err;
    std::mutex mu;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&] {
        for (int e = next++; e < num_pairs; e = next++) {
          try {
            work(e);
          } catch (const std::exception& ex) {
            std::lock_guard<std::mutex> lk(mu);
            err = ex.what();
          }
        }
      });
    }
    for (auto& th : pool) th.join();
    if (!err.empty()) throw std::invalid_argument(err);
  });
}

int orc_match_stats(const orc_matchset* m, int32_t num_pixels_a, int64_t* valid_count,
                    double* unique_fraction) {
  return guard([&] {
    const MatchSet s = to_matchset(m);
    *valid_count = s.valid_count();
    *unique_fraction = s.unique_pixel_fraction(num_pixels_a);
  });
}

int orc_keyframe_decision(const orc_matchset* m, int32_t height, int32_t width, double omega_k,
                          int32_t* out) {
  return guard([&] { *out = keyframe_decision(to_matchset(m), height, width, omega_k) ? 1 : 0; });
}

int orc_residual_blocks(const pmx_sim3* T, const orc_matchset* matches, const pmx_pointmap* X_ref,
                        const pmx_pointmap* X_src, pmx_track_mode mode,
                        const pmx_robust_weight_params* params, const pmx_intrinsics* K,
                        double* residual, double* jacobian, double* weight, double* info,
                        uint8_t* used) {
  return guard([&] {
    PinholeIntrinsics Ki;
    if (K) Ki = PinholeIntrinsics{K->fx, K->fy, K->cx, K->cy};
    const auto blocks = residual_blocks(to_sim3(T), to_matchset(matches), to_pointmap(X_ref),
                                        to_pointmap(X_src), (TrackMode)mode, to_weights(params),
                                        K ? &Ki : nullptr);
    for (size_t k = 0; k < blocks.size(); ++k) {
      const auto& b = blocks[k];
      for (int r = 0; r < 4; ++r) {
        residual[4 * k + r] = b.residual[r];
        weight[4 * k + r] = b.weight[r];
      }
      for (int r = 0; r < 28; ++r) jacobian[28 * k + r] = b.jacobian[r];
      info[k] = b.info;
      used[k] = b.used ? 1 : 0;
    }
  });
}

int orc_normal_equations(const pmx_sim3* T, const orc_matchset* matches, const pmx_pointmap* X_ref,
                         const pmx_pointmap* X_src, pmx_track_mode mode,
                         const pmx_robust_weight_params* params, const pmx_intrinsics* K,
                         double* H, double* g, double* cost, int64_t* used) {
  return guard([&] {
    PinholeIntrinsics Ki;
    if (K) Ki = PinholeIntrinsics{K->fx, K->fy, K->cx, K->cy};
    const RobustWeightParams w = to_weights(params);
    const auto blocks = residual_blocks(to_sim3(T), to_matchset(matches), to_pointmap(X_ref),
                                        to_pointmap(X_src), (TrackMode)mode, w, K ? &Ki : nullptr);
    for (int i = 0; i < 49; ++i) H[i] = 0.0;
    for (int i = 0; i < 7; ++i) g[i] = 0.0;
    int64_t u = 0;
    for (const auto& b : blocks) {
      if (!b.used) continue;
      ++u;
      for (int r = 0; r < 4; ++r) {
        const double wr = b.weight[r];
        if (wr <= 0.0) continue;
        const double* j = b.jacobian + r * 7;
        for (int a = 0; a < 7; ++a) {
          for (int c = 0; c < 7; ++c) H[a * 7 + c] += wr * j[a] * j[c];
          g[a] += wr * j[a] * b.residual[r];
        }
      }
    }
    *cost = block_cost(blocks, w, (TrackMode)mode);
    if (used) *used = u;
  });
}

int orc_track_given_matches(const pmx_pointmap* canonical, const pmx_pointmap* X_f_f,
                            const orc_matchset* matches, const pmx_sim3* init, pmx_track_mode mode,
                            const pmx_solve_pose_params* params, pmx_track_result* result) {
  return guard([&] {
    const SolvePoseParams sp = to_solve(params);
    if (mode == PMX_TRACK_PIXEL && !sp.intrinsics)
      throw std::invalid_argument("residual_blocks: pixel mode requires intrinsics");
    const TrackResult r = track_given_matches(to_pointmap(canonical), to_pointmap(X_f_f),
                                              to_matchset(matches), to_sim3(init), (TrackMode)mode, sp);
    fill_track_result(r, result);
  });
}

int orc_solve_pose(const pmx_pointmap* canonical, const pmx_pointmap* X_f_f,
                   const pmx_pointmap* X_k_f, const pmx_featuremap* F_f, const pmx_featuremap* F_k,
                   const pmx_sim3* init, pmx_track_mode mode, const pmx_solve_pose_params* params,
                   const orc_matchset* match_seed, pmx_track_result* result,
                   orc_matchset* matches_out) {
  return guard([&] {
    MatchSet seed;
    if (match_seed) seed = to_matchset(match_seed);
    const TrackResult r =
        solve_pose(to_pointmap(canonical), to_pointmap(X_f_f), to_pointmap(X_k_f),
                   to_featuremap(F_f), to_featuremap(F_k), to_sim3(init), (TrackMode)mode,
                   to_solve(params), match_seed ? &seed : nullptr);
    fill_track_result(r, result);
    if (matches_out) from_matchset(r.matches, matches_out);
  });
}

int orc_fuse_canonical(int32_t height, int32_t width, double* canonical_xyz,
                       uint8_t* canonical_valid, double* canonical_confidence,
                       const pmx_pointmap* X_k_f, const float* confidence, const pmx_sim3* T_kf) {
  return guard([&] {
    Pointmap can;
    can.height = height;
    can.width = width;
    const int n = height * width;
    can.points.resize(n);
    can.valid.resize(n);
    std::vector<double> conf(n), c(n);
    for (int i = 0; i < n; ++i) {
      can.points[i] = Vec3(canonical_xyz[3 * i], canonical_xyz[3 * i + 1], canonical_xyz[3 * i + 2]);
      can.valid[i] = canonical_valid[i];
      conf[i] = canonical_confidence[i];
      c[i] = confidence[i];
    }
    fuse_canonical(can, conf, to_pointmap(X_k_f), c, to_sim3(T_kf));
    for (int i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) canonical_xyz[3 * i + k] = can.points[i][k];
      canonical_valid[i] = can.valid[i];
      canonical_confidence[i] = conf[i];
    }
  });
}

int orc_assemble_system(const orc_graph* g, const pmx_backend_params* p, double* H, double* grad) {
  return guard([&] {
    const Graph G = to_graph(g);
    const AssembledSystem sys = assemble_system(G, to_backend(p));
    std::memcpy(H, sys.hessian.data(), sizeof(double) * sys.hessian.size());
    std::memcpy(grad, sys.gradient.data(), sizeof(double) * sys.gradient.size());
  });
}

int orc_backend_cost(const orc_graph* g, const pmx_backend_params* p, double* cost) {
  return guard([&] { *cost = backend_cost(to_graph(g), to_backend(p)); });
}

int orc_backend_edge_terms(const orc_graph* g, const pmx_backend_params* p, int32_t edge_begin,
                           int32_t edge_end, double* out, int32_t threads) {
  return guard([&] {
    const Graph G = to_graph(g);
    const BackendParams bp = to_backend(p);
    if (threads <= 1) {
      for (int e = edge_begin; e < edge_end; ++e)
        backend_edge_terms(G, bp, e, out + (size_t)(e - edge_begin) * PMX_EDGE_TERMS);
      return;
    }
    std::vector<std::thread> pool;
    std::atomic<int> next{edge_begin};
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (int e = next++; e < edge_end; e = next++)
          backend_edge_terms(G, bp, e, out + (size_t)(e - edge_begin) * PMX_EDGE_TERMS);
      });
    for (auto& th : pool) th.join();
  });
}

int orc_global_optimize(orc_graph* g, const pmx_backend_params* p, pmx_optimize_result* result,
                        pmx_sim3* pose_trace) {
  return guard([&] {
    Graph G = to_graph(g);
    const BackendParams bp = to_backend(p);
    std::vector<std::vector<Sim3>> trace;
    const OptimizeResult r = global_optimize(G, bp, &trace);
    for (int k = 0; k < g->num_keyframes; ++k) from_sim3(G.poses[k], &g->poses[k]);
    result->iterations = r.iterations;
    result->converged = r.converged ? 1 : 0;
    result->cost_trace_len = (int)std::min<size_t>(r.cost_trace.size(), PMX_MAX_TRACE);
    for (int i = 0; i < result->cost_trace_len; ++i) result->cost_trace[i] = r.cost_trace[i];
    if (pose_trace) {
      for (size_t it = 0; it < trace.size(); ++it)
        for (int k = 0; k < g->num_keyframes; ++k)
          from_sim3(trace[it][k], &pose_trace[it * g->num_keyframes + k]);
    }
  });
}

int orc_ldlt_solve(int32_t n, const double* A, const double* b, double* x, int32_t* ok) {
  return guard([&] {
    std::vector<double> Av(A, A + (size_t)n * n), bv(b, b + n), xv;
    *ok = sparse_ldlt_solve(n, Av, bv, &xv) ? 1 : 0;
    if (*ok) std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}

double orc_robust_weight(double q, double sigma2, double q_min) { return robust_weight(q, sigma2, q_min); }
double orc_huber_cost(double e, double delta) { return huber_cost(e, delta); }
double orc_huber_factor(double e, double delta) { return huber_factor(e, delta); }

int orc_sim3_exp(const double* tau7, pmx_sim3* out) {
  return guard([&] {
    Vec7 t;
    for (int i = 0; i < 7; ++i) t[i] = tau7[i];
    from_sim3(Sim3::exp(t), out);
  });
}
int orc_sim3_log(const pmx_sim3* T, double* tau7) {
  return guard([&] {
    const Vec7 t = to_sim3(T).log();
    for (int i = 0; i < 7; ++i) tau7[i] = t[i];
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
    for (int i = 0; i < 49; ++i) ad49[i] = m[i];
  });
}

}  // extern "C"
