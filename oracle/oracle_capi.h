/* ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
 * C ABI of the FP64 CPU restatement, shaped like include/pmx.h so one pytest
 * harness can drive both.  Matchsets carry FP64 confidences (the reference's
 * Match::confidence is double, camera.hpp:76). */
#ifndef ORC_CAPI_H_
#define ORC_CAPI_H_
#include "../include/pmx.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_matchset {
  int64_t count;
  int32_t* pixel_a;
  int32_t* pixel_b; /* NULL => dense (pixel_b = index) on input; must be non-NULL on output */
  double* confidence;
  uint8_t* valid;
} orc_matchset;

typedef struct orc_graph {
  int32_t num_keyframes;
  const pmx_pointmap* canonicals;
  pmx_sim3* poses;
  int32_t anchor_index;
  int32_t num_edges;
  const int32_t* edge_i;
  const int32_t* edge_j;
  const orc_matchset* edge_matches;
} orc_graph;

const char* orc_last_error(void);
int orc_normalize_rays(const pmx_pointmap* pm, double* rays, double* distances, uint8_t* valid);
int orc_interpolate_ray(const pmx_pointmap* pm, int64_t n, const double* p, double* ray,
                        double* J, uint8_t* ok);
int orc_iterative_project(const pmx_pointmap* pm, int64_t n, const float* x, const double* p0,
                          const pmx_iter_proj_params* params, double* pixel, uint8_t* converged,
                          int32_t* iterations);
int orc_median_scene_distance(const pmx_pointmap* pm, double* out);
int orc_match_pointmaps(const pmx_pointmap* X_a, const pmx_pointmap* X_b_in_a,
                        const pmx_featuremap* F_a, const pmx_featuremap* F_b,
                        const orc_matchset* init, const pmx_match_params* params,
                        orc_matchset* out);
int orc_feature_refine(const orc_matchset* in, const pmx_featuremap* F_a,
                       const pmx_featuremap* F_b, const pmx_refine_params* params,
                       orc_matchset* out);
/* Batched match(+refine) of independent pairs on `threads` host threads
 * (the all-core CPU baseline; threads <= 1 runs single-threaded). */
int orc_match_batch(int32_t num_pairs, const pmx_pair* pairs, const orc_matchset* const* inits,
                    const pmx_match_params* params, const pmx_refine_params* refine,
                    orc_matchset* outs, int32_t threads);
int orc_match_stats(const orc_matchset* m, int32_t num_pixels_a, int64_t* valid_count,
                    double* unique_fraction);
int orc_keyframe_decision(const orc_matchset* m, int32_t height, int32_t width, double omega_k,
                          int32_t* out);
int orc_residual_blocks(const pmx_sim3* T, const orc_matchset* matches, const pmx_pointmap* X_ref,
                        const pmx_pointmap* X_src, pmx_track_mode mode,
                        const pmx_robust_weight_params* params, const pmx_intrinsics* K,
                        double* residual, double* jacobian, double* weight, double* info,
                        uint8_t* used);
int orc_normal_equations(const pmx_sim3* T, const orc_matchset* matches, const pmx_pointmap* X_ref,
                         const pmx_pointmap* X_src, pmx_track_mode mode,
                         const pmx_robust_weight_params* params, const pmx_intrinsics* K,
                         double* H, double* g, double* cost, int64_t* used);
int orc_track_given_matches(const pmx_pointmap* canonical, const pmx_pointmap* X_f_f,
                            const orc_matchset* matches, const pmx_sim3* init,
                            pmx_track_mode mode, const pmx_solve_pose_params* params,
                            pmx_track_result* result);
int orc_solve_pose(const pmx_pointmap* canonical, const pmx_pointmap* X_f_f,
                   const pmx_pointmap* X_k_f, const pmx_featuremap* F_f, const pmx_featuremap* F_k,
                   const pmx_sim3* init, pmx_track_mode mode, const pmx_solve_pose_params* params,
                   const orc_matchset* match_seed, pmx_track_result* result,
                   orc_matchset* matches_out);
/* canonical_xyz double[HW*3] in/out, canonical_valid in/out, conf double in/out */
int orc_fuse_canonical(int32_t height, int32_t width, double* canonical_xyz,
                       uint8_t* canonical_valid, double* canonical_confidence,
                       const pmx_pointmap* X_k_f, const float* confidence, const pmx_sim3* T_kf);
int orc_assemble_system(const orc_graph* g, const pmx_backend_params* p, double* H, double* grad);
int orc_backend_cost(const orc_graph* g, const pmx_backend_params* p, double* cost);
int orc_backend_edge_terms(const orc_graph* g, const pmx_backend_params* p, int32_t edge_begin,
                           int32_t edge_end, double* out, int32_t threads);
int orc_global_optimize(orc_graph* g, const pmx_backend_params* p, pmx_optimize_result* result,
                        pmx_sim3* pose_trace);
int orc_ldlt_solve(int32_t n, const double* A, const double* b, double* x, int32_t* ok);
/* tracking.cpp:10-30 scalar helpers. */
double orc_robust_weight(double q, double sigma2, double q_min);
double orc_huber_cost(double e, double delta);
double orc_huber_factor(double e, double delta);
/* Lie helpers for tests: exp/log/compose/inverse/adjoint. */
int orc_sim3_exp(const double* tau7, pmx_sim3* out);
int orc_sim3_log(const pmx_sim3* T, double* tau7);
int orc_sim3_compose(const pmx_sim3* a, const pmx_sim3* b, pmx_sim3* out);
int orc_sim3_inverse(const pmx_sim3* a, pmx_sim3* out);
int orc_sim3_adjoint(const pmx_sim3* a, double* ad49);

#ifdef __cplusplus
}
#endif
#endif
