/*
 * pmx.h — C ABI of the B200-native hot paths of pointmap SLAM
 * (MASt3R-SLAM, arXiv 2412.12392), drop-in for the matching / tracking /
 * optimiser API of the CPU reference "pmslam".
 *
 * Every entry point is extern "C", takes plain pointers + sizes and POD
 * structs, and returns an int status (PMX_OK = 0).  No C++ types or
 * exceptions cross this boundary; pmx_last_error() returns a message.  The
 * reference's exceptions map to status codes:
 *   std::invalid_argument -> PMX_ERR_INVALID_ARGUMENT
 *   std::domain_error     -> PMX_ERR_DOMAIN
 * Algorithmic outcomes (match validity, tracking lost, non-convergence) are
 * result fields, never errors — exactly as in the reference.
 *
 * Memory: every compute entry point takes a pmx_memory flag.  PMX_MEM_HOST
 * means every array argument is host memory (the library stages it through
 * pinned buffers, H2D, computes, D2H, and returns synchronously).
 * PMX_MEM_DEVICE means every array argument is device memory on the
 * context's device; the call is enqueued on the context stream and returns
 * without synchronising, except where a host-side scalar result is returned
 * (those entry points synchronise).
 *
 * Layouts (all row-major, pixel index = v * width + u, reference
 * include/pmslam/camera.hpp:16-31):
 *   pointmap      xyz: float32[H*W*3] interleaved, valid: uint8[H*W] or NULL
 *   featuremap    descriptors: IEEE fp16 bits uint16[H*W*dim], pixel-major
 *                 (the reference's dim x HW column-per-pixel Eigen matrix,
 *                 camera.hpp:59), match_confidence: float32[H*W]
 *   matchset      SoA: pixel_a int32, pixel_b int32 (NULL = dense, pixel_b
 *                 implicit = index), confidence float32, valid uint8
 *   Sim(3) pose   double R[9] (row-major), t[3], s   (lie.hpp:35-70)
 */
#ifndef PMX_H_
#define PMX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMX_ABI_VERSION 1

enum pmx_status {
  PMX_OK = 0,
  PMX_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  PMX_ERR_DOMAIN = 2,           /* std::domain_error in the reference */
  PMX_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
  PMX_ERR_NO_DEVICE = 4,        /* no sm_100 device / extension unusable */
  PMX_ERR_OUT_OF_MEMORY = 5,
  PMX_ERR_NCCL = 6
};

typedef enum pmx_memory { PMX_MEM_HOST = 0, PMX_MEM_DEVICE = 1 } pmx_memory;

/* TrackMode, reference include/pmslam/tracking.hpp:40 */
typedef enum pmx_track_mode {
  PMX_TRACK_RAY = 0,
  PMX_TRACK_POINT = 1,
  PMX_TRACK_PIXEL = 2
} pmx_track_mode;

typedef struct pmx_context pmx_context;

/* ---------------------------------------------------------------- types */

typedef struct pmx_pointmap { /* Pointmap, camera.hpp:17-31 */
  int32_t height;
  int32_t width;
  const float* xyz;     /* H*W*3 */
  const uint8_t* valid; /* H*W, NULL = all valid */
} pmx_pointmap;

typedef struct pmx_featuremap { /* FeatureMap, camera.hpp:55-71 */
  int32_t height;
  int32_t width;
  int32_t dim;
  const uint16_t* descriptors;   /* H*W*dim fp16 bits, pixel-major */
  const float* match_confidence; /* H*W (Q) */
} pmx_featuremap;

typedef struct pmx_matchset { /* MatchSet, camera.hpp:73-89 */
  int64_t count;
  int32_t* pixel_a;
  int32_t* pixel_b; /* NULL => pixel_b[k] == k (dense, as match_pointmaps emits) */
  float* confidence;
  uint8_t* valid;
} pmx_matchset;

typedef struct pmx_sim3 { /* Sim3Pose, lie.hpp:36-70: x -> s R x + t */
  double R[9];
  double t[3];
  double s;
} pmx_sim3;

typedef struct pmx_iter_proj_params { /* IterProjParams, camera.hpp:102-108 */
  double lambda_init;
  double lambda_up;
  double lambda_down;
  double angle_tol; /* rad */
  int32_t max_iterations;
} pmx_iter_proj_params;

typedef struct pmx_match_params { /* MatchParams, camera.hpp:126-131 */
  pmx_iter_proj_params projection;
  double invalidation_median_fraction;
} pmx_match_params;

#define PMX_MAX_REFINE_LEVELS 8
typedef struct pmx_refine_params { /* RefineParams, camera.hpp:140-143 */
  int32_t num_levels;
  int32_t stride[PMX_MAX_REFINE_LEVELS];
  int32_t radius[PMX_MAX_REFINE_LEVELS];
} pmx_refine_params;

typedef struct pmx_intrinsics { /* PinholeIntrinsics, camera.hpp:91-96 */
  double fx, fy, cx, cy;
} pmx_intrinsics;

typedef struct pmx_robust_weight_params { /* RobustWeightParams, tracking.hpp:26-34 */
  double sigma2_point;
  double sigma2_ray;
  double sigma2_pixel;
  double q_min;
  double q_min_fraction;
  double huber_delta;
  double distance_weight;
} pmx_robust_weight_params;

typedef struct pmx_solve_pose_params { /* SolvePoseParams, tracking.hpp:82-91 */
  pmx_robust_weight_params weights;
  pmx_match_params matching;
  pmx_refine_params refinement;
  int32_t refine_features;
  int32_t max_iterations;
  double update_tol;
  int32_t min_valid_matches;
  int32_t has_intrinsics;
  pmx_intrinsics intrinsics;
} pmx_solve_pose_params;

#define PMX_MAX_TRACE 64
typedef struct pmx_track_result { /* TrackResult, tracking.hpp:93-99 (matches returned separately) */
  pmx_sim3 T_kf;
  int32_t iterations;
  int32_t lost;
  int32_t cost_trace_len;
  double cost_trace[PMX_MAX_TRACE];
} pmx_track_result;

typedef struct pmx_backend_params { /* BackendParams, backend.hpp:38-46 */
  pmx_robust_weight_params weights;
  pmx_track_mode mode;
  int32_t has_intrinsics;
  pmx_intrinsics intrinsics;
  int32_t max_iterations;
  double update_tol;
  double damping_init;
  int32_t damping_retries;
} pmx_backend_params;

typedef struct pmx_graph { /* Graph, backend.hpp:18-32 (keyframes by index) */
  int32_t num_keyframes;
  const pmx_pointmap* canonicals; /* [num_keyframes] */
  pmx_sim3* poses;                /* [num_keyframes] T_WC, in/out for optimize */
  int32_t anchor_index;           /* index_of(anchor_id), -1 = none */
  int32_t num_edges;
  const int32_t* edge_i;          /* [num_edges] keyframe indices (host memory) */
  const int32_t* edge_j;
  const pmx_matchset* edge_matches; /* [num_edges]: pixel_a in i, pixel_b in j */
} pmx_graph;

typedef struct pmx_optimize_result { /* OptimizeResult, backend.hpp:59-63 */
  int32_t iterations;
  int32_t converged;
  int32_t cost_trace_len;
  double cost_trace[PMX_MAX_TRACE];
} pmx_optimize_result;

/* One edge of a batched matching call: the pair prediction of edge (a, b). */
typedef struct pmx_pair { /* arguments of match_pointmaps, camera.hpp:135-138 */
  pmx_pointmap X_a;
  pmx_pointmap X_b_in_a;
  pmx_featuremap F_a;
  pmx_featuremap F_b;
  const pmx_matchset* init; /* nullable seed */
} pmx_pair;

/* ------------------------------------------------------------ defaults */
void pmx_default_match_params(pmx_match_params* p);
void pmx_default_refine_params(pmx_refine_params* p);
void pmx_default_robust_weight_params(pmx_robust_weight_params* p);
void pmx_default_solve_pose_params(pmx_solve_pose_params* p);
void pmx_default_backend_params(pmx_backend_params* p);
void pmx_sim3_identity(pmx_sim3* T);
/* Host-only FP64 Sim(3) helpers (no device needed): left-plus retract
 * Exp(tau) * T (lie.hpp:54) and relative_pose T_wi^-1 T_wj (lie.cpp:171). */
void pmx_sim3_retract(const pmx_sim3* T, const double* tau7, pmx_sim3* out);
void pmx_sim3_relative(const pmx_sim3* T_wi, const pmx_sim3* T_wj, pmx_sim3* out);

/* ----------------------------------------------------------- lifecycle */
int pmx_abi_version(void);
int pmx_create(int device, pmx_context** out);
int pmx_destroy(pmx_context* ctx);
const char* pmx_last_error(const pmx_context* ctx);
/* Adopt an existing cudaStream_t (NULL = the context's own stream). */
int pmx_set_stream(pmx_context* ctx, void* cuda_stream);
void* pmx_get_stream(pmx_context* ctx);
int pmx_synchronize(pmx_context* ctx);
/* Number of pmx kernels launched by this context since creation. */
int64_t pmx_kernel_launch_count(const pmx_context* ctx);
/* Live kernel timing: when enabled, the hot kernels (k_match, k_track_gn,
 * k_edge_terms, k_ldlt) are bracketed by CUDA events on the context stream.
 * pmx_profile_get synchronises and returns the summed duration (ms) and the
 * launch count of every bracketed launch of `kernel` since the last reset. */
int pmx_profile_enable(pmx_context* ctx, int on);
int pmx_profile_reset(pmx_context* ctx);
int pmx_profile_get(pmx_context* ctx, const char* kernel, double* total_ms, int64_t* launches);
/* Device-side loops (the global_optimize GN loop) run as one CUDA graph with
 * a conditional WHILE node (default on): the loop stops on the device when it
 * converges, without enqueueing max_iterations iterations.  Off: the loop is
 * enqueued kernel by kernel (every kernel checks the stop flag), which is what
 * the per-kernel profile brackets need. */
int pmx_set_device_graphs(pmx_context* ctx, int on);

/* -------------------------------------------------- matching (camera.cpp) */

/* normalize_rays, camera.hpp:100 / camera.cpp:39-56 (FP64, as the
 * reference's RayMap).  rays: double[H*W*3], distances: double[H*W],
 * valid: uint8[H*W]. */
int pmx_normalize_rays(pmx_context* ctx, pmx_memory mem, const pmx_pointmap* pm,
                       double* rays, double* distances, uint8_t* valid);

/* interpolate_ray, camera.hpp:118-119 / camera.cpp:58-100, at n continuous
 * pixels p (double[n*2], (u, v)) of the ray map of `pm`: ray (double[n*3]),
 * jacobian (double[n*6], nullable; column-major 3x2: d/du then d/dv),
 * ok (uint8[n]: 0 = std::nullopt, ray / jacobian then zero). */
int pmx_interpolate_ray(pmx_context* ctx, pmx_memory mem, const pmx_pointmap* pm, int64_t n,
                        const double* p, double* ray, double* jacobian, uint8_t* ok);

/* median_scene_distance, camera.cpp:178-191 (the reference's file-local
 * helper behind match_pointmaps' 3D invalidation threshold, exported as a
 * test surface): the rank floor(n/2) FP64 norm over valid pixels with
 * norm > 1e-12, 0 when there are none.  out: one double (host memory for
 * PMX_MEM_HOST, device memory for PMX_MEM_DEVICE). */
int pmx_median_scene_distance(pmx_context* ctx, pmx_memory mem, const pmx_pointmap* pm, double* out);

/* iterative_project, camera.hpp:123-124 / camera.cpp:115-174, for a batch
 * of n query points x (float[n*3]) with seeds p0 (double[n*2]) against the
 * ray map of `pm`.  Outputs pixel (double[n*2]), converged (uint8[n]),
 * iterations (int32[n]). */
int pmx_iterative_project(pmx_context* ctx, pmx_memory mem, const pmx_pointmap* pm,
                          int64_t n, const float* x, const double* p0,
                          const pmx_iter_proj_params* params, double* pixel,
                          uint8_t* converged, int32_t* iterations);

/* match_pointmaps, camera.hpp:135-138 / camera.cpp:195-237.
 * out must hold H_b*W_b entries (pixel_b may be NULL: dense). */
int pmx_match_pointmaps(pmx_context* ctx, pmx_memory mem, const pmx_pointmap* X_a,
                        const pmx_pointmap* X_b_in_a, const pmx_featuremap* F_a,
                        const pmx_featuremap* F_b, const pmx_matchset* init,
                        const pmx_match_params* params, pmx_matchset* out);

/* feature_refine, camera.hpp:147-148 / camera.cpp:239-271. */
int pmx_feature_refine(pmx_context* ctx, pmx_memory mem, const pmx_matchset* in,
                       const pmx_featuremap* F_a, const pmx_featuremap* F_b,
                       const pmx_refine_params* params, pmx_matchset* out);

/* Fused match_pointmaps + feature_refine over a batch of independent edges
 * (the loop-edge / per-keyframe "Match" step, retrieval.cpp:232-234,
 * tracking.cpp:156-162).  refine may be NULL (projective matching only).
 * outs[e] must hold H_b*W_b entries. */
int pmx_match_batch(pmx_context* ctx, pmx_memory mem, int32_t num_pairs,
                    const pmx_pair* pairs, const pmx_match_params* params,
                    const pmx_refine_params* refine, pmx_matchset* outs);

/* accept_loop_edge, retrieval.cpp:226-251, for a batch of candidate loop
 * edges (X_a = X_i_i, X_b_in_a = X_j_in_i, F_a = F_i, F_b = F_j): match +
 * refine, then the descriptor-agreement gate (exact FP64 dot of the two
 * endpoints' descriptors < 0.5 invalidates a match, retrieval.cpp:238-244),
 * then accepted[e] = valid_fraction() >= omega_l (else the reference's
 * nullopt).  outs[e] receives the gated matches (Edge::matches). */
int pmx_accept_loop_edges(pmx_context* ctx, pmx_memory mem, int32_t num_pairs, const pmx_pair* pairs,
                          double omega_l, const pmx_match_params* params, const pmx_refine_params* refine,
                          pmx_matchset* outs, int32_t* accepted);

/* MatchSet::valid_count / unique_pixel_fraction, camera.cpp:10-28, and
 * keyframe_decision, tracking.cpp:249-257. */
int pmx_match_stats(pmx_context* ctx, pmx_memory mem, const pmx_matchset* m,
                    int32_t num_pixels_a, int64_t* valid_count,
                    double* unique_pixel_fraction);
int pmx_keyframe_decision(pmx_context* ctx, pmx_memory mem, const pmx_matchset* m,
                          int32_t height, int32_t width, double omega_k,
                          int32_t* new_keyframe);

/* ------------------------------------- inputs of the path (pipeline.cpp) */

/* One PMPAIR01 pair record (StreamPredictor::predict, pipeline.cpp:642-676):
 * 8-byte magic, then float32 X_i_in_i [HW*3], X_j_in_i [HW*3], C_i [HW],
 * C_j [HW], D_i [HW*dim] (pixel-major), D_j, Q_i [HW], Q_j [HW].  Unpacked
 * into the layouts above: valid = allFinite(point) (pipeline.cpp:536-543),
 * descriptors converted to fp16 (inexact_descriptors counts values that are
 * not exactly representable: parity with the reference needs 0).  All
 * output arrays are caller-allocated (host or device per mem, like record). */
typedef struct pmx_pair_record {
  float* X_i;
  uint8_t* valid_i;
  float* X_j;
  uint8_t* valid_j;
  float* C_i;
  float* C_j;
  uint16_t* D_i;
  uint16_t* D_j;
  float* Q_i;
  float* Q_j;
} pmx_pair_record;
int pmx_ingest_pair_record(pmx_context* ctx, pmx_memory mem, const void* record, int64_t nbytes,
                           int32_t height, int32_t width, int32_t dim, pmx_pair_record* out,
                           int64_t* inexact_descriptors);

/* constrain_to_rays, pipeline.cpp:32-46 (calibrated mode), in place:
 * valid points with z > 0 become z * ((u - cx) / fx, (v - cy) / fy, 1),
 * z <= 0 invalidates. */
int pmx_constrain_to_rays(pmx_context* ctx, pmx_memory mem, int32_t height, int32_t width, float* xyz,
                          uint8_t* valid, const pmx_intrinsics* K);

/* ------------------------------------------------- tracking (tracking.cpp) */

/* residual_blocks, tracking.hpp:56-59 / tracking.cpp:46-132, materialised
 * (test/parity entry point; the hot path never writes these):
 * residual double[n*4], jacobian double[n*28] (row-major 4x7),
 * weight double[n*4], info double[n], used uint8[n]. */
int pmx_residual_blocks(pmx_context* ctx, pmx_memory mem, const pmx_sim3* T_ref_src,
                        const pmx_matchset* matches, const pmx_pointmap* X_ref,
                        const pmx_pointmap* X_src, pmx_track_mode mode,
                        const pmx_robust_weight_params* params,
                        const pmx_intrinsics* K, double* residual, double* jacobian,
                        double* weight, double* info, uint8_t* used);

/* Fused normal equations of one residual pass (tracking.cpp:134-147 and
 * :188-198): H = sum w J^T J (double[49]), g = sum w J^T r (double[7]),
 * cost = block_cost (double), used count.  Host outputs, synchronises. */
int pmx_normal_equations(pmx_context* ctx, pmx_memory mem, const pmx_sim3* T_ref_src,
                         const pmx_matchset* matches, const pmx_pointmap* X_ref,
                         const pmx_pointmap* X_src, pmx_track_mode mode,
                         const pmx_robust_weight_params* params,
                         const pmx_intrinsics* K, double* H, double* g, double* cost,
                         int64_t* used);

/* The IRLS/LM Gauss-Newton loop of solve_pose (tracking.cpp:165-225) on
 * GIVEN matches (frame pixel_a, keyframe pixel_b).  params->weights.q_min is
 * recomputed from the matches (tracking.cpp:170-171). */
int pmx_track_given_matches(pmx_context* ctx, pmx_memory mem,
                            const pmx_pointmap* canonical, const pmx_pointmap* X_f_f,
                            const pmx_matchset* matches, const pmx_sim3* init,
                            pmx_track_mode mode, const pmx_solve_pose_params* params,
                            pmx_track_result* result);

/* solve_pose, tracking.hpp:105-108 / tracking.cpp:149-226: match + refine
 * (frame = a, keyframe image = b) then the GN loop.  matches_out (H*W
 * entries) receives TrackResult::matches; may be NULL. */
int pmx_solve_pose(pmx_context* ctx, pmx_memory mem, const pmx_pointmap* canonical,
                   const pmx_pointmap* X_f_f, const pmx_pointmap* X_k_f,
                   const pmx_featuremap* F_f, const pmx_featuremap* F_k,
                   const pmx_sim3* init, pmx_track_mode mode,
                   const pmx_solve_pose_params* params, const pmx_matchset* match_seed,
                   pmx_track_result* result, pmx_matchset* matches_out);

/* fuse_canonical, tracking.hpp:112-113 / tracking.cpp:228-247, in place on
 * the keyframe canonical (xyz, valid, confidence). */
int pmx_fuse_canonical(pmx_context* ctx, pmx_memory mem, int32_t height, int32_t width,
                       float* canonical_xyz, uint8_t* canonical_valid,
                       float* canonical_confidence, const pmx_pointmap* X_k_f,
                       const float* confidence, const pmx_sim3* T_kf);

/* --------------------------------------------------- backend (backend.cpp) */

/* assemble_system, backend.hpp:57 / backend.cpp:91-173, dense output:
 * H double[7N*7N] row-major (gauge-fixed), g double[7N]. Host outputs. */
int pmx_assemble_system(pmx_context* ctx, pmx_memory mem, const pmx_graph* graph,
                        const pmx_backend_params* params, double* H, double* g);

/* backend_cost, backend.hpp:72 / backend.cpp:175-190. */
int pmx_backend_cost(pmx_context* ctx, pmx_memory mem, const pmx_graph* graph,
                     const pmx_backend_params* params, double* cost);

/* global_optimize, backend.hpp:69 / backend.cpp:192-256.  graph->poses is
 * updated in place (host memory always).  pose_trace (nullable) receives
 * the poses after every iteration: pmx_sim3[max_iterations * N]. */
int pmx_global_optimize(pmx_context* ctx, pmx_memory mem, pmx_graph* graph,
                        const pmx_backend_params* params, pmx_optimize_result* result,
                        pmx_sim3* pose_trace);

/* Edge-sharded building blocks (multi-GPU backend, one process per GPU).
 * pmx_backend_edge_terms: for the edges [edge_begin, edge_end) of graph,
 * the per-edge relative-frame normal equations of both directions:
 * out double[(edge_end-edge_begin) * PMX_EDGE_TERMS] (device or host per
 * mem), layout per edge: dir1 {H 28 (upper, row-major), g 7, cost 1},
 * dir2 {H 28, g 7, cost 1}. */
#define PMX_EDGE_TERMS 72
int pmx_backend_edge_terms(pmx_context* ctx, pmx_memory mem, const pmx_graph* graph,
                           const pmx_backend_params* params, int32_t edge_begin,
                           int32_t edge_end, double* out);

/* Given all edges' terms (host or device per mem, [num_edges*72]), assemble
 * the gauge-fixed dense system, solve with the damping-retry schedule of
 * backend.cpp:208-230, and return tau (double[7N]) and the summed cost.
 * solved = 0 when every attempt failed (state intact). */
int pmx_backend_solve_terms(pmx_context* ctx, pmx_memory mem, const pmx_graph* graph,
                            const pmx_backend_params* params, const double* terms,
                            double* tau, double* cost, int32_t* solved);

/* Prepared graph: a graph staged once (canonicals packed, the frozen matches
 * of edges [edge_begin, edge_end) compacted, the solver's frontal plan built)
 * for repeated per-iteration calls at changing poses — the building blocks
 * of the edge-sharded backend without per-iteration re-staging.  Edges
 * outside the range may carry empty match sets.  poses are host memory;
 * terms / tau are device memory (float64, layouts as above). */
typedef struct pmx_prepared_graph pmx_prepared_graph;
int pmx_graph_prepare(pmx_context* ctx, pmx_memory mem, const pmx_graph* graph,
                      const pmx_backend_params* params, int32_t edge_begin, int32_t edge_end,
                      pmx_prepared_graph** out);
/* terms of the prepared edge range: out double[(edge_end-edge_begin)*PMX_EDGE_TERMS] */
int pmx_graph_edge_terms(pmx_context* ctx, pmx_prepared_graph* pg, const pmx_sim3* poses, double* out);
/* all edges' terms (double[num_edges*PMX_EDGE_TERMS]) -> cost, damped solve, tau double[7N] */
int pmx_graph_solve(pmx_context* ctx, pmx_prepared_graph* pg, const pmx_sim3* poses, const double* terms,
                    double* tau, double* cost, int32_t* solved);
int pmx_graph_release(pmx_context* ctx, pmx_prepared_graph* pg);

/* NCCL communicator of the context (one process per GPU).  Rank 0 creates
 * the 128-byte unique id, the caller ships it to every rank (any side
 * channel, e.g. torch.distributed), and every rank initialises with its
 * rank / rank count.  NCCL is resolved at run time (libnccl.so.2, shared
 * with a copy already loaded in the process). */
int pmx_nccl_unique_id(pmx_context* ctx, uint8_t id[128]);
int pmx_nccl_init(pmx_context* ctx, const uint8_t id[128], int32_t rank, int32_t nranks);

/* global_optimize (backend.cpp:192-256) edge-sharded over the context's
 * communicator, every iteration enqueued on the context stream with no host
 * round trip: each rank's prepared edge range (pmx_graph_prepare) gives its
 * per-edge terms, one ncclReduce(sum) of the E x 72 FP64 terms reaches rank
 * 0, rank 0 assembles, solves (damping retries) and decides accept / revert
 * (on FP64 costs when ambiguous), and broadcasts of the loop state and tau
 * keep every rank's FP64 poses identical.  poses: host pmx_sim3[N], in/out
 * (every rank).  pose_trace (nullable, rank 0): as pmx_global_optimize.
 * timings (nullable): double[3] device ms of the call spent in
 * accumulation / communication / rank-0 solve.  Without a communicator the
 * loop runs on one process (rank 0, all edges prepared). */
int pmx_graph_optimize_sharded(pmx_context* ctx, pmx_prepared_graph* pg, pmx_sim3* poses,
                               pmx_optimize_result* result, pmx_sim3* pose_trace, double* timings);

/* Dense symmetric LDL^T solve of A x = b (n x n, row-major, FP64) on the
 * device, no pivoting, fails (status field 0) on an exactly zero pivot —
 * the factorisation semantics of SimplicialLDLT (backend.cpp:216-218). */
int pmx_ldlt_solve(pmx_context* ctx, pmx_memory mem, int32_t n, const double* A,
                   const double* b, double* x, int32_t* ok);

#ifdef __cplusplus
}
#endif
#endif /* PMX_H_ */
