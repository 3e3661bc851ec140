// C-ABI glue of libpmx_cuda.so: context lifecycle, reference defaults,
// exception -> status translation.  The compute lives in match.cu,
// track.cu and backend.cu (pmx_impl_* entry points).
#include <cstring>
#include <string>

#include "nccl_dl.cuh"
#include "pmx_common.cuh"

using pmx::Context;

extern "C" {
int pmx_impl_match_batch(pmx_context*, pmx_memory, int32_t, const pmx_pair*, const pmx_match_params*,
                         const pmx_refine_params*, pmx_matchset*);
int pmx_impl_accept_loop_edges(pmx_context*, pmx_memory, int32_t, const pmx_pair*, double,
                               const pmx_match_params*, const pmx_refine_params*, pmx_matchset*, int32_t*);
int pmx_impl_ingest_pair_record(pmx_context*, pmx_memory, const void*, int64_t, int32_t, int32_t, int32_t,
                                pmx_pair_record*, int64_t*);
int pmx_impl_constrain_to_rays(pmx_context*, pmx_memory, int32_t, int32_t, float*, uint8_t*, const pmx_intrinsics*);
int pmx_impl_graph_prepare(pmx_context*, pmx_memory, const pmx_graph*, const pmx_backend_params*, int32_t, int32_t,
                           pmx_prepared_graph**);
int pmx_impl_graph_edge_terms(pmx_context*, pmx_prepared_graph*, const pmx_sim3*, double*);
int pmx_impl_graph_solve(pmx_context*, pmx_prepared_graph*, const pmx_sim3*, const double*, double*, double*, int32_t*);
int pmx_impl_graph_release(pmx_context*, pmx_prepared_graph*);
int pmx_impl_feature_refine(pmx_context*, pmx_memory, const pmx_matchset*, const pmx_featuremap*,
                            const pmx_featuremap*, const pmx_refine_params*, pmx_matchset*);
int pmx_impl_normalize_rays(pmx_context*, pmx_memory, const pmx_pointmap*, double*, double*, uint8_t*);
int pmx_impl_interpolate_ray(pmx_context*, pmx_memory, const pmx_pointmap*, int64_t, const double*, double*, double*,
                             uint8_t*);
int pmx_impl_median_scene_distance(pmx_context*, pmx_memory, const pmx_pointmap*, double*);
int pmx_impl_nccl_unique_id(pmx_context*, uint8_t*);
int pmx_impl_nccl_init(pmx_context*, const uint8_t*, int32_t, int32_t);
int pmx_impl_graph_optimize_sharded(pmx_context*, pmx_prepared_graph*, pmx_sim3*, pmx_optimize_result*, pmx_sim3*,
                                    double*);
int pmx_impl_iterative_project(pmx_context*, pmx_memory, const pmx_pointmap*, int64_t, const float*,
                               const double*, const pmx_iter_proj_params*, double*, uint8_t*, int32_t*);
int pmx_impl_match_stats(pmx_context*, pmx_memory, const pmx_matchset*, int32_t, int64_t*, double*);
int pmx_impl_residual_blocks(pmx_context*, pmx_memory, const pmx_sim3*, const pmx_matchset*,
                             const pmx_pointmap*, const pmx_pointmap*, pmx_track_mode,
                             const pmx_robust_weight_params*, const pmx_intrinsics*, double*, double*,
                             double*, double*, uint8_t*);
int pmx_impl_normal_equations(pmx_context*, pmx_memory, const pmx_sim3*, const pmx_matchset*,
                              const pmx_pointmap*, const pmx_pointmap*, pmx_track_mode,
                              const pmx_robust_weight_params*, const pmx_intrinsics*, double*, double*,
                              double*, int64_t*);
int pmx_impl_track_given_matches(pmx_context*, pmx_memory, const pmx_pointmap*, const pmx_pointmap*,
                                 const pmx_matchset*, const pmx_sim3*, pmx_track_mode,
                                 const pmx_solve_pose_params*, pmx_track_result*);
int pmx_impl_fuse_canonical(pmx_context*, pmx_memory, int32_t, int32_t, float*, uint8_t*, float*,
                            const pmx_pointmap*, const float*, const pmx_sim3*);
int pmx_impl_assemble_system(pmx_context*, pmx_memory, const pmx_graph*, const pmx_backend_params*, double*,
                             double*);
int pmx_impl_backend_cost(pmx_context*, pmx_memory, const pmx_graph*, const pmx_backend_params*, double*);
int pmx_impl_global_optimize(pmx_context*, pmx_memory, pmx_graph*, const pmx_backend_params*,
                             pmx_optimize_result*, pmx_sim3*);
int pmx_impl_backend_edge_terms(pmx_context*, pmx_memory, const pmx_graph*, const pmx_backend_params*,
                                int32_t, int32_t, double*);
int pmx_impl_backend_solve_terms(pmx_context*, pmx_memory, const pmx_graph*, const pmx_backend_params*,
                                 const double*, double*, double*, int32_t*);
int pmx_impl_ldlt_solve(pmx_context*, pmx_memory, int32_t, const double*, const double*, double*, int32_t*);
}

namespace {

template <class F>
int guarded(pmx_context* c, F&& f) {
  if (!c) return PMX_ERR_INVALID_ARGUMENT;
  Context& ctx = *reinterpret_cast<Context*>(c);
  try {
    PMX_CUDA(cudaSetDevice(ctx.device));
    const int r = f();
    return r;
  } catch (const pmx::Error& e) {
    ctx.err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx.err = e.what();
    return PMX_ERR_INVALID_ARGUMENT;
  }
}

}  // namespace

extern "C" {

void pmx_default_match_params(pmx_match_params* p) {  // camera.hpp:102-108, 126-131
  p->projection.lambda_init = 1e-4;
  p->projection.lambda_up = 10.0;
  p->projection.lambda_down = 0.3;
  p->projection.angle_tol = 1e-5;
  p->projection.max_iterations = 10;
  p->invalidation_median_fraction = 0.1;
}

void pmx_default_refine_params(pmx_refine_params* p) {  // camera.hpp:140-143
  std::memset(p, 0, sizeof(*p));
  p->num_levels = 2;
  p->stride[0] = 2;
  p->radius[0] = 2;
  p->stride[1] = 1;
  p->radius[1] = 2;
}

void pmx_default_robust_weight_params(pmx_robust_weight_params* p) {  // tracking.hpp:26-34
  p->sigma2_point = 1e-2;
  p->sigma2_ray = 1e-3;
  p->sigma2_pixel = 4.0;
  p->q_min = 0.0;
  p->q_min_fraction = 0.1;
  p->huber_delta = 1.345;
  p->distance_weight = 0.01;
}

void pmx_default_solve_pose_params(pmx_solve_pose_params* p) {  // tracking.hpp:82-91
  std::memset(p, 0, sizeof(*p));
  pmx_default_robust_weight_params(&p->weights);
  pmx_default_match_params(&p->matching);
  pmx_default_refine_params(&p->refinement);
  p->refine_features = 1;
  p->max_iterations = 20;
  p->update_tol = 1e-6;
  p->min_valid_matches = 12;
  p->has_intrinsics = 0;
}

void pmx_default_backend_params(pmx_backend_params* p) {  // backend.hpp:38-46
  std::memset(p, 0, sizeof(*p));
  pmx_default_robust_weight_params(&p->weights);
  p->mode = PMX_TRACK_RAY;
  p->has_intrinsics = 0;
  p->max_iterations = 10;
  p->update_tol = 1e-6;
  p->damping_init = 1e-6;
  p->damping_retries = 3;
}

void pmx_sim3_identity(pmx_sim3* T) {
  std::memset(T, 0, sizeof(*T));
  T->R[0] = T->R[4] = T->R[8] = 1.0;
  T->s = 1.0;
}

void pmx_sim3_retract(const pmx_sim3* T, const double* tau7, pmx_sim3* out) {
  *out = pmx::to_pmx(pmx::sim3_mul(pmx::sim3_exp(tau7), pmx::to_dsim3(*T)));
}

void pmx_sim3_relative(const pmx_sim3* T_wi, const pmx_sim3* T_wj, pmx_sim3* out) {
  *out = pmx::to_pmx(pmx::sim3_mul(pmx::sim3_inv(pmx::to_dsim3(*T_wi)), pmx::to_dsim3(*T_wj)));
}

int pmx_abi_version(void) { return PMX_ABI_VERSION; }

int pmx_create(int device, pmx_context** out) {
  if (!out) return PMX_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
    cudaGetLastError();
    return PMX_ERR_NO_DEVICE;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return PMX_ERR_NO_DEVICE;
  auto* ctx = new Context();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return PMX_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  // keep freed scratch in the stream-ordered pool between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = reinterpret_cast<pmx_context*>(ctx);
  return (int)PMX_OK;
}

int pmx_destroy(pmx_context* c) {
  if (!c) return (int)PMX_OK;
  Context* ctx = reinterpret_cast<Context*>(c);
  cudaSetDevice(ctx->device);
  if (ctx->stream && ctx->stream != ctx->own_stream) cudaStreamSynchronize(ctx->stream);  // adopted stream
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->own_stream);
    cudaStreamDestroy(ctx->own_stream);
  }
  for (cudaStream_t s : {ctx->copy_in, ctx->copy_in2, ctx->copy_out, ctx->aux})
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  for (auto& kv : ctx->dev_counters) cudaFree(kv.second);
  if (ctx->nccl_comm) {
    try {
      if (pmx::nccl_api().CommDestroy) pmx::nccl_api().CommDestroy((ncclComm_t)ctx->nccl_comm);
    } catch (...) {
    }
  }
  delete ctx;
  return (int)PMX_OK;
}

const char* pmx_last_error(const pmx_context* c) {
  if (!c) return "null context";
  return reinterpret_cast<const Context*>(c)->err.c_str();
}

int pmx_set_stream(pmx_context* c, void* s) {
  return guarded(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    ctx.stream = s ? static_cast<cudaStream_t>(s) : ctx.own_stream;
    return (int)PMX_OK;
  });
}

void* pmx_get_stream(pmx_context* c) { return c ? reinterpret_cast<Context*>(c)->stream : nullptr; }

int pmx_synchronize(pmx_context* c) {
  return guarded(c, [&] {
    PMX_CUDA(cudaStreamSynchronize(reinterpret_cast<Context*>(c)->stream));
    return (int)PMX_OK;
  });
}

int64_t pmx_kernel_launch_count(const pmx_context* c) {
  return c ? reinterpret_cast<const Context*>(c)->launches : 0;
}

static void prof_clear(Context& ctx) {
  for (auto& e : ctx.prof) {
    cudaEventDestroy(e.start);
    cudaEventDestroy(e.stop);
  }
  ctx.prof.clear();
}

int pmx_profile_enable(pmx_context* c, int on) {
  return guarded(c, [&] {
    reinterpret_cast<Context*>(c)->profiling = on != 0;
    return (int)PMX_OK;
  });
}

int pmx_set_device_graphs(pmx_context* c, int on) {
  return guarded(c, [&] {
    reinterpret_cast<Context*>(c)->graphs = on != 0;
    return (int)PMX_OK;
  });
}

int pmx_profile_reset(pmx_context* c) {
  return guarded(c, [&] {
    Context& ctx = *reinterpret_cast<Context*>(c);
    PMX_CUDA(cudaStreamSynchronize(ctx.stream));
    prof_clear(ctx);
    ctx.counters.clear();
    for (auto& kv : ctx.dev_counters) PMX_CUDA(cudaMemset(kv.second, 0, sizeof(unsigned long long)));
    return (int)PMX_OK;
  });
}

unsigned long long pmx_checked_violations_match();
unsigned long long pmx_checked_violations_backend();

int pmx_profile_get(pmx_context* c, const char* kernel, double* total_ms, int64_t* launches) {
  return guarded(c, [&] {
    pmx::require(kernel && total_ms && launches, "profile_get: null arguments");
    Context& ctx = *reinterpret_cast<Context*>(c);
    double t = 0.0;
    int64_t n = 0;
    for (auto& e : ctx.prof) {
      if (std::strcmp(e.name, kernel) != 0) continue;
      PMX_CUDA(cudaEventSynchronize(e.stop));
      float ms = 0.0f;
      PMX_CUDA(cudaEventElapsedTime(&ms, e.start, e.stop));
      t += ms;
      ++n;
    }
    auto it = ctx.counters.find(kernel);
    if (it != ctx.counters.end()) n = it->second;  // counters report through `launches`
    if (std::strcmp(kernel, "checked_violations") == 0) {  // range violations of a -DPMX_CHECKED build
      PMX_CUDA(cudaDeviceSynchronize());
      n = (int64_t)(pmx_checked_violations_match() + pmx_checked_violations_backend());
    }
    auto dc = ctx.dev_counters.find(kernel);
    if (dc != ctx.dev_counters.end()) {
      unsigned long long v = 0;
      PMX_CUDA(cudaStreamSynchronize(ctx.stream));
      PMX_CUDA(cudaMemcpy(&v, dc->second, sizeof(v), cudaMemcpyDeviceToHost));
      n += (int64_t)v;
    }
    *total_ms = t;
    *launches = n;
    return (int)PMX_OK;
  });
}

int pmx_normalize_rays(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, double* rays, double* dist,
                       uint8_t* valid) {
  return guarded(c, [&] { return pmx_impl_normalize_rays(c, mem, pm, rays, dist, valid); });
}

int pmx_interpolate_ray(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, int64_t n, const double* p,
                        double* ray, double* jacobian, uint8_t* ok) {
  return guarded(c, [&] { return pmx_impl_interpolate_ray(c, mem, pm, n, p, ray, jacobian, ok); });
}

int pmx_nccl_unique_id(pmx_context* c, uint8_t id[128]) {
  return guarded(c, [&] { return pmx_impl_nccl_unique_id(c, id); });
}

int pmx_nccl_init(pmx_context* c, const uint8_t id[128], int32_t rank, int32_t nranks) {
  return guarded(c, [&] { return pmx_impl_nccl_init(c, id, rank, nranks); });
}

int pmx_graph_optimize_sharded(pmx_context* c, pmx_prepared_graph* pg, pmx_sim3* poses, pmx_optimize_result* result,
                               pmx_sim3* pose_trace, double* timings) {
  return guarded(c, [&] { return pmx_impl_graph_optimize_sharded(c, pg, poses, result, pose_trace, timings); });
}

int pmx_median_scene_distance(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, double* out) {
  return guarded(c, [&] { return pmx_impl_median_scene_distance(c, mem, pm, out); });
}

int pmx_iterative_project(pmx_context* c, pmx_memory mem, const pmx_pointmap* pm, int64_t n, const float* x,
                          const double* p0, const pmx_iter_proj_params* params, double* pixel,
                          uint8_t* converged, int32_t* iterations) {
  return guarded(c, [&] {
    return pmx_impl_iterative_project(c, mem, pm, n, x, p0, params, pixel, converged, iterations);
  });
}

int pmx_match_pointmaps(pmx_context* c, pmx_memory mem, const pmx_pointmap* X_a, const pmx_pointmap* X_b_in_a,
                        const pmx_featuremap* F_a, const pmx_featuremap* F_b, const pmx_matchset* init,
                        const pmx_match_params* params, pmx_matchset* out) {
  return guarded(c, [&] {
    pmx::require(X_a && X_b_in_a && F_a && F_b && out, "match_pointmaps: null arguments");
    pmx_pair p{*X_a, *X_b_in_a, *F_a, *F_b, init};
    return pmx_impl_match_batch(c, mem, 1, &p, params, nullptr, out);
  });
}

int pmx_feature_refine(pmx_context* c, pmx_memory mem, const pmx_matchset* in, const pmx_featuremap* F_a,
                       const pmx_featuremap* F_b, const pmx_refine_params* params, pmx_matchset* out) {
  return guarded(c, [&] { return pmx_impl_feature_refine(c, mem, in, F_a, F_b, params, out); });
}

int pmx_match_batch(pmx_context* c, pmx_memory mem, int32_t num_pairs, const pmx_pair* pairs,
                    const pmx_match_params* params, const pmx_refine_params* refine, pmx_matchset* outs) {
  return guarded(c, [&] { return pmx_impl_match_batch(c, mem, num_pairs, pairs, params, refine, outs); });
}

int pmx_accept_loop_edges(pmx_context* c, pmx_memory mem, int32_t num_pairs, const pmx_pair* pairs, double omega_l,
                          const pmx_match_params* params, const pmx_refine_params* refine, pmx_matchset* outs,
                          int32_t* accepted) {
  return guarded(c, [&] {
    return pmx_impl_accept_loop_edges(c, mem, num_pairs, pairs, omega_l, params, refine, outs, accepted);
  });
}

int pmx_ingest_pair_record(pmx_context* c, pmx_memory mem, const void* record, int64_t nbytes, int32_t height,
                           int32_t width, int32_t dim, pmx_pair_record* out, int64_t* inexact_descriptors) {
  return guarded(c, [&] {
    return pmx_impl_ingest_pair_record(c, mem, record, nbytes, height, width, dim, out, inexact_descriptors);
  });
}

int pmx_constrain_to_rays(pmx_context* c, pmx_memory mem, int32_t height, int32_t width, float* xyz,
                          uint8_t* valid, const pmx_intrinsics* K) {
  return guarded(c, [&] { return pmx_impl_constrain_to_rays(c, mem, height, width, xyz, valid, K); });
}

int pmx_graph_prepare(pmx_context* c, pmx_memory mem, const pmx_graph* g, const pmx_backend_params* p, int32_t e0,
                      int32_t e1, pmx_prepared_graph** out) {
  return guarded(c, [&] { return pmx_impl_graph_prepare(c, mem, g, p, e0, e1, out); });
}
int pmx_graph_edge_terms(pmx_context* c, pmx_prepared_graph* pg, const pmx_sim3* poses, double* out) {
  return guarded(c, [&] { return pmx_impl_graph_edge_terms(c, pg, poses, out); });
}
int pmx_graph_solve(pmx_context* c, pmx_prepared_graph* pg, const pmx_sim3* poses, const double* terms, double* tau,
                    double* cost, int32_t* solved) {
  return guarded(c, [&] { return pmx_impl_graph_solve(c, pg, poses, terms, tau, cost, solved); });
}
int pmx_graph_release(pmx_context* c, pmx_prepared_graph* pg) {
  return guarded(c, [&] { return pmx_impl_graph_release(c, pg); });
}

int pmx_match_stats(pmx_context* c, pmx_memory mem, const pmx_matchset* m, int32_t num_pixels_a,
                    int64_t* valid_count, double* unique_fraction) {
  return guarded(c, [&] { return pmx_impl_match_stats(c, mem, m, num_pixels_a, valid_count, unique_fraction); });
}

int pmx_keyframe_decision(pmx_context* c, pmx_memory mem, const pmx_matchset* m, int32_t height, int32_t width,
                          double omega_k, int32_t* new_keyframe) {  // tracking.cpp:249-257
  return guarded(c, [&] {
    pmx::require(m && new_keyframe, "keyframe_decision: null arguments");
    const int total = height * width;
    if (total <= 0) {
      *new_keyframe = 1;
      return (int)PMX_OK;
    }
    int64_t vc = 0;
    double uf = 0.0;
    const int r = pmx_impl_match_stats(c, mem, m, total, &vc, &uf);
    if (r != PMX_OK) return r;
    const double vf = (double)vc / total;
    *new_keyframe = (vf < omega_k || uf < omega_k) ? 1 : 0;
    return (int)PMX_OK;
  });
}

int pmx_residual_blocks(pmx_context* c, pmx_memory mem, const pmx_sim3* T, const pmx_matchset* m,
                        const pmx_pointmap* X_ref, const pmx_pointmap* X_src, pmx_track_mode mode,
                        const pmx_robust_weight_params* params, const pmx_intrinsics* K, double* residual,
                        double* jacobian, double* weight, double* info, uint8_t* used) {
  return guarded(c, [&] {
    return pmx_impl_residual_blocks(c, mem, T, m, X_ref, X_src, mode, params, K, residual, jacobian, weight,
                                    info, used);
  });
}

int pmx_normal_equations(pmx_context* c, pmx_memory mem, const pmx_sim3* T, const pmx_matchset* m,
                         const pmx_pointmap* X_ref, const pmx_pointmap* X_src, pmx_track_mode mode,
                         const pmx_robust_weight_params* params, const pmx_intrinsics* K, double* H, double* g,
                         double* cost, int64_t* used) {
  return guarded(c, [&] {
    return pmx_impl_normal_equations(c, mem, T, m, X_ref, X_src, mode, params, K, H, g, cost, used);
  });
}

int pmx_track_given_matches(pmx_context* c, pmx_memory mem, const pmx_pointmap* canonical,
                            const pmx_pointmap* X_f_f, const pmx_matchset* matches, const pmx_sim3* init,
                            pmx_track_mode mode, const pmx_solve_pose_params* params, pmx_track_result* result) {
  return guarded(c, [&] {
    return pmx_impl_track_given_matches(c, mem, canonical, X_f_f, matches, init, mode, params, result);
  });
}

int pmx_solve_pose(pmx_context* c, pmx_memory mem, const pmx_pointmap* canonical, const pmx_pointmap* X_f_f,
                   const pmx_pointmap* X_k_f, const pmx_featuremap* F_f, const pmx_featuremap* F_k,
                   const pmx_sim3* init, pmx_track_mode mode, const pmx_solve_pose_params* params,
                   const pmx_matchset* match_seed, pmx_track_result* result, pmx_matchset* matches_out) {
  // tracking.cpp:149-226: match + refine (frame = a, keyframe image = b), then GN
  return guarded(c, [&] {
    pmx::require(canonical && X_f_f && X_k_f && F_f && F_k && init && result, "solve_pose: null arguments");
    pmx_solve_pose_params sp;
    pmx_default_solve_pose_params(&sp);
    if (params) sp = *params;
    Context& ctx = *reinterpret_cast<Context*>(c);
    const int64_t hw = (int64_t)X_k_f->height * X_k_f->width;
    // matches live on the device between the two stages
    pmx::DevBuf pa(sizeof(int32_t) * hw, ctx.stream), q(sizeof(float) * hw, ctx.stream),
        v(sizeof(uint8_t) * hw, ctx.stream);
    pmx::Stager st(ctx, mem);
    pmx_pair pair{*X_f_f, *X_k_f, *F_f, *F_k, match_seed};
    // stage inputs once; device pointers from here on
    pmx_pointmap dXf = *X_f_f, dXk = *X_k_f, dC = *canonical;
    pmx_featuremap dFf = *F_f, dFk = *F_k;
    const size_t hwf = (size_t)X_f_f->height * X_f_f->width;
    dXf.xyz = st.in(X_f_f->xyz, 3 * hwf);
    dXf.valid = st.in(X_f_f->valid, hwf);
    dXk.xyz = st.in(X_k_f->xyz, 3 * (size_t)hw);
    dXk.valid = st.in(X_k_f->valid, (size_t)hw);
    const size_t hwc = (size_t)canonical->height * canonical->width;
    dC.xyz = st.in(canonical->xyz, 3 * hwc);
    dC.valid = st.in(canonical->valid, hwc);
    dFf.descriptors = st.in(F_f->descriptors, hwf * F_f->dim);
    dFf.match_confidence = st.in(F_f->match_confidence, hwf);
    dFk.descriptors = st.in(F_k->descriptors, (size_t)hw * F_k->dim);
    dFk.match_confidence = st.in(F_k->match_confidence, (size_t)hw);
    pmx_matchset dseed{};
    if (match_seed) {
      dseed.count = match_seed->count;
      dseed.pixel_a = const_cast<int32_t*>(st.in(match_seed->pixel_a, (size_t)match_seed->count));
      dseed.pixel_b = const_cast<int32_t*>(st.in(match_seed->pixel_b, (size_t)match_seed->count));
      dseed.confidence = const_cast<float*>(st.in(match_seed->confidence, (size_t)match_seed->count));
      dseed.valid = const_cast<uint8_t*>(st.in(match_seed->valid, (size_t)match_seed->count));
    }
    pair = pmx_pair{dXf, dXk, dFf, dFk, match_seed ? &dseed : nullptr};
    pmx_matchset dm{hw, pa.as<int32_t>(), nullptr, q.as<float>(), v.as<uint8_t>()};
    int r = pmx_impl_match_batch(c, PMX_MEM_DEVICE, 1, &pair, &sp.matching,
                                 sp.refine_features ? &sp.refinement : nullptr, &dm);
    if (r != PMX_OK) return r;
    r = pmx_impl_track_given_matches(c, PMX_MEM_DEVICE, &dC, &dXf, &dm, init, mode, &sp, result);
    if (r != PMX_OK) return r;
    if (matches_out) {
      pmx::require(matches_out->count >= hw, "solve_pose: matches_out too small");
      const cudaMemcpyKind k = mem == PMX_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
      PMX_CUDA(cudaMemcpyAsync(matches_out->pixel_a, pa.p, pa.bytes, k, ctx.stream));
      PMX_CUDA(cudaMemcpyAsync(matches_out->confidence, q.p, q.bytes, k, ctx.stream));
      PMX_CUDA(cudaMemcpyAsync(matches_out->valid, v.p, v.bytes, k, ctx.stream));
      if (matches_out->pixel_b) {
        std::vector<int32_t> idx(hw);
        for (int64_t i = 0; i < hw; ++i) idx[i] = (int32_t)i;
        PMX_CUDA(cudaMemcpyAsync(matches_out->pixel_b, idx.data(), sizeof(int32_t) * hw,
                                 mem == PMX_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice,
                                 ctx.stream));
        PMX_CUDA(cudaStreamSynchronize(ctx.stream));
      }
      matches_out->count = hw;
    }
    PMX_CUDA(cudaStreamSynchronize(ctx.stream));
    return (int)PMX_OK;
  });
}

int pmx_fuse_canonical(pmx_context* c, pmx_memory mem, int32_t height, int32_t width, float* canonical_xyz,
                       uint8_t* canonical_valid, float* canonical_confidence, const pmx_pointmap* X_k_f,
                       const float* confidence, const pmx_sim3* T_kf) {
  return guarded(c, [&] {
    return pmx_impl_fuse_canonical(c, mem, height, width, canonical_xyz, canonical_valid, canonical_confidence,
                                   X_k_f, confidence, T_kf);
  });
}

int pmx_assemble_system(pmx_context* c, pmx_memory mem, const pmx_graph* g, const pmx_backend_params* p,
                        double* H, double* grad) {
  return guarded(c, [&] { return pmx_impl_assemble_system(c, mem, g, p, H, grad); });
}

int pmx_backend_cost(pmx_context* c, pmx_memory mem, const pmx_graph* g, const pmx_backend_params* p,
                     double* cost) {
  return guarded(c, [&] { return pmx_impl_backend_cost(c, mem, g, p, cost); });
}

int pmx_global_optimize(pmx_context* c, pmx_memory mem, pmx_graph* g, const pmx_backend_params* p,
                        pmx_optimize_result* result, pmx_sim3* pose_trace) {
  return guarded(c, [&] { return pmx_impl_global_optimize(c, mem, g, p, result, pose_trace); });
}

int pmx_backend_edge_terms(pmx_context* c, pmx_memory mem, const pmx_graph* g, const pmx_backend_params* p,
                           int32_t edge_begin, int32_t edge_end, double* out) {
  return guarded(c, [&] { return pmx_impl_backend_edge_terms(c, mem, g, p, edge_begin, edge_end, out); });
}

int pmx_backend_solve_terms(pmx_context* c, pmx_memory mem, const pmx_graph* g, const pmx_backend_params* p,
                            const double* terms, double* tau, double* cost, int32_t* solved) {
  return guarded(c, [&] { return pmx_impl_backend_solve_terms(c, mem, g, p, terms, tau, cost, solved); });
}

int pmx_ldlt_solve(pmx_context* c, pmx_memory mem, int32_t n, const double* A, const double* b, double* x,
                   int32_t* ok) {
  return guarded(c, [&] { return pmx_impl_ldlt_solve(c, mem, n, A, b, x, ok); });
}

}  // extern "C"
