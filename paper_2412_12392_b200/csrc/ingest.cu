// Input-side neighbours of the hot path:
//
//   PMPAIR01 pair records (reference src/pipeline.cpp:510-676, the stream
//   format of RecordingPredictor / StreamPredictor) unpacked on the device
//   into the layouts the matcher consumes: interleaved fp32 points + the
//   allFinite validity of read_pointmap_f32 (pipeline.cpp:536-543), fp32
//   confidences, fp16 descriptors (pixel-major, the Eigen column-per-pixel
//   order of the record), fp32 match confidences.  The record's descriptors
//   are fp32; the fp16 conversion is exact for predictor outputs quantised to
//   fp16 and every inexact conversion is counted (parity with the FP64
//   reference holds iff the count is 0).
//
//   constrain_to_rays (pipeline.cpp:32-46), calibrated mode: canonical points
//   are put back on their pixel rays, only the depth stays free.
#include <cuda_fp16.h>

#include <cstring>

#include "pmx_common.cuh"

namespace pmx {

struct RecordLayout {  // element offsets (floats) after the 8-byte magic
  int64_t X_i, X_j, C_i, C_j, D_i, D_j, Q_i, Q_j, total;
};

static RecordLayout record_layout(int64_t hw, int64_t dim) {
  RecordLayout L;
  L.X_i = 0;
  L.X_j = L.X_i + 3 * hw;
  L.C_i = L.X_j + 3 * hw;
  L.C_j = L.C_i + hw;
  L.D_i = L.C_j + hw;
  L.D_j = L.D_i + dim * hw;
  L.Q_i = L.D_j + dim * hw;
  L.Q_j = L.Q_i + hw;
  L.total = L.Q_j + hw;
  return L;
}

struct IngestOut {
  float *X_i, *X_j, *C_i, *C_j, *Q_i, *Q_j;
  uint8_t *valid_i, *valid_j;
  __half *D_i, *D_j;
};

// One thread per pixel: points + validity, confidences, descriptors.
__global__ void __launch_bounds__(256) k_ingest_pair(const float* __restrict__ rec, RecordLayout L, int64_t hw,
                                                     int dim, IngestOut o, unsigned long long* __restrict__ inexact) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
    for (int side = 0; side < 2; ++side) {
      const float* X = rec + (side ? L.X_j : L.X_i) + 3 * i;
      const float x = X[0], y = X[1], z = X[2];
      float* Xo = (side ? o.X_j : o.X_i) + 3 * i;
      Xo[0] = x;
      Xo[1] = y;
      Xo[2] = z;
      (side ? o.valid_j : o.valid_i)[i] = (isfinite(x) && isfinite(y) && isfinite(z)) ? 1 : 0;  // allFinite
      const float* D = rec + (side ? L.D_j : L.D_i) + (int64_t)dim * i;
      __half* Do = (side ? o.D_j : o.D_i) + (int64_t)dim * i;
      for (int k = 0; k < dim; ++k) {
        const float v = D[k];
        const __half h = __float2half_rn(v);
        bad += (__half2float(h) != v && !(v != v)) ? 1 : 0;  // NaN stays NaN
        Do[k] = h;
      }
    }
    o.C_i[i] = rec[L.C_i + i];
    o.C_j[i] = rec[L.C_j + i];
    o.Q_i[i] = rec[L.Q_i + i];
    o.Q_j[i] = rec[L.Q_j + i];
  }
  for (int s = 16; s > 0; s >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, s);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(inexact, (unsigned long long)bad);
}

// constrain_to_rays, pipeline.cpp:32-46 (z <= 0 invalidates; invalid stays).
__global__ void k_constrain_to_rays(int H, int W, float* __restrict__ xyz, uint8_t* __restrict__ valid, double fx,
                                    double fy, double cx, double cy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= H * W || !valid[i]) return;
  const int u = i % W, v = i / W;
  const double z = xyz[3 * i + 2];
  if (z <= 0.0) {
    valid[i] = 0;
    return;
  }
  xyz[3 * i] = (float)(z * ((u - cx) / fx));
  xyz[3 * i + 1] = (float)(z * ((v - cy) / fy));
  xyz[3 * i + 2] = (float)z;
}

}  // namespace pmx

using namespace pmx;

extern "C" int pmx_impl_ingest_pair_record(pmx_context* c, pmx_memory mem, const void* record, int64_t nbytes,
                                           int32_t height, int32_t width, int32_t dim, pmx_pair_record* out,
                                           int64_t* inexact_descriptors) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(record && out && height > 0 && width > 0 && dim > 0, "ingest_pair_record: bad arguments");
  const int64_t hw = (int64_t)height * width;
  const RecordLayout L = record_layout(hw, dim);
  require(nbytes >= 8 + 4 * L.total, "StreamPredictor: truncated record");  // pipeline.cpp:667
  static const char kPairMagic[8] = {'P', 'M', 'P', 'A', 'I', 'R', '0', '1'};
  char magic[8];
  if (mem == PMX_MEM_HOST)
    std::memcpy(magic, record, 8);
  else
    PMX_CUDA(cudaMemcpy(magic, record, 8, cudaMemcpyDeviceToHost));
  require(std::memcmp(magic, kPairMagic, 8) == 0, "StreamPredictor: bad magic");  // pipeline.cpp:652-654
  Stager st(ctx, mem);
  const float* rec = st.in(reinterpret_cast<const float*>(static_cast<const char*>(record) + 8), (size_t)L.total);
  IngestOut o;
  o.X_i = st.out(out->X_i, 3 * hw);
  o.X_j = st.out(out->X_j, 3 * hw);
  o.valid_i = st.out(out->valid_i, hw);
  o.valid_j = st.out(out->valid_j, hw);
  o.C_i = st.out(out->C_i, hw);
  o.C_j = st.out(out->C_j, hw);
  o.Q_i = st.out(out->Q_i, hw);
  o.Q_j = st.out(out->Q_j, hw);
  o.D_i = reinterpret_cast<__half*>(st.out(out->D_i, dim * hw));
  o.D_j = reinterpret_cast<__half*>(st.out(out->D_j, dim * hw));
  require(o.X_i && o.X_j && o.valid_i && o.valid_j && o.C_i && o.C_j && o.Q_i && o.Q_j && o.D_i && o.D_j,
          "ingest_pair_record: null output array");
  DevBuf cnt(sizeof(unsigned long long), ctx.stream);
  PMX_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes, ctx.stream));
  const int grid = (int)std::min<int64_t>((hw + 255) / 256, 8LL * ctx.num_sms);
  k_ingest_pair<<<grid, 256, 0, ctx.stream>>>(rec, L, hw, dim, o, cnt.as<unsigned long long>());
  launch_check(ctx, "k_ingest_pair");
  st.back(out->X_i, o.X_i, 3 * hw);
  st.back(out->X_j, o.X_j, 3 * hw);
  st.back(out->valid_i, o.valid_i, hw);
  st.back(out->valid_j, o.valid_j, hw);
  st.back(out->C_i, o.C_i, hw);
  st.back(out->C_j, o.C_j, hw);
  st.back(out->Q_i, o.Q_i, hw);
  st.back(out->Q_j, o.Q_j, hw);
  st.back(out->D_i, reinterpret_cast<uint16_t*>(o.D_i), dim * hw);
  st.back(out->D_j, reinterpret_cast<uint16_t*>(o.D_j), dim * hw);
  unsigned long long bad = 0;
  PMX_CUDA(cudaMemcpyAsync(&bad, cnt.p, sizeof(bad), cudaMemcpyDeviceToHost, ctx.stream));
  PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  if (inexact_descriptors) *inexact_descriptors = (int64_t)bad;
  return PMX_OK;
}

extern "C" int pmx_impl_constrain_to_rays(pmx_context* c, pmx_memory mem, int32_t height, int32_t width,
                                          float* xyz, uint8_t* valid, const pmx_intrinsics* K) {
  Context& ctx = *reinterpret_cast<Context*>(c);
  require(xyz && valid && K && height >= 0 && width >= 0, "constrain_to_rays: null arguments");
  const int64_t hw = (int64_t)height * width;
  Stager st(ctx, mem);
  float* dx = st.inout(xyz, 3 * hw);
  uint8_t* dv = st.inout(valid, hw);
  if (hw > 0) {
    k_constrain_to_rays<<<(unsigned)((hw + 255) / 256), 256, 0, ctx.stream>>>(height, width, dx, dv, K->fx, K->fy,
                                                                              K->cx, K->cy);
    launch_check(ctx, "k_constrain_to_rays");
  }
  st.back(xyz, dx, 3 * hw);
  st.back(valid, dv, hw);
  if (mem == PMX_MEM_HOST) PMX_CUDA(cudaStreamSynchronize(ctx.stream));
  return PMX_OK;
}
