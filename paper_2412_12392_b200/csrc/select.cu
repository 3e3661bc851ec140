// Segmented exact upper median (see select.cuh).
#include <algorithm>

#include "select.cuh"

namespace pmx {

namespace {
constexpr int N1 = 4096, N2 = 4096, N3 = 256, NT = N1 + N2 + N3 + 8;

__device__ __forceinline__ uint32_t fkey(float f) {  // order-preserving float -> uint32
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

template <int PASS>
__global__ void __launch_bounds__(256) k_hist(const SelSeg* __restrict__ segs, uint32_t* __restrict__ scratch,
                                              int64_t per_block, int seg0) {
  const int seg = seg0 + (int)blockIdx.y;
  const SelSeg S = segs[seg];
  uint32_t* base = scratch + (size_t)NT * seg;
  uint32_t* state = base + N1 + N2 + N3;  // [0]=n [1]=krem [2]=prefix
  constexpr int NB = PASS == 3 ? N3 : 4096;
  uint32_t* h = base + (PASS == 1 ? 0 : PASS == 2 ? N1 : N1 + N2);
  __shared__ uint32_t sh[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t prefix = 0;
  if (PASS > 1) {
    if (state[0] == 0) return;
    prefix = state[2];
  }
  const int64_t b0 = (int64_t)blockIdx.x * per_block;
  const int64_t b1 = min(S.n, b0 + per_block);
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const bool ok = !(S.valid && !S.valid[i]);
    const float v = S.vals[i];
    // NaN never orders; std::nth_element is UB on it, we drop it
    const uint32_t k = fkey(v);
    const bool take = ok && v == v &&
                      (PASS == 1 || (PASS == 2 ? (k >> 20) == prefix : (k >> 8) == prefix));
    if (PASS == 1)  // the top bits of neighbouring values collide: warp-aggregated
      hist_add(sh, k >> 20, take);
    else if (take)  // the low bits inside one bucket spread: plain shared atomics
      atomicAdd(&sh[PASS == 2 ? (k >> 8) & 0xfff : k & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += blockDim.x)
    if (sh[i]) atomicAdd(&h[i], sh[i]);
}

template <int PASS>
__global__ void __launch_bounds__(1024) k_scan(const SelSeg* __restrict__ segs, uint32_t* __restrict__ scratch) {
  const SelSeg S = segs[blockIdx.x];
  uint32_t* base = scratch + (size_t)NT * blockIdx.x;  // gridDim.x = nseg (no 65535 limit on x)
  uint32_t* state = base + N1 + N2 + N3;
  constexpr int NB = PASS == 3 ? N3 : 4096;
  const uint32_t* h = base + (PASS == 1 ? 0 : PASS == 2 ? N1 : N1 + N2);
  constexpr int PER = (NB + 1023) / 1024;
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t total, krem_s, prefix_s;
  const int t = threadIdx.x;
  uint32_t local[PER], s = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int b = t * PER + j;
    local[j] = b < NB ? h[b] : 0u;
    s += local[j];
  }
  uint32_t incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += y;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    const uint32_t w = wsum[t];
    uint32_t wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (t >= o) wi += y;
    }
    wsum[t] = wi - w;
    if (t == 31) total = wi;
  }
  __syncthreads();
  if (PASS == 1 && t == 0) {
    state[0] = total;
    state[1] = total / 2;
    if (total == 0) *S.out = S.scale * 0.0;
  }
  if (t == 0) {  // one read of the state before the matching thread rewrites it
    krem_s = state[1];
    prefix_s = state[2];
  }
  __syncthreads();
  if (total == 0) return;
  const uint32_t krem = krem_s;
  uint32_t excl = wsum[t >> 5] + incl - s;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int b = t * PER + j;
    if (b < NB && local[j] > 0 && excl <= krem && krem < excl + local[j]) {
      if (PASS == 1) state[2] = (uint32_t)b;
      if (PASS == 2) state[2] = (prefix_s << 12) | (uint32_t)b;
      if (PASS == 3) *S.out = S.scale * (double)unkey((prefix_s << 8) | (uint32_t)b);
      state[1] = krem - excl;
    }
    excl += local[j];
  }
}
}  // namespace

void segmented_median(Context& ctx, const SelSeg* dev_segs, int nseg, int64_t max_n, DevBuf& scratch) {
  if (nseg == 0) return;
  scratch = DevBuf(sizeof(uint32_t) * (size_t)NT * nseg, ctx.stream);
  PMX_CUDA(cudaMemsetAsync(scratch.p, 0, scratch.bytes, ctx.stream));
  // elements per block: 8 blocks per SM over all segments, 1024..32768 (one
  // 196,608-element segment - tracking's q_min median - gets 192 blocks, not 24)
  const int64_t want = (max_n * nseg + (int64_t)ctx.num_sms * 8 - 1) / ((int64_t)ctx.num_sms * 8);
  const int64_t per_block = std::min<int64_t>(32768, std::max<int64_t>(1024, (want + 1023) / 1024 * 1024));
  const unsigned gx = (unsigned)std::max<int64_t>(1, (max_n + per_block - 1) / per_block);
  uint32_t* s = scratch.as<uint32_t>();
  // gridDim.y is capped at 65535: the histogram passes run over segment chunks
  auto hist = [&](auto kernel, const char* what) {
    for (int s0 = 0; s0 < nseg; s0 += 65535) {
      kernel<<<dim3(gx, std::min(65535, nseg - s0)), 256, 0, ctx.stream>>>(dev_segs, s, per_block, s0);
      launch_check(ctx, what);
    }
  };
  hist(k_hist<1>, "sel k_hist1");
  k_scan<1><<<nseg, 1024, 0, ctx.stream>>>(dev_segs, s);
  launch_check(ctx, "sel k_scan1");
  hist(k_hist<2>, "sel k_hist2");
  k_scan<2><<<nseg, 1024, 0, ctx.stream>>>(dev_segs, s);
  launch_check(ctx, "sel k_scan2");
  hist(k_hist<3>, "sel k_hist3");
  k_scan<3><<<nseg, 1024, 0, ctx.stream>>>(dev_segs, s);
  launch_check(ctx, "sel k_scan3");
}

}  // namespace pmx
