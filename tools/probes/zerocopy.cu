// Dev probe: host->device copy of pinned memory by the copy engine vs by SM
// loads through the mapped (UVA) pointer, one big buffer and many segments.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
struct Seg { const uint4* s; uint4* d; size_t n; };
__global__ void k_copy_segs(const Seg* segs, int nseg) {
  for (int g = blockIdx.y; g < nseg; g += gridDim.y) {
    const Seg sg = segs[g];
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < sg.n; i += (size_t)gridDim.x * blockDim.x)
      sg.d[i] = sg.s[i];
  }
}
int main() {
  const size_t bytes = size_t(1) << 30;
  char* h; char* d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  for (size_t i = 0; i < bytes; i += 4096) h[i] = (char)i;
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto timeit = [&](const char* name, auto fn) {
    fn(); cudaStreamSynchronize(s);
    cudaEventRecord(a, s); for (int r = 0; r < 3; ++r) fn(); cudaEventRecord(b, s);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("%-28s %8.3f ms %7.2f GB/s  (%s)\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("dma one copy", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); });
  // 512 segments of mixed sizes like the config-2 arrays (ratios 12:1:12:1:48:48:4:4)
  const int w[8] = {12, 1, 12, 1, 48, 48, 4, 4};
  std::vector<size_t> off, len;
  size_t per = bytes / 64 / 130 & ~size_t(15), o = 0;
  for (int p = 0; p < 64; ++p) for (int k = 0; k < 8; ++k) { off.push_back(o); len.push_back(per * w[k]); o += per * w[k]; }
  timeit("dma 512 copies", [&] { for (size_t i = 0; i < off.size(); ++i) cudaMemcpyAsync(d + off[i], h + off[i], len[i], cudaMemcpyHostToDevice, s); });
  for (int nq : {2, 4}) {
    std::vector<cudaStream_t> qs(nq);
    std::vector<cudaEvent_t> qe(nq);
    for (int k = 0; k < nq; ++k) { cudaStreamCreateWithFlags(&qs[k], cudaStreamNonBlocking); cudaEventCreateWithFlags(&qe[k], cudaEventDisableTiming); }
    char name[64]; snprintf(name, 64, "dma 512 copies / %d queues", nq);
    timeit(name, [&] {
      cudaEvent_t st; cudaEventCreateWithFlags(&st, cudaEventDisableTiming); cudaEventRecord(st, s);
      for (int k = 0; k < nq; ++k) cudaStreamWaitEvent(qs[k], st, 0);
      for (size_t i = 0; i < off.size(); ++i) cudaMemcpyAsync(d + off[i], h + off[i], len[i], cudaMemcpyHostToDevice, qs[i % nq]);
      for (int k = 0; k < nq; ++k) { cudaEventRecord(qe[k], qs[k]); cudaStreamWaitEvent(s, qe[k], 0); }
      cudaEventDestroy(st);
    });
  }
  for (int blocks : {148, 296, 592, 1184}) {
    char name[64]; snprintf(name, 64, "sm copy %d x 256", blocks);
    timeit(name, [&] { k_copy<<<blocks, 256, 0, s>>>((const uint4*)h, (uint4*)d, bytes / 16); });
  }
  std::vector<Seg> segs;
  for (size_t i = 0; i < off.size(); ++i) segs.push_back({(const uint4*)(h + off[i]), (uint4*)(d + off[i]), len[i] / 16});
  Seg* dsegs; cudaMalloc(&dsegs, sizeof(Seg) * segs.size());
  cudaMemcpy(dsegs, segs.data(), sizeof(Seg) * segs.size(), cudaMemcpyHostToDevice);
  {  // mixed: DMA for the large arrays (X, D), one SM kernel for the small ones (valid, Q)
    std::vector<Seg> small;
    for (size_t i = 0; i < off.size(); ++i)
      if (w[i % 8] <= 4) small.push_back({(const uint4*)(h + off[i]), (uint4*)(d + off[i]), len[i] / 16});
    Seg* ds; cudaMalloc(&ds, sizeof(Seg) * small.size());
    cudaMemcpy(ds, small.data(), sizeof(Seg) * small.size(), cudaMemcpyHostToDevice);
    cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e2; cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
    timeit("dma large + sm small", [&] {
      cudaEventRecord(e2, s); cudaStreamWaitEvent(s2, e2, 0);
      k_copy_segs<<<dim3(2, (unsigned)small.size()), 256, 0, s2>>>(ds, (int)small.size());
      for (size_t i = 0; i < off.size(); ++i)
        if (w[i % 8] > 4) cudaMemcpyAsync(d + off[i], h + off[i], len[i], cudaMemcpyHostToDevice, s);
      cudaEventRecord(e2, s2); cudaStreamWaitEvent(s, e2, 0);
    });
    timeit("dma large only", [&] {
      for (size_t i = 0; i < off.size(); ++i)
        if (w[i % 8] > 4) cudaMemcpyAsync(d + off[i], h + off[i], len[i], cudaMemcpyHostToDevice, s);
    });
    timeit("sm small only", [&] { k_copy_segs<<<dim3(2, (unsigned)small.size()), 256, 0, s>>>(ds, (int)small.size()); });
  }
  timeit("sm copy 512 segs", [&] { k_copy_segs<<<dim3(4, 512), 256, 0, s>>>(dsegs, 512); });
  timeit("sm copy 512 segs (16x)", [&] { k_copy_segs<<<dim3(16, 128), 256, 0, s>>>(dsegs, 512); });
  return 0;
}
