// K9, banded form: block cyclic reduction of the gauge-fixed system.
//
// Keyframe graphs of SLAM are chains plus loop closures.  Reordered by
// reverse Cuthill-McKee (host, on the keyframe graph), a ring of keyframes
// folds into a band of a few keyframes; grouping m consecutive keyframes
// (m = the bandwidth in keyframes) into super-blocks of w = 7m unknowns makes
// the system block tridiagonal:  T = tridiag(L_s, D_s, L_{s+1}^T).
// Odd-even (cyclic) reduction then eliminates half of the super-blocks per
// level, all of them in parallel (one CTA per block): at level l with stride
// s, every odd active block j factorises D_j (LDL^T, no pivoting, failure
// iff an exact-zero pivot: the SimplicialLDLT semantics) and solves
// D_j [Y_jL, Y_jR, y_j] = [L_j, L_{j+s}^T, b_j]; every even active block i
// then takes  D_i -= L_i Y_{i-s,R} + L_{i+s}^T Y_{i+s,L},
//             b_i -= L_i y_{i-s} + L_{i+s}^T y_{i+s},   L'_i = -L_i Y_{i-s,L}.
// log2(S) levels instead of N sequential panels (the frontal form's chain);
// the last block is solved directly and the back substitution
// x_j = y_j - Y_jL x_{j-s} - Y_jR x_{j+s} walks the levels down.  This is
// LDL^T in an odd-even permuted order — rounding-level differences from the
// reference's AMD-ordered SimplicialLDLT only.
// (included inside namespace pmx by backend.cu, after GNState)

constexpr int kBandMaxW = 84;      // max super-block size (12 keyframes): D + 2w+1 RHS in smem
constexpr int kBandThreads = 256;

struct BandArgs {
  const double* D0;  // [S][w*w] assembled diagonal blocks (undamped, full symmetric)
  const double* L0;  // [S][w*w] L0[j] = A(j, j-1)
  const double* b0;  // [S][w]   rhs = -g (band order)
  double* D;         // work copies (reduced in place)
  double* L;         // L[j] = A(j, j - s) of the active blocks at the current level
  double* b;
  double* Y;         // [S][2][w*w]: Y_jL, Y_jR of block j (each block is odd at exactly one level)
  double* y;         // [S][w]
  double* x;         // [S][w] solution (band order)
  int S, w, npad;    // npad: rows of the last block beyond the system (identity)
  int* status;       // 0 once a pivot was exactly zero
  GNState* st;
};

// LDL^T of the w x w block in shared memory (row-major, full symmetric on
// input; unit L below the diagonal and D on it on output), blocked by 8
// columns: warp 0 factorises the panel's diagonal block in registers (lane r
// holds row r), every thread then forms one row of the panel below it
// (W = A_rp L_pp^-T, L_rp = W D^-1), and the trailing lower triangle takes
// A_rc -= W_r L_c^T.  tmp: 8 * w doubles (W of the panel).  Returns false
// (on every thread) on an exact-zero pivot.
__device__ bool band_ldlt(double* A, int w, double* tmp) {
  constexpr int P = 8;
  __shared__ int bad;
  __shared__ double piv[P];  // 1 / pivot
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) bad = 0;
  for (int p0 = 0; p0 < w; p0 += P) {
    const int nb = min(P, w - p0);
    if (threadIdx.x < 32) {  // diagonal block
      double a[P];
#pragma unroll
      for (int c = 0; c < P; ++c) a[c] = (lane < nb && c <= lane) ? A[(p0 + lane) * w + p0 + c] : 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (p < nb) {
          const double D = __shfl_sync(0xffffffffu, a[p], p);
          if (lane == 0 && D == 0.0) bad = 1;
          const double iD = fast_rcp(D);
          const double wv = a[p];
#pragma unroll
          for (int c = p + 1; c < P; ++c) {
            const double wc = __shfl_sync(0xffffffffu, wv, c);
            if (lane >= c) a[c] -= wv * (wc * iD);
          }
          if (lane > p) a[p] = wv * iD;
          if (lane == p) piv[p] = iD;
        }
      }
      if (lane < nb) {
#pragma unroll
        for (int c = 0; c < P; ++c)
          if (c <= lane) A[(p0 + lane) * w + p0 + c] = a[c];
      }
    }
    __syncthreads();
    if (bad) return false;
    // rows below the panel
    for (int r = p0 + nb + threadIdx.x; r < w; r += blockDim.x) {
      double wv[P];
#pragma unroll
      for (int t = 0; t < P; ++t) wv[t] = t < nb ? A[r * w + p0 + t] : 0.0;
#pragma unroll
      for (int t = 1; t < P; ++t)
#pragma unroll
        for (int u = 0; u < t; ++u) wv[t] -= wv[u] * A[(p0 + t) * w + p0 + u];
#pragma unroll
      for (int t = 0; t < P; ++t) {
        if (t < nb) {
          tmp[t * w + r] = wv[t];
          A[r * w + p0 + t] = wv[t] * piv[t];
        }
      }
    }
    __syncthreads();
    // trailing update of the lower triangle, 2x2 register tiles
    const int m = w - p0 - nb, tiles = (m + 1) / 2;
    for (int t = threadIdx.x; t < tiles * tiles; t += blockDim.x) {
      const int ti = t / tiles, tj = t % tiles;
      if (tj > ti) continue;
      const int r0 = p0 + nb + 2 * ti, c0 = p0 + nb + 2 * tj;
      double acc[2][2] = {};
      for (int u = 0; u < nb; ++u) {
        const double w0 = tmp[u * w + r0], w1 = r0 + 1 < w ? tmp[u * w + r0 + 1] : 0.0;
        const double l0 = A[c0 * w + p0 + u], l1 = c0 + 1 < w ? A[(c0 + 1) * w + p0 + u] : 0.0;
        acc[0][0] = fma(w0, l0, acc[0][0]);
        acc[0][1] = fma(w0, l1, acc[0][1]);
        acc[1][0] = fma(w1, l0, acc[1][0]);
        acc[1][1] = fma(w1, l1, acc[1][1]);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (r0 + i < w && c0 + j <= r0 + i) A[(r0 + i) * w + c0 + j] -= acc[i][j];
    }
    __syncthreads();
  }
  return true;
}

// In place: X (w x n, row-major, leading dimension ld) <- (L D L^T)^-1 X.
// Blocked substitution by 8-row blocks: the diagonal block is solved per
// column (one thread per column, the block's column in registers), then the
// rows below (forward) / above (backward) take a rank-8 update in 4 x 4
// register tiles (columns strided across the threads: conflict-free X rows,
// broadcast L loads) - two FMAs per shared load instead of one per two.
__device__ void band_solve_cols(const double* A, int w, double* X, int n, int ld) {
  constexpr int B = 8;
  __shared__ double rdiag[kBandMaxW];
  for (int r = threadIdx.x; r < w; r += blockDim.x) rdiag[r] = fast_rcp(A[r * w + r]);
  const int ct = (n + 3) / 4;  // column tiles: thread column tc takes tc, tc + ct, tc + 2 ct, tc + 3 ct
  auto col = [&](int tc, int j) { return tc + j * ct; };
  for (int r0 = 0; r0 < w; r0 += B) {  // L z = x
    const int r1 = min(w, r0 + B), nb = r1 - r0;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      double z[B];
#pragma unroll
      for (int i = 0; i < B; ++i) z[i] = i < nb ? X[(r0 + i) * ld + c] : 0.0;
#pragma unroll
      for (int r = 1; r < B; ++r)
#pragma unroll
        for (int k = 0; k < r; ++k)
          if (r < nb) z[r] -= A[(r0 + r) * w + r0 + k] * z[k];
#pragma unroll
      for (int i = 1; i < B; ++i)
        if (i < nb) X[(r0 + i) * ld + c] = z[i];
    }
    __syncthreads();
    const int rt = (w - r1 + 3) / 4;
    for (int t = threadIdx.x; t < rt * ct; t += blockDim.x) {
      const int ra = r1 + 4 * (t / ct), tc = t % ct;
      double acc[4][4] = {};
      for (int k = 0; k < nb; ++k) {
        double av[4], zv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = A[min(ra + i, w - 1) * w + r0 + k];
#pragma unroll
        for (int j = 0; j < 4; ++j) zv[j] = X[(r0 + k) * ld + min(col(tc, j), n - 1)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], zv[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ra + i < w && col(tc, j) < n) X[(ra + i) * ld + col(tc, j)] -= acc[i][j];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < w * n; t += blockDim.x) X[(t / n) * ld + t % n] *= rdiag[t / n];  // D
  __syncthreads();
  for (int r1 = w; r1 > 0; r1 -= B) {  // L^T x = z, from the bottom
    const int r0 = max(0, r1 - B), nb = r1 - r0;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      double z[B];
#pragma unroll
      for (int i = 0; i < B; ++i) z[i] = i < nb ? X[(r0 + i) * ld + c] : 0.0;
#pragma unroll
      for (int r = B - 2; r >= 0; --r)
#pragma unroll
        for (int k = r + 1; k < B; ++k)
          if (k < nb) z[r] -= A[(r0 + k) * w + r0 + r] * z[k];
#pragma unroll
      for (int i = 0; i < B - 1; ++i)
        if (i < nb) X[(r0 + i) * ld + c] = z[i];
    }
    __syncthreads();
    const int rt = (r0 + 3) / 4;
    for (int t = threadIdx.x; t < rt * ct; t += blockDim.x) {
      const int ra = 4 * (t / ct), tc = t % ct;
      double acc[4][4] = {};
      for (int k = 0; k < nb; ++k) {
        double av[4], zv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = A[(r0 + k) * w + min(ra + i, w - 1)];  // L^T
#pragma unroll
        for (int j = 0; j < 4; ++j) zv[j] = X[(r0 + k) * ld + min(col(tc, j), n - 1)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], zv[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ra + i < r0 && col(tc, j) < n) X[(ra + i) * ld + col(tc, j)] -= acc[i][j];
    }
    __syncthreads();
  }
}

// C (w x w, smem) -= op(P) Q with P, Q in shared memory (row-major w x w);
// transP: use P^T.  Each thread owns a 4 x 4 tile of C (register blocking).
__device__ void band_gemm_sub(double* C, const double* P, const double* Q, int w, bool transP, int rb = 0,
                              int re = -1) {
  if (re < 0) re = w;  // output rows [rb, re) (rb a multiple of 4)
  const int tiles = (w + 3) / 4, rtiles = (re - rb + 3) / 4;
  for (int t = threadIdx.x; t < rtiles * tiles; t += blockDim.x) {
    const int r0 = rb + (t / tiles) * 4, c0 = (t % tiles) * 4;
    double acc[4][4] = {};
    for (int q = 0; q < w; ++q) {
      double pv[4], qv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = min(r0 + i, w - 1), c = min(c0 + i, w - 1);
        pv[i] = transP ? P[q * w + r] : P[r * w + q];
        qv[i] = Q[q * w + c];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(pv[i], qv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (r0 + i < re && c0 + j < w) C[(r0 + i) * w + c0 + j] -= acc[i][j];
  }
  __syncthreads();
}

// Global -> shared copy with 8 loads in flight per thread (a plain loop
// exposes one L2 round trip per element per thread).
__device__ __forceinline__ void band_copy_in(double* __restrict__ dst, const double* __restrict__ src, int n) {
  int i = threadIdx.x;
  for (; i + 7 * (int)blockDim.x < n; i += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(src + i + k * blockDim.x);
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[i + k * blockDim.x] = v[k];
  }
  for (; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

// The same into rows of length `w` at stride `ld` (a sub-block of a wider matrix).
__device__ __forceinline__ void band_copy_in_strided(double* __restrict__ dst, const double* __restrict__ src, int n,
                                                     int w, int ld) {
  int i = threadIdx.x;
  for (; i + 7 * (int)blockDim.x < n; i += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(src + i + k * blockDim.x);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = i + k * blockDim.x;
      dst[(e / w) * ld + e % w] = v[k];
    }
  }
  for (; i < n; i += blockDim.x) dst[(i / w) * ld + i % w] = __ldg(src + i);
}

// Attempt `attempt` (backend.cpp:208-227): fresh copies, lambda on every
// diagonal entry, padding rows of the last block as identity.
__global__ void k_bcr_init(BandArgs A, int attempt, double damping_init) {
  if (A.st->stop || A.st->solved) return;
  double lambda = 0.0;
  if (attempt > 0) {
    lambda = damping_init;
    for (int a = 1; a < attempt; ++a) lambda *= 10.0;
  }
  const int w = A.w, S = A.S;
  const size_t nb = (size_t)S * w * w;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nb; i += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / ((size_t)w * w)), rc = (int)(i % ((size_t)w * w)), r = rc / w, c = rc % w;
    const bool pad = s == S - 1 && r >= w - A.npad;
    A.D[i] = (r == c) ? (pad ? 1.0 : A.D0[i] + lambda) : A.D0[i];
    A.L[i] = A.L0[i];
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)S * w; i += (size_t)gridDim.x * blockDim.x)
    A.b[i] = A.b0[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.status = 1;
}

// Level with stride s: odd active block j = s (2t + 1) -> Y_jL, Y_jR, y_j.
__global__ void __launch_bounds__(kBandThreads) k_bcr_eliminate(BandArgs A, int s) {
  if (A.st->stop || A.st->solved) return;
  const int j = s * (2 * blockIdx.x + 1);
  if (j >= A.S) return;
  extern __shared__ double sm[];
  const int w = A.w, n = 2 * w + 1;
  double* Dj = sm;            // w*w
  double* X = Dj + w * w;     // w*n
  double* tmp = X + w * n;    // 8*w
  const bool right = j + s < A.S;
  // X = [A(j, j-s) | A(j, j+s) | b_j] = [L_j | L_{j+s}^T | b_j]: L_{j+s} lands in
  // the D_j slot first and is transposed from there
  if (right) {
    band_copy_in(Dj, A.L + (size_t)(j + s) * w * w, w * w);
    __syncthreads();
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) X[(i % w) * n + w + i / w] = Dj[i];
  } else {
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) X[(i / w) * n + w + i % w] = 0.0;
  }
  __syncthreads();
  band_copy_in(Dj, A.D + (size_t)j * w * w, w * w);
  band_copy_in_strided(X, A.L + (size_t)j * w * w, w * w, w, n);
  for (int r = threadIdx.x; r < w; r += blockDim.x) X[r * n + 2 * w] = A.b[(size_t)j * w + r];
  __syncthreads();
  if (!band_ldlt(Dj, w, tmp)) {
    if (threadIdx.x == 0) *A.status = 0;
    return;
  }
  // this CTA's share of the 2w+1 right-hand sides (blockIdx.y of gridDim.y;
  // every CTA of the block factorises D_j itself)
  const int cb = (int)(((int64_t)n * blockIdx.y) / gridDim.y), ce = (int)(((int64_t)n * (blockIdx.y + 1)) / gridDim.y);
  band_solve_cols(Dj, w, X + cb, ce - cb, n);
  double* Y = A.Y + (size_t)j * 2 * w * w;
  const int nc = ce - cb;
  for (int i = threadIdx.x; i < w * nc; i += blockDim.x) {
    const int r = i / nc, c = cb + i % nc;
    const double v = X[r * n + c];
    if (c < w)
      Y[r * w + c] = v;
    else if (c < 2 * w)
      Y[w * w + r * w + c - w] = v;
    else
      A.y[(size_t)j * w + r] = v;
  }
}

// Level with stride s: even active block i = 2 s t absorbs its odd neighbours.
__global__ void __launch_bounds__(kBandThreads) k_bcr_update(BandArgs A, int s) {
  if (A.st->stop || A.st->solved) return;
  const int i = 2 * s * blockIdx.x;
  if (i >= A.S) return;
  extern __shared__ double sm[];
  const int w = A.w, ww = w * w;
  double* Li = sm;        // A(i, i-s)
  double* Lr = Li + ww;   // A(i+s, i)
  double* Dn = Lr + ww;   // D_i being updated
  double* T = Dn + ww;    // staged Y block
  const bool left = i >= s, right = i + s < A.S;
  const double* YlR = A.Y + (size_t)(i - s) * 2 * ww + ww;  // Y_{i-s,R}
  const double* YlL = A.Y + (size_t)(i - s) * 2 * ww;       // Y_{i-s,L}
  const double* YrL = A.Y + (size_t)(i + s) * 2 * ww;       // Y_{i+s,L}
  double* Di = A.D + (size_t)i * ww;
  // this CTA's rows [rb, re) of every output of block i (blockIdx.y of
  // gridDim.y, multiples of 4).  A CTA reads only its own rows of A(i,i-s),
  // D_i and b_i -- the rows it overwrites itself below -- so the CTAs of one
  // block never read what another one writes in this launch.
  const int rq = (((w + 3) / 4) + gridDim.y - 1) / gridDim.y;
  const int rb = min(w, (int)blockIdx.y * rq * 4), re = min(w, rb + rq * 4);
  if (left)
    band_copy_in(Li + rb * w, A.L + (size_t)i * ww + rb * w, (re - rb) * w);
  else
    for (int k = rb * w + threadIdx.x; k < re * w; k += blockDim.x) Li[k] = 0.0;
  if (right)
    band_copy_in(Lr, A.L + (size_t)(i + s) * ww, ww);  // odd block: not written at this level
  else
    for (int k = threadIdx.x; k < ww; k += blockDim.x) Lr[k] = 0.0;
  band_copy_in(Dn + rb * w, Di + rb * w, (re - rb) * w);
  if (left) band_copy_in(T, YlR, ww);
  __syncthreads();
  // b_i -= A(i,i-s) y_{i-s} + A(i,i+s) y_{i+s}  (rows [rb, re))
  __shared__ double yl[kBandMaxW], yr[kBandMaxW];
  for (int q = threadIdx.x; q < w; q += blockDim.x) {
    yl[q] = left ? A.y[(size_t)(i - s) * w + q] : 0.0;
    yr[q] = right ? A.y[(size_t)(i + s) * w + q] : 0.0;
  }
  __syncthreads();
  for (int r = rb + threadIdx.x; r < re; r += blockDim.x) {
    double acc = A.b[(size_t)i * w + r];
    for (int q = 0; q < w; ++q) acc -= Li[r * w + q] * yl[q] + Lr[q * w + r] * yr[q];
    A.b[(size_t)i * w + r] = acc;
  }
  if (left) band_gemm_sub(Dn, Li, T, w, false, rb, re);  // D_i -= A(i,i-s) Y_{i-s,R}
  if (right) {                                   // D_i -= A(i,i+s) Y_{i+s,L} = L_{i+s}^T Y_{i+s,L}
    band_copy_in(T, YrL, ww);
    __syncthreads();
    band_gemm_sub(Dn, Lr, T, w, true, rb, re);
  }
  // the factorisations read the lower triangle only: rows written as computed
  for (int k = rb * w + threadIdx.x; k < re * w; k += blockDim.x) Di[k] = Dn[k];
  if (left && i >= 2 * s) {  // coupling to the next active block on the left: -A(i,i-s) Y_{i-s,L}
    __syncthreads();         // every thread's Dn rows are in D_i before Dn is reused
    band_copy_in(T, YlL, ww);
    for (int k = rb * w + threadIdx.x; k < re * w; k += blockDim.x) Dn[k] = 0.0;
    __syncthreads();
    band_gemm_sub(Dn, Li, T, w, false, rb, re);
    for (int k = rb * w + threadIdx.x; k < re * w; k += blockDim.x) A.L[(size_t)i * ww + k] = Dn[k];
  }
}

// The last active block: x_0 = D_0^-1 b_0.
__global__ void __launch_bounds__(kBandThreads) k_bcr_top(BandArgs A) {
  if (A.st->stop || A.st->solved) return;
  extern __shared__ double sm[];
  const int w = A.w;
  double* D = sm;
  double* X = D + w * w;
  double* tmp = X + w;  // 8*w
  band_copy_in(D, A.D, w * w);
  for (int r = threadIdx.x; r < w; r += blockDim.x) X[r] = A.b[r];
  __syncthreads();
  if (!band_ldlt(D, w, tmp)) {
    if (threadIdx.x == 0) *A.status = 0;
    return;
  }
  band_solve_cols(D, w, X, 1, 1);
  for (int r = threadIdx.x; r < w; r += blockDim.x) A.x[r] = X[r];
}

// Back substitution at stride s: x_j = y_j - Y_jL x_{j-s} - Y_jR x_{j+s}.
__global__ void __launch_bounds__(kBandThreads) k_bcr_back(BandArgs A, int s) {
  if (A.st->stop || A.st->solved) return;
  const int j = s * (2 * blockIdx.x + 1);
  if (j >= A.S) return;
  const int w = A.w;
  __shared__ double xl[kBandMaxW], xr[kBandMaxW];
  const double* Y = A.Y + (size_t)j * 2 * w * w;
  const bool right = j + s < A.S;
  for (int q = threadIdx.x; q < w; q += blockDim.x) {
    xl[q] = A.x[(size_t)(j - s) * w + q];
    xr[q] = right ? A.x[(size_t)(j + s) * w + q] : 0.0;
  }
  __syncthreads();
  // warp per output row, lanes over q
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < w; r += nw) {
    double acc = 0.0;
    for (int q = lane; q < w; q += 32) acc += Y[r * w + q] * xl[q] + Y[w * w + r * w + q] * xr[q];
    acc = warp_sum(acc);
    if (lane == 0) A.x[(size_t)j * w + r] = A.y[(size_t)j * w + r] - acc;
  }
}

// tau in keyframe order + the accept test of backend.cpp:220-223.
__global__ void k_bcr_finish(BandArgs A, const int* __restrict__ kf_pos, int N, double* __restrict__ tau) {
  if (A.st->stop || A.st->solved) return;
  __shared__ int good;
  if (threadIdx.x == 0) good = *A.status;
  __syncthreads();
  for (int i = threadIdx.x; i < 7 * N; i += blockDim.x) {
    const int k = i / 7, pos = kf_pos[k];
    const double v = pos < 0 ? 0.0 : A.x[(size_t)pos * 7 + i % 7];  // the anchor: tau = 0 (g_a = 0, H_aa = I)
    tau[i] = v;
    if (!isfinite(v) || !(fabs(v) < 1e3)) good = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0 && good) A.st->solved = 1;
}
