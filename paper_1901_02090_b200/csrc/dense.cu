// Dense FP64 building blocks on the Blackwell FP64 tensor pipe (DMMA).
//
//  * bddc_dgemm_batched: C[b] = alpha*op(A[b])*op(B[b]) + beta*C[b], row-major,
//    64x64x16 CTA tiles, 4 warps x (32x32) warp tiles of mma.sync m8n8k4 f64
//    (SASS DMMA.8x8x4), cp.async double-buffered shared-memory staging.
//    Optional upper-tile mask for symmetric updates.
//  * bddc_spd_inverse_batched: in-place inverse of a batch of SPD matrices by
//    the blocked symmetric sweep (Gauss-Jordan without pivoting; every pivot
//    block is a Schur complement of an SPD matrix, hence SPD).  Each step is
//    a small pivot-block inverse plus two DMMA GEMMs; the bulk of the flops is
//    the symmetric rank-b trailing update.
//
// These replace SuperLU / LAPACK getrf+getrs / dense inverses of the
// reference (substructure.py:66, coarse.py:159,196) with explicit inverses
// that turn every later solve into a bandwidth-bound GEMV.
#include "common.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDK = BK + 4;    // [m][k] layout stride (doubles)
constexpr int LDM = BM + 4;    // [k][m] layout stride (doubles)
constexpr int TILE_ELEMS = (BM * LDK > BK * LDM) ? BM * LDK : BK * LDM;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Load a BM x BK (or BK x BM when K-major) operand tile into shared memory.
// kmajor == false: element (r, k) at g[(r0+r)*ld + k0 + k]  -> s[r*LDK + k]
// kmajor == true : element (r, k) at g[(k0+k)*ld + r0 + r]  -> s[k*LDM + r]
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

template <bool kmajor, bool aligned>
__device__ __forceinline__ void load_tile(double* s, const double* g, int ld, int R, int K,
                                          int r0, int k0) {
  const int tid = threadIdx.x;
  if (!aligned) {
    // element-wise 8-byte copies (odd leading dimensions)
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int c = tid + it * 128;
      int r, k;
      if (!kmajor) {
        r = c >> 4;
        k = c & 15;
      } else {
        k = c >> 6;
        r = c & 63;
      }
      int gr = r0 + r, gk = k0 + k;
      bool ok = gr < R && gk < K;
      const double* src = ok ? (kmajor ? g + (size_t)gk * ld + gr : g + (size_t)gr * ld + gk) : g;
      double* dst = kmajor ? s + k * LDM + r : s + r * LDK + k;
      cp_async8(dst, src, ok ? 8 : 0);
    }
    return;
  }
  if (!kmajor) {
    // 64 rows x 16 doubles = 64 x 8 chunks of 2 doubles; 128 threads x 4
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int c = tid + it * 128;
      int r = c >> 3, kc = (c & 7) * 2;
      int gr = r0 + r, gk = k0 + kc;
      int bytes = 0;
      const double* src = g;
      if (gr < R && gk < K) {
        bytes = (K - gk >= 2) ? 16 : 8;
        src = g + (size_t)gr * ld + gk;
      }
      cp_async16(s + r * LDK + kc, src, bytes);
    }
  } else {
    // 16 k-rows x 64 doubles = 16 x 32 chunks
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int c = tid + it * 128;
      int k = c >> 5, rc = (c & 31) * 2;
      int gk = k0 + k, gr = r0 + rc;
      int bytes = 0;
      const double* src = g;
      if (gk < K && gr < R) {
        bytes = (R - gr >= 2) ? 16 : 8;
        src = g + (size_t)gk * ld + gr;
      }
      cp_async16(s + k * LDM + rc, src, bytes);
    }
  }
}

template <bool kmajor>
__device__ __forceinline__ double frag(const double* s, int r, int k) {
  return kmajor ? s[k * LDM + r] : s[r * LDK + k];
}

// transA: A stored K x M (so op(A) = A^T); transB: B stored N x K.
template <bool transA, bool transB, bool aligned>
__global__ void __launch_bounds__(128) dgemm_kernel(int M, int N, int K, double alpha,
                                                    const double* __restrict__ A, int lda, long long sA,
                                                    const double* __restrict__ B, int ldb, long long sB,
                                                    double beta, double* __restrict__ C, int ldc,
                                                    long long sC, int upper) {
  const int bn = blockIdx.x, bm = blockIdx.y, bz = blockIdx.z;
  if (upper && bm > bn) return;
  A += bz * sA;
  B += bz * sB;
  C += bz * sC;
  __shared__ __align__(16) double As[2][TILE_ELEMS];
  __shared__ __align__(16) double Bs[2][TILE_ELEMS];
  const int m0 = bm * BM, n0 = bn * BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, t = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + BK - 1) / BK;
  // A operand rows are m (R = M); B operand rows are n (R = N).
  load_tile<transA, aligned>(As[0], A, lda, M, K, m0, 0);
  load_tile<!transB, aligned>(Bs[0], B, ldb, N, K, n0, 0);
  cp_async_commit();
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_tile<transA, aligned>(As[(kt + 1) & 1], A, lda, M, K, m0, (kt + 1) * BK);
      load_tile<!transB, aligned>(Bs[(kt + 1) & 1], B, ldb, N, K, n0, (kt + 1) * BK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[kt & 1];
    const double* bs = Bs[kt & 1];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = frag<transA>(as, wm + i * 8 + g, kk + t);
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = frag<!transB>(bs, wn + j * 8 + g, kk + t);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = m0 + wm + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = n0 + wn + j * 8 + 2 * t;
      double* cp = C + (size_t)r * ldc + c;
      if (c < N) {
        double v = alpha * acc[i][j][0];
        cp[0] = (beta == 0.0) ? v : v + beta * cp[0];
      }
      if (c + 1 < N) {
        double v = alpha * acc[i][j][1];
        cp[1] = (beta == 0.0) ? v : v + beta * cp[1];
      }
    }
  }
}

// ---------------------------------------------------------------- sweep

// Pivot step of the blocked symmetric sweep: per matrix, read the b x b pivot
// block D (upper storage), invert it in shared memory (scalar sweep), write
// Dinv and the pre-step row panel X[k][c] = M[kb+k][c] (full row, read from the
// upper triangle).
__global__ void sweep_pivot_kernel(double* M, int n, int ld, long long sM, int kb, int b,
                                   double* X, double* Dinv, int* info) {
  extern __shared__ double sd[];  // b*b
  const int z = blockIdx.x;
  double* Mz = M + z * sM;
  double* Xz = X + (size_t)z * b * n;
  double* Dz = Dinv + (size_t)z * b * b;
  const int nt = blockDim.x;
  for (int e = threadIdx.x; e < b * b; e += nt) {
    int r = e / b, c = e % b;
    int rr = imin(r, c), cc = imax(r, c);
    sd[e] = Mz[(size_t)(kb + rr) * ld + kb + cc];
  }
  __syncthreads();
  // scalar symmetric sweep on the b x b block: result -D^{-1}
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    double piv = sd[k * b + k];
    if (!(piv > 0.0)) {
      if (threadIdx.x == 0) bad = 1;
      piv = 1.0;
    }
    double ip = 1.0 / piv;
    __syncthreads();
    for (int e = threadIdx.x; e < b * b; e += nt) {
      int r = e / b, c = e % b;
      if (r == k || c == k) continue;
      sd[e] -= sd[r * b + k] * sd[k * b + c] * ip;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < b; e += nt) {
      if (e == k) continue;
      double v = sd[e * b + k] * ip;
      sd[e * b + k] = v;
      sd[k * b + e] = v;
    }
    if (threadIdx.x == 0) sd[k * b + k] = -ip;
    __syncthreads();
  }
  if (threadIdx.x == 0 && bad) atomicAdd(info, 1);
  for (int e = threadIdx.x; e < b * b; e += nt) Dz[e] = -sd[e];
  // row panel: c >= kb from row kb+k; c < kb from column (upper storage)
  for (int e = threadIdx.x; e < b * n; e += nt) {
    int c, k;
    double v;
    if (e < b * kb) {  // k fastest: read rows c < kb contiguous over k
      c = e / b;
      k = e % b;
      v = Mz[(size_t)c * ld + kb + k];
    } else {
      int e2 = e - b * kb;
      int w = n - kb;
      k = e2 / w;
      c = kb + e2 % w;
      int r = kb + k;
      v = (c >= r) ? Mz[(size_t)r * ld + c] : Mz[(size_t)c * ld + r];
    }
    Xz[(size_t)k * n + c] = v;
  }
}

// Write the swept K row/column: M[K, c] = W[:, c] (upper part), M[K,K] = -Dinv.
__global__ void sweep_fix_kernel(double* M, int n, int ld, long long sM, int kb, int b,
                                 const double* W, const double* Dinv) {
  const int z = blockIdx.y;
  double* Mz = M + z * sM;
  const double* Wz = W + (size_t)z * b * n;
  const double* Dz = Dinv + (size_t)z * b * b;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= b * n) return;
  int k = e / n, c = e % n;
  if (c >= kb && c < kb + b) {
    int r = c - kb;
    if (k <= r) Mz[(size_t)(kb + k) * ld + c] = -Dz[k * b + r];
  } else if (c >= kb + b) {
    Mz[(size_t)(kb + k) * ld + c] = Wz[(size_t)k * n + c];
  } else {
    Mz[(size_t)c * ld + kb + k] = Wz[(size_t)k * n + c];
  }
}

// A^{-1} = -M (upper) mirrored to full storage.
__global__ void sweep_final_kernel(double* M, int n, int ld, long long sM) {
  const int z = blockIdx.y;
  double* Mz = M + z * sM;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  int r = (int)(e / n), c = (int)(e % n);
  if (r > c) return;
  double v = -Mz[(size_t)r * ld + c];
  Mz[(size_t)r * ld + c] = v;
  if (r != c) Mz[(size_t)c * ld + r] = v;
}

}  // namespace

extern "C" int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha,
                                  const double* A, int lda, long long sA, const double* B, int ldb,
                                  long long sB, double beta, double* C, int ldc, long long sC,
                                  int batch, int upper, void* stream) {
  if (M <= 0 || N <= 0 || batch <= 0) return 0;
  if (K <= 0) {
    // C = beta*C is not needed by any caller; require K > 0
    return bddc_set_error(BDDC_ERR_ARG, "dgemm: K must be positive");
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  cudaStream_t s = (cudaStream_t)stream;
  bool al = ((((uintptr_t)A) | ((uintptr_t)B)) % 16 == 0) && !((lda | ldb) & 1) && !((sA | sB) & 1);
#define DG_LAUNCH(TA, TB)                                                                                   \
  if (al)                                                                                                   \
    dgemm_kernel<TA, TB, true><<<grid, 128, 0, s>>>(M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, upper); \
  else                                                                                                      \
    dgemm_kernel<TA, TB, false><<<grid, 128, 0, s>>>(M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, upper);
  if (!transA && !transB) {
    DG_LAUNCH(false, false)
  } else if (transA && !transB) {
    DG_LAUNCH(true, false)
  } else if (!transA && transB) {
    DG_LAUNCH(false, true)
  } else {
    DG_LAUNCH(true, true)
  }
#undef DG_LAUNCH
  LAUNCH_OK();
  return 0;
}

extern "C" size_t bddc_spd_inverse_workspace(int n, int batch, int b) {
  return (size_t)batch * (2 * (size_t)b * n + (size_t)b * b) * sizeof(double) + 16;
}

// In-place inverse of `batch` SPD matrices of order n (leading dim ld, batch
// stride sM).  Only the upper triangle of the input is read.  `ws` must hold
// bddc_spd_inverse_workspace(n, batch, b) bytes; `info` (device int) counts
// non-positive pivots (NumericalFailureError on the host side).
extern "C" int bddc_spd_inverse_batched(double* Mat, int n, int ld, long long sM, int batch, int b,
                                        void* ws, int* info, void* stream) {
  if (n <= 0 || batch <= 0) return 0;
  if (n % b) return bddc_set_error(BDDC_ERR_ARG, "spd_inverse: n must be a multiple of b");
  if (ld & 1) return bddc_set_error(BDDC_ERR_ARG, "spd_inverse: ld must be even");
  cudaStream_t s = (cudaStream_t)stream;
  double* X = (double*)ws;
  double* W = X + (size_t)batch * b * n;
  double* Dinv = W + (size_t)batch * b * n;
  size_t shm = (size_t)b * b * sizeof(double);
  if (shm > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(sweep_pivot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  for (int kb = 0; kb < n; kb += b) {
    sweep_pivot_kernel<<<batch, 256, shm, s>>>(Mat, n, ld, sM, kb, b, X, Dinv, info);
    LAUNCH_OK();
    // W = Dinv * X   (b x n)
    int r = bddc_dgemm_batched(0, 0, b, n, b, 1.0, Dinv, b, (long long)b * b, X, n, (long long)b * n,
                               0.0, W, n, (long long)b * n, batch, 0, stream);
    if (r) return r;
    // M -= X^T W   (upper tiles only)
    r = bddc_dgemm_batched(1, 0, n, n, b, -1.0, X, n, (long long)b * n, W, n, (long long)b * n, 1.0,
                           Mat, ld, sM, batch, 1, stream);
    if (r) return r;
    dim3 gf((b * n + 255) / 256, batch);
    sweep_fix_kernel<<<gf, 256, 0, s>>>(Mat, n, ld, sM, kb, b, W, Dinv);
    LAUNCH_OK();
  }
  dim3 gfin((unsigned)(((long long)n * n + 255) / 256), batch);
  sweep_final_kernel<<<gfin, 256, 0, s>>>(Mat, n, ld, sM);
  LAUNCH_OK();
  return 0;
}
