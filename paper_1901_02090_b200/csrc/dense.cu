// Dense FP64 building blocks on the Blackwell FP64 tensor pipe (DMMA).
//
//  * bddc_dgemm_batched: C[b] = alpha*op(A[b])*op(B[b]) + beta*C[b], row-major,
//    64x64x16 CTA tiles, 4 warps x (32x32) warp tiles of mma.sync m8n8k4 f64
//    (SASS DMMA.8x8x4), cp.async double-buffered shared-memory staging.
//    `upper` flags: 1 = upper tiles only (symmetric results); 2/4 = op(A)
//    upper/lower triangular, 8/16 = op(B) upper/lower triangular (skip the
//    K blocks that are zero for the tile).
//  * bddc_spd_inverse_batched: in-place inverse of a batch of SPD matrices the
//    LAPACK potrf -> trtri -> lauum way (M = U^T U, V = U^-1, M^-1 = V V^T),
//    each phase recursive 2x2-blocked with large-K DMMA GEMMs and leaves
//    (<= 64) in shared memory.  Schur complements are Gram updates of the
//    factor, so the result is as accurate as a Cholesky solve (an explicit
//    block inversion loses a further factor of the condition number).
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


__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Load a BM x BK (or BK x BM when K-major) operand tile into shared memory.
// kmajor == false: element (r, k) at g[(r0+r)*ld + k0 + k]  -> s[r*LDK + k]
// kmajor == true : element (r, k) at g[(k0+k)*ld + r0 + r]  -> s[k*LDM + r]

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

// One 64x64 output tile: acc += op(A)[m0.., kbeg..kend) * op(B)[kbeg..kend), n0..),
// cp.async double-buffered through As/Bs (2 x TILE_ELEMS each), DMMA m8n8k4.
// transA: A stored K x M (so op(A) = A^T); transB: B stored N x K.
template <bool transA, bool transB, bool aligned>
__device__ __forceinline__ void tile_mma(double (&acc)[4][4][2], const double* __restrict__ A, int lda,
                                         const double* __restrict__ B, int ldb, int Ml, int Nl, int K, int m0,
                                         int n0, int kbeg, int kend, double (*As)[TILE_ELEMS],
                                         double (*Bs)[TILE_ELEMS], bool idle = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, t = lane & 3;
  kbeg = (kbeg / BK) * BK;
  const int kt0 = kbeg / BK;
  const int nk = (kend > kbeg) ? (kend + BK - 1) / BK : kt0;
  if (kt0 < nk) {
    // A operand rows are m (R = M); B operand rows are n (R = N).
    load_tile<transA, aligned>(As[kt0 & 1], A, lda, Ml, K, m0, kbeg);
    load_tile<!transB, aligned>(Bs[kt0 & 1], B, ldb, Nl, K, n0, kbeg);
    cp_async_commit();
  }
  for (int kt = kt0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_tile<transA, aligned>(As[(kt + 1) & 1], A, lda, Ml, K, m0, (kt + 1) * BK);
      load_tile<!transB, aligned>(Bs[(kt + 1) & 1], B, ldb, Nl, K, n0, (kt + 1) * BK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[kt & 1];
    const double* bs = Bs[kt & 1];
    // idle: this warp's 32x32 output lies strictly below the diagonal of an
    // upper-only diagonal tile (it still stages and synchronises with the CTA)
    if (!idle)
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
}

__device__ __forceinline__ void tile_store(const double (&acc)[4][4][2], double* __restrict__ C, int ldc, int M,
                                           int N, int m0, int n0, double alpha, double beta) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, t = lane & 3;
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

__device__ __forceinline__ void acc_zero(double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

template <bool transA, bool transB, bool aligned>
__global__ void __launch_bounds__(128) dgemm_kernel(int M, int N, int K, double alpha,
                                                    const double* __restrict__ A, int lda, long long sA,
                                                    const double* __restrict__ B, int ldb, long long sB,
                                                    double beta, double* __restrict__ C, int ldc,
                                                    long long sC, int upper, const int* __restrict__ dims,
                                                    int dstride) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  const int bn = blockIdx.x, bm = blockIdx.y, bz = blockIdx.z;
  if ((upper & 1) && bm > bn) return;
  A += bz * sA;
  B += bz * sB;
  C += bz * sC;
  int Ml = M, Nl = N;
  if (dims) {
    // per-batch live sizes (padded batches): operands beyond them read as zero,
    // tiles entirely outside are zero-filled (beta == 0) or skipped
    const int* d = dims + (size_t)bz * dstride;
    const int Mb = imin(d[0], M), Nb = imin(d[1], N);
    K = imin(d[2], K);
    if (bm * BM >= Mb || bn * BN >= Nb) {
      if (beta == 0.0) {
        for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
          const int r = bm * BM + e / BN, c = bn * BN + e % BN;
          if (r < M && c < N) C[(size_t)r * ldc + c] = 0.0;
        }
      }
      return;
    }
    Ml = Mb;
    Nl = Nb;
  }
  __shared__ __align__(16) double As[2][TILE_ELEMS];
  __shared__ __align__(16) double Bs[2][TILE_ELEMS];
  const int m0 = bm * BM, n0 = bn * BN;
  if (beta != 0.0) {
    // the epilogue reads C: start its HBM fetch now (two 128-byte lines of a row
    // per thread), so the read-modify-write does not add a full memory latency
    const int r = m0 + (threadIdx.x >> 1);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = n0 + (threadIdx.x & 1) * 32 + q * 16;
      if (r < M && c < N) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(C + (size_t)r * ldc + c));
    }
  }
  double acc[4][4][2];
  acc_zero(acc);
  // triangular operands: only the K range that can be nonzero for this tile
  int kbeg = 0, kend = K;
  if (upper & 2) kbeg = max(kbeg, m0);           // op(A) upper: k >= m
  if (upper & 4) kend = min(kend, m0 + BM);      // op(A) lower: k <= m
  if (upper & 8) kend = min(kend, n0 + BN);      // op(B) upper: k <= n
  if (upper & 16) kbeg = max(kbeg, n0);          // op(B) lower: k >= n
  // upper-only output: in a diagonal tile the warp at (32, 0) holds only strictly
  // lower entries, which no caller of an upper-only product reads: no DMMA, no store
  const bool idle = (upper & 1) && bm == bn && (threadIdx.x >> 5) == 2;
  tile_mma<transA, transB, aligned>(acc, A, lda, B, ldb, Ml, Nl, K, m0, n0, kbeg, kend, As, Bs, idle);
  if (!idle) tile_store(acc, C, ldc, M, N, m0, n0, alpha, beta);
}

// In-place triangular products (TRMM) of the SPD inverse, no scratch copy:
//  left:  B <- alpha U B   (U upper n1 x n1, B n1 x n2): a CTA owns a 64-column strip
//         and walks its row tiles top-down (tile m reads rows >= m only);
//  right: B <- alpha B U^T (U upper n2 x n2, B n1 x n2): a CTA owns a 64-row strip
//         and walks its column tiles left to right (tile n reads columns >= n only).
template <bool aligned>
__global__ void __launch_bounds__(128) trmm_left_upper_kernel(int n1, int n2, double alpha,
                                                              const double* __restrict__ U, double* B, int ld,
                                                              long long sM) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  const int n0 = blockIdx.x * BN, bz = blockIdx.y;
  const double* Uz = U + bz * sM;
  double* Bz = B + bz * sM;
  __shared__ __align__(16) double As[2][TILE_ELEMS];
  __shared__ __align__(16) double Bs[2][TILE_ELEMS];
  for (int m0 = 0; m0 < n1; m0 += BM) {
    double acc[4][4][2];
    acc_zero(acc);
    tile_mma<false, false, aligned>(acc, Uz, ld, Bz, ld, n1, n2, n1, m0, n0, m0, n1, As, Bs);
    tile_store(acc, Bz, ld, n1, n2, m0, n0, alpha, 0.0);
    __syncthreads();
  }
}

template <bool aligned>
__global__ void __launch_bounds__(128) trmm_right_upperT_kernel(int n1, int n2, double alpha,
                                                                const double* __restrict__ U, double* B, int ld,
                                                                long long sM) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  const int m0 = blockIdx.x * BM, bz = blockIdx.y;
  const double* Uz = U + bz * sM;
  double* Bz = B + bz * sM;
  __shared__ __align__(16) double As[2][TILE_ELEMS];
  __shared__ __align__(16) double Bs[2][TILE_ELEMS];
  for (int n0 = 0; n0 < n2; n0 += BN) {
    double acc[4][4][2];
    acc_zero(acc);
    // op(B)[k][n] = U[n][k]: nonzero for k >= n
    tile_mma<false, true, aligned>(acc, Bz, ld, Uz, ld, n1, n2, n2, m0, n0, n0, n2, As, Bs);
    tile_store(acc, Bz, ld, n1, n2, m0, n0, alpha, 0.0);
    __syncthreads();
  }
}

// ------------------------------------------------------- SPD inverse leaves

// Leaf of the Cholesky-based inverse, on the nb x nb (nb <= 64) diagonal block
// of every matrix: ONE WARP per matrix, block in shared memory (row stride
// nb + 1: column walks are bank-conflict free), warp-synchronous (no CTA
// barriers in the sequential column loops).
//  mode 1 (factor): read the upper triangle, M = U^T U (upper Cholesky),
//          V = U^-1 in place (column-oriented trtri), write V to the upper
//          triangle and zeros below it.
//  mode 2 (lauum):  read V (upper triangle; lower taken as zero), write V V^T.
//  mode 3: both (the whole matrix fits one leaf).
__global__ void __launch_bounds__(32) leaf_chol_inv_kernel(double* M, int nb, int ld, long long sM, int* info,
                                                           int mode) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  extern __shared__ double sd[];
  const int ldp = nb + 1;
  const int lane = threadIdx.x;
  double* Mz = M + blockIdx.x * sM;
  for (int r = 0; r < nb; ++r)
    for (int c = lane; c < nb; c += 32) sd[r * ldp + c] = (c >= r) ? Mz[(size_t)r * ld + c] : 0.0;
  __syncwarp();
  int bad = 0;
  if (mode & 1) {
    // right-looking upper Cholesky: lanes own columns
    for (int k = 0; k < nb; ++k) {
      double d = sd[k * ldp + k];
      if (!(d > 0.0)) {
        bad = 1;
        d = 1.0;
      }
      d = sqrt(d);
      const double id = 1.0 / d;
      __syncwarp();
      for (int c = k + lane; c < nb; c += 32) sd[k * ldp + c] = (c == k) ? d : sd[k * ldp + c] * id;
      __syncwarp();
      for (int c = k + 1 + lane; c < nb; c += 32) {
        const double ukc = sd[k * ldp + c];
        for (int r = k + 1; r <= c; ++r) sd[r * ldp + c] -= sd[k * ldp + r] * ukc;
      }
      __syncwarp();
    }
    // V = U^-1 column by column: V[i][j] = -V[j][j] sum_{k=i}^{j-1} V[i][k] U[k][j]
    for (int j = 0; j < nb; ++j) {
      const double vjj = 1.0 / sd[j * ldp + j];
      double nv[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int i = lane + 32 * t;
        double acc = 0.0;
        if (i < j)
          for (int k = i; k < j; ++k) acc += sd[i * ldp + k] * sd[k * ldp + j];
        nv[t] = -vjj * acc;
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int i = lane + 32 * t;
        if (i < j) sd[i * ldp + j] = nv[t];
      }
      if (lane == 0) sd[j * ldp + j] = vjj;
      __syncwarp();
    }
  }
  if (lane == 0 && bad) atomicCAS(info, 0, (int)blockIdx.x + 1);   // first failing matrix + 1
  if (mode & 2) {
    // X = V V^T: X[r][c] = sum_{k >= max(r,c)} V[r][k] V[c][k]
    for (int r = 0; r < nb; ++r)
      for (int c = r + lane; c < nb; c += 32) {
        double acc = 0.0;
        for (int k = c; k < nb; ++k) acc += sd[r * ldp + k] * sd[c * ldp + k];
        Mz[(size_t)r * ld + c] = acc;
        if (mode == 3) Mz[(size_t)c * ld + r] = acc;
      }
  } else {
    for (int r = 0; r < nb; ++r)
      for (int c = lane; c < nb; c += 32) Mz[(size_t)r * ld + c] = (c >= r) ? sd[r * ldp + c] : 0.0;
  }
}

// The same leaf for nb <= 32 entirely in registers: lane c owns column c (padding
// columns c >= nb carry the identity), the row broadcasts go through warp
// shuffles instead of shared-memory column walks (the shared-memory version is
// bound by shared-memory bandwidth: 2 loads per FMA).  Cholesky and the
// triangular inverse are 496 shuffle+FMA steps each, V V^T 528.
template <int MODE>
__global__ void __launch_bounds__(32) leaf32_chol_inv_kernel(double* M, int nb, int ld, long long sM, int* info) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  __shared__ double tsm[32][33];
  const unsigned FULL = 0xffffffffu;
  const int c = threadIdx.x;
  double* Mz = M + blockIdx.x * sM;
  double x[32];
  if (MODE & 1) {
    double u[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      double v = (c >= nb && r == c) ? 1.0 : 0.0;
      if (r < nb && c < nb && r <= c) v = Mz[(size_t)r * ld + c];
      u[r] = v;
    }
    // right-looking upper Cholesky M = U^T U
    int bad = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      double d = __shfl_sync(FULL, u[k], k);
      if (!(d > 0.0)) {
        bad = 1;
        d = 1.0;
      }
      d = sqrt(d);
      const double id = 1.0 / d;
      u[k] = (c > k) ? u[k] * id : (c == k ? d : u[k]);
#pragma unroll
      for (int r = k + 1; r < 32; ++r) {
        const double ukr = __shfl_sync(FULL, u[k], r);
        if (c >= r) u[r] -= ukr * u[k];
      }
    }
    if (c == 0 && bad) atomicCAS(info, 0, (int)blockIdx.x + 1);   // first failing matrix + 1
    // V = U^-1: column c solves U v = e_c by a backward sweep over the columns of U
#pragma unroll
    for (int r = 0; r < 32; ++r) x[r] = (r == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      const double ukk = __shfl_sync(FULL, u[k], k);
      x[k] = x[k] / ukk;
#pragma unroll
      for (int i = 0; i < k; ++i) {
        const double uik = __shfl_sync(FULL, u[i], k);
        x[i] -= uik * x[k];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < 32; ++r) x[r] = (r < nb && c < nb && r <= c) ? Mz[(size_t)r * ld + c] : 0.0;
  }
  if (MODE & 2) {
    // X = V V^T: lane c takes row c of V through shared memory, then
    // X[i][c] = sum_k V[i][k] V[c][k] with V[i][k] (k >= i) shuffled from lane i
#pragma unroll
    for (int r = 0; r < 32; ++r) tsm[r][c] = x[r];
    __syncwarp();
    double rw[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) rw[k] = tsm[c][k];
    double o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
#pragma unroll
      for (int i = 0; i <= k; ++i) o[i] += __shfl_sync(FULL, rw[k], i) * rw[k];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      if (r < nb && c < nb && r <= c) {
        Mz[(size_t)r * ld + c] = o[r];
        if (MODE == 3) Mz[(size_t)c * ld + r] = o[r];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r < nb && c < nb) Mz[(size_t)r * ld + c] = (r <= c) ? x[r] : 0.0;
  }
}

// The leaf for 32 < nb <= 64: two warps per matrix, thread c owns column c of
// the block in registers (padding columns c >= nb carry the identity); one
// replaces the seven launches of a 64 -> 32 + 32 recursion step.  Row
// broadcasts go through shared memory (double-buffered, ONE barrier per step,
// 16-byte broadcast loads: the leaf is bound by the one-warp-load-per-clock
// shared-memory pipe and the FP64 FMA rate), every thread derives 1/U_kk itself
// from the broadcast unscaled row and updates with a_kr * (U[k][c] / U_kk).
//  MODE 1: upper Cholesky M = U^T U, V = U^-1 (column c solves U v = e_c
//          against U in shared memory), V to the upper triangle, zeros below.
//  MODE 2: X = V V^T from V (upper), upper triangle written.
//  MODE 3: both, full symmetric result.
//  MODE 4 / 5: the two halves of MODE 1 as separate kernels (U through global
//          memory): each unrolled body is half the code, which keeps the
//          instruction cache from thrashing (ncu: "no instruction" was the top stall).
constexpr int L64 = 66;   // shared row stride (doubles): 16-byte rows, 2-way worst case
template <int MODE>
__global__ void __launch_bounds__(64) leaf64_chol_inv_kernel(double* M, int nb, int ld, long long sM, int* info) {
  constexpr bool CHOL = MODE == 1 || MODE == 3 || MODE == 4;
  constexpr bool TRTRI = MODE == 1 || MODE == 3 || MODE == 5;
  constexpr bool LAUUM = MODE == 2 || MODE == 3;
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  __shared__ __align__(16) double sU[64 * L64];
  __shared__ __align__(16) double srow[2][64];
  __shared__ double sinv[64];
  const int c = threadIdx.x;
  double* Mz = M + blockIdx.x * sM;
  if (CHOL) {
    double u[64];
#pragma unroll
    for (int r = 0; r < 64; ++r) {
      double v = (c >= nb && r == c) ? 1.0 : 0.0;
      if (r < nb && c < nb && r <= c) v = Mz[(size_t)r * ld + c];
      u[r] = v;
    }
    int bad = 0;
    // right-looking: row k (unscaled) is broadcast, every thread scales it itself
    // (only 1/U_kk is ever needed: rsqrt); the broadcast reads are 16-byte
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      double* rb = srow[k & 1];
      rb[c] = u[k];
      __syncthreads();
      double a = rb[k];
      if (!(a > 0.0)) {
        bad = 1;
        a = 1.0;
      }
      const double id = rsqrt(a);
      if (c == 0) sinv[k] = id;
      const double ukc = (c > k) ? u[k] * id : (c == k ? a * id : 0.0);
      u[k] = ukc;
      const double w = ukc * id;   // U[k][r] U[k][c] = a_kr (U[k][c] / U_kk)
      const double2* rb2 = reinterpret_cast<const double2*>(rb);
#pragma unroll
      for (int r2 = (k + 1) / 2; r2 < 32; ++r2) {
        const double2 v = rb2[r2];
        if (2 * r2 >= k + 1) u[2 * r2] -= v.x * w;
        u[2 * r2 + 1] -= v.y * w;
      }
    }
    if (c == 0 && bad) atomicCAS(info, 0, (int)blockIdx.x + 1);   // first failing matrix + 1
    if (MODE == 4) {   // U (upper) and 1/U_kk on the otherwise-zero diagonal-below slot
#pragma unroll
      for (int r = 0; r < 64; ++r)
        if (r < nb && c < nb) Mz[(size_t)r * ld + c] = (r <= c) ? u[r] : 0.0;
      __syncthreads();
      if (c < nb && c + 1 < nb) Mz[(size_t)(c + 1) * ld + c] = sinv[c];
      return;
    }
    // U to shared memory (upper; the strict lower part is never read)
#pragma unroll
    for (int r = 0; r < 64; ++r) sU[r * L64 + c] = u[r];
  } else if (TRTRI) {
    // MODE 5: U from MODE 4 (1/U_kk parked in the sub-diagonal slot k+1, k)
#pragma unroll
    for (int r = 0; r < 64; ++r)
      sU[r * L64 + c] = (r < nb && c < nb && r <= c) ? Mz[(size_t)r * ld + c] : (r == c ? 1.0 : 0.0);
    if (c < nb) sinv[c] = (c + 1 < nb) ? Mz[(size_t)(c + 1) * ld + c] : 1.0 / Mz[(size_t)c * ld + c];
    else sinv[c] = 1.0;
  }
  if (TRTRI) {
    __syncthreads();
    // column c of V = U^-1: x[i] = -(1/U_ii) sum_{j>i} U[i][j] x[j], x[c] = 1/U_cc,
    // x[j] = 0 for j > c (so the same unrolled code runs in every thread)
    double x[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) x[j] = 0.0;
#pragma unroll
    for (int i = 63; i >= 0; --i) {
      const double2* ur = reinterpret_cast<const double2*>(sU + i * L64);
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int j2 = (i + 1) / 2; j2 < 32; ++j2) {
        const double2 v = ur[j2];
        if (2 * j2 >= i + 1) s0 += v.x * x[2 * j2];
        s1 += v.y * x[2 * j2 + 1];
      }
      const double vi = sinv[i];
      x[i] = (i == c) ? vi : (i < c ? -vi * (s0 + s1) : 0.0);
    }
    if (!LAUUM) {
#pragma unroll
      for (int r = 0; r < 64; ++r)
        if (r < nb && c < nb) Mz[(size_t)r * ld + c] = (r <= c) ? x[r] : 0.0;
      return;
    }
    __syncthreads();   // every thread is done reading U
#pragma unroll
    for (int r = 0; r < 64; ++r) sU[r * L64 + c] = x[r];   // V, zeros below the diagonal
  } else {
#pragma unroll
    for (int r = 0; r < 64; ++r)
      sU[r * L64 + c] = (r < nb && c < nb && r <= c) ? Mz[(size_t)r * ld + c] : 0.0;
  }
  __syncthreads();
  // X[i][c] = sum_{k >= max(i, c)} V[i][k] V[c][k]: thread c keeps row c of V
  // (zero below k = c), rows i are broadcast from shared memory
  double rw[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) rw[k] = (k >= c) ? sU[c * L64 + k] : 0.0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const double2* vr = reinterpret_cast<const double2*>(sU + i * L64);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k2 = i / 2; k2 < 32; ++k2) {
      const double2 v = vr[k2];
      if (2 * k2 >= i) s0 += v.x * rw[2 * k2];
      s1 += v.y * rw[2 * k2 + 1];
    }
    if (i < nb && c < nb && i <= c) {
      Mz[(size_t)i * ld + c] = s0 + s1;
      if (MODE == 3) Mz[(size_t)c * ld + i] = s0 + s1;
    }
  }
}

// Zero / copy an r x c block (row-major, leading dim ld, batch stride sM / sW).
__global__ void block_copy_kernel(double* dst, int ld, long long sD, const double* src, int lds, long long sS,
                                  int rows, int cols) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  const int z = blockIdx.y;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    int r = (int)(e / cols), c = (int)(e % cols);
    dst[z * sD + (size_t)r * ld + c] = src ? src[z * sS + (size_t)r * lds + c] : 0.0;
  }
}

// Lower triangle of an n x n block from its upper triangle: one 64 x 64 tile
// transpose per CTA, only the nt(nt+1)/2 tiles on or below the diagonal are
// launched (blockIdx.x enumerates them), 16 loads in flight per thread.
__global__ void __launch_bounds__(256) lower_from_upper_kernel(double* M, int n, int ld, long long sM) {
  pdl_trigger();   // dependents may launch once every CTA started (tail overlap)
  pdl_wait();      // all memory of the predecessor grid visible
  __shared__ double t[64][65];
  int bi = (int)((sqrtf(8.0f * blockIdx.x + 1.0f) - 1.0f) * 0.5f);   // target tile row
  while ((bi + 1) * (bi + 2) / 2 <= (int)blockIdx.x) ++bi;
  while (bi * (bi + 1) / 2 > (int)blockIdx.x) --bi;
  const int bj = blockIdx.x - bi * (bi + 1) / 2;                     // bj <= bi
  double* Mz = M + blockIdx.y * sM;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {             // source tile (bj, bi) in the upper triangle
    const int r = bj * 64 + ty + 4 * q, c = bi * 64 + tx;
    v[q] = (r < n && c < n) ? Mz[(size_t)r * ld + c] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) t[ty + 4 * q][tx] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) {             // coalesced rows of the target tile
    const int rr = ty + 4 * q;
    const int r = bi * 64 + rr, c = bj * 64 + tx;
    if (r < n && c < n && r > c) Mz[(size_t)r * ld + c] = t[tx][rr];
  }
}

}  // namespace

extern "C" int bddc_dgemm_batched_dims(int transA, int transB, int M, int N, int K, double alpha,
                                       const double* A, int lda, long long sA, const double* B, int ldb,
                                       long long sB, double beta, double* C, int ldc, long long sC,
                                       int batch, int upper, const int* dims, int dstride, void* stream);

extern "C" int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha,
                                  const double* A, int lda, long long sA, const double* B, int ldb,
                                  long long sB, double beta, double* C, int ldc, long long sC,
                                  int batch, int upper, void* stream) {
  return bddc_dgemm_batched_dims(transA, transB, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, batch,
                                 upper, nullptr, 0, stream);
}

extern "C" int bddc_dgemm_batched_dims(int transA, int transB, int M, int N, int K, double alpha,
                                       const double* A, int lda, long long sA, const double* B, int ldb,
                                       long long sB, double beta, double* C, int ldc, long long sC,
                                       int batch, int upper, const int* dims, int dstride, void* stream) {
  if (M <= 0 || N <= 0 || batch <= 0) return 0;
  if (K <= 0) {
    // C = beta*C is not needed by any caller; require K > 0
    return bddc_set_error(BDDC_ERR_ARG, "dgemm: K must be positive");
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  cudaStream_t s = (cudaStream_t)stream;
  bool al = ((((uintptr_t)A) | ((uintptr_t)B)) % 16 == 0) && !((lda | ldb) & 1) && !((sA | sB) & 1);
#define DG_LAUNCH(TA, TB)                                                                                   \
  {                                                                                                         \
    auto kfn = al ? dgemm_kernel<TA, TB, true> : dgemm_kernel<TA, TB, false>;                               \
    CUDA_OK(launch_pdl(kfn, grid, dim3(128), 0, s, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, \
                       upper, dims, dstride));                                                              \
  }
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
  (void)b;
  return (size_t)batch * ((size_t)n * n / 2 + 2 * (size_t)n + 64) * sizeof(double) + 64;
}

namespace {

int block_copy(double* dst, int ld, long long sD, const double* src, int lds, long long sS, int rows, int cols,
               int batch, cudaStream_t s) {
  long long tot = (long long)rows * cols;
  int gx = (int)((tot + 255) / 256);
  if (gx > 64) gx = 64;
  CUDA_OK(launch_pdl(block_copy_kernel, dim3(gx, batch), dim3(256), 0, s, dst, ld, sD, src, lds, sS, rows, cols));
  LAUNCH_OK();
  return 0;
}

// The in-place TRMMs walk a strip's tiles in sequence: worth it only when the
// strips alone fill the GPU (batched small matrices), not for a few large ones.
bool trmm_inplace_pays(int n1, int n2, int batch) {
  const long long strips = (long long)batch * ((imin(n1, n2) + 63) / 64);
  return strips >= 2 * 148 && imax(n1, n2) <= 512;
}

int trmm_launch(int right, int n1, int n2, double alpha, const double* U, double* B, int ld, long long sM,
                int batch, cudaStream_t s) {
  const bool al = !(((uintptr_t)U | (uintptr_t)B) & 15) && !(ld & 1) && !(sM & 1);
  if (!right) {
    dim3 g((n2 + BN - 1) / BN, batch);
    auto kfn = al ? trmm_left_upper_kernel<true> : trmm_left_upper_kernel<false>;
    CUDA_OK(launch_pdl(kfn, g, dim3(128), 0, s, n1, n2, alpha, U, B, ld, sM));
  } else {
    dim3 g((n1 + BM - 1) / BM, batch);
    auto kfn = al ? trmm_right_upperT_kernel<true> : trmm_right_upperT_kernel<false>;
    CUDA_OK(launch_pdl(kfn, g, dim3(128), 0, s, n1, n2, alpha, U, B, ld, sM));
  }
  LAUNCH_OK();
  return 0;
}

static int g_leaf_regs = 1;
static int g_leaf_split = 1;

int leaf_launch(double* M, int n, int ld, long long sM, int batch, int* info, int mode, cudaStream_t s) {
  if (n <= 32 && g_leaf_regs) {
    auto kfn = mode == 1 ? leaf32_chol_inv_kernel<1> : (mode == 2 ? leaf32_chol_inv_kernel<2> : leaf32_chol_inv_kernel<3>);
    CUDA_OK(launch_pdl(kfn, dim3(batch), dim3(32), 0, s, M, n, ld, sM, info));
    LAUNCH_OK();
    return 0;
  }
  if (n <= 64 && g_leaf_regs) {
    if (mode == 1 && g_leaf_split) {
      CUDA_OK(launch_pdl(leaf64_chol_inv_kernel<4>, dim3(batch), dim3(64), 0, s, M, n, ld, sM, info));
      CUDA_OK(launch_pdl(leaf64_chol_inv_kernel<5>, dim3(batch), dim3(64), 0, s, M, n, ld, sM, info));
      LAUNCH_OK();
      return 0;
    }
    auto kfn = mode == 1 ? leaf64_chol_inv_kernel<1> : (mode == 2 ? leaf64_chol_inv_kernel<2> : leaf64_chol_inv_kernel<3>);
    CUDA_OK(launch_pdl(kfn, dim3(batch), dim3(64), 0, s, M, n, ld, sM, info));
    LAUNCH_OK();
    return 0;
  }
  size_t shm = (size_t)n * (n + 1) * sizeof(double);
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(leaf_chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  CUDA_OK(launch_pdl(leaf_chol_inv_kernel, dim3(batch), dim3(32), shm, s, M, n, ld, sM, info, mode));
  LAUNCH_OK();
  return 0;
}

// Split point of the 2x2 recursion: a multiple of the GEMM tile (64) when the
// block is large, so the DMMA GEMMs run on whole tiles (448 -> 256 + 192 rather
// than 224 + 224, whose 3.5-tile edges waste a quarter of every product);
// otherwise a multiple of the leaf size.
int split_of(int n, int b) {
  const int q = (n > 128) ? 64 : b;
  int n1 = ((n / 2 + q - 1) / q) * q;
  if (n1 >= n) n1 = ((n / 2 + b - 1) / b) * b;
  if (n1 >= n) n1 = n - b;
  return n1;
}

// Factor phase: overwrite the upper triangle of every n x n block with
// V = U^-1 where M = U^T U, and the strict lower triangle with zeros.
//   M = [A B; B^T C]:  V11 = rec(A);  U12 = V11^T B;  C <- C - U12^T U12;
//   V22 = rec(C);  V12 = -V11 U12 V22.
// The Schur complement is formed as a Gram update of the Cholesky factor, so
// rounding never sees an explicitly inverted pivot block (LAPACK potrf/trtri).
int chol_inv_rec(double* M, int n, int ld, long long sM, int batch, int b, double* ws, int* info, cudaStream_t s,
                 bool tile_aligned) {
  if (n <= b) return leaf_launch(M, n, ld, sM, batch, info, 1, s);
  const int n1 = split_of(n, b), n2 = n - n1;
  double* A = M;
  double* B = M + n1;
  double* C = M + (size_t)n1 * ld + n1;
  double* W = ws;                                  // batch x n1 x n2
  double* ws_next = ws + (size_t)batch * n1 * n2;
  const long long sW = (long long)n1 * n2;
  int r;
  if ((r = chol_inv_rec(A, n1, ld, sM, batch, b, ws_next, info, s, tile_aligned))) return r;
  if ((r = bddc_dgemm_batched(1, 0, n1, n2, n1, 1.0, A, ld, sM, B, ld, sM, 0.0, W, n2, sW, batch, 4, s))) return r;
  if ((r = bddc_dgemm_batched(1, 0, n2, n2, n1, -1.0, W, n2, sW, W, n2, sW, 1.0, C, ld, sM, batch, 1, s))) return r;
  if ((r = chol_inv_rec(C, n2, ld, sM, batch, b, ws_next, info, s, tile_aligned && n1 % BM == 0))) return r;
  if (trmm_inplace_pays(n1, n2, batch)) {
    if ((r = bddc_dgemm_batched(0, 0, n1, n2, n2, 1.0, W, n2, sW, C, ld, sM, 0.0, B, ld, sM, batch, 8, s))) return r;
    if ((r = trmm_launch(0, n1, n2, -1.0, A, B, ld, sM, batch, s))) return r;   // B <- -V11 B
  } else {
    // few matrices: full-grid GEMMs through the scratch block, then a copy
    if ((r = bddc_dgemm_batched(0, 0, n1, n2, n2, 1.0, W, n2, sW, C, ld, sM, 0.0, B, ld, sM, batch, 8, s))) return r;
    if ((r = bddc_dgemm_batched(0, 0, n1, n2, n1, -1.0, A, ld, sM, B, ld, sM, 0.0, W, n2, sW, batch, 2, s))) return r;
    if ((r = block_copy(B, ld, sM, W, n2, sW, n1, n2, batch, s))) return r;
  }
  // The strict lower block is read only where it lies inside a diagonal GEMM
  // tile (the triangular K-range skipping works on whole 64-tiles): when this
  // block and all its ancestors start on a tile boundary and the split is one,
  // it is never read and the final lower_from_upper overwrites it.
  if (tile_aligned && n1 % BM == 0) return 0;
  return block_copy(M + (size_t)n1 * ld, ld, sM, nullptr, 0, 0, n2, n1, batch, s);
}

// Lauum phase: upper triangle of V V^T from V (upper, zeros below):
//   [V11 V12; 0 V22] -> [V11 V11^T + V12 V12^T, V12 V22^T; ., V22 V22^T].
int lauum_rec(double* M, int n, int ld, long long sM, int batch, int b, double* ws, int* info, cudaStream_t s) {
  if (n <= b) return leaf_launch(M, n, ld, sM, batch, info, 2, s);
  const int n1 = split_of(n, b), n2 = n - n1;
  double* A = M;
  double* B = M + n1;
  double* C = M + (size_t)n1 * ld + n1;
  double* W = ws;
  double* ws_next = ws + (size_t)batch * n1 * n2;
  const long long sW = (long long)n1 * n2;
  int r;
  if ((r = lauum_rec(A, n1, ld, sM, batch, b, ws_next, info, s))) return r;
  if ((r = bddc_dgemm_batched(0, 1, n1, n1, n2, 1.0, B, ld, sM, B, ld, sM, 1.0, A, ld, sM, batch, 1, s))) return r;
  if (trmm_inplace_pays(n1, n2, batch)) {
    if ((r = trmm_launch(1, n1, n2, 1.0, C, B, ld, sM, batch, s))) return r;   // B <- V12 V22^T
  } else {
    if ((r = bddc_dgemm_batched(0, 1, n1, n2, n2, 1.0, B, ld, sM, C, ld, sM, 0.0, W, n2, sW, batch, 16, s))) return r;
    if ((r = block_copy(B, ld, sM, W, n2, sW, n1, n2, batch, s))) return r;
  }
  return lauum_rec(C, n2, ld, sM, batch, b, ws_next, info, s);
}

}  // namespace

extern "C" void bddc_set_leaf_regs(int on) {
  g_leaf_regs = on & 1;
  g_leaf_split = (on >> 1) & 1;
}

// In-place inverse of `batch` SPD matrices of order n (full symmetric storage,
// leading dim ld, batch stride sM): M = U^T U, V = U^-1, M^-1 = V V^T, all
// recursive with DMMA GEMMs above leaves of order <= b.  (No diagonal
// rescaling: Cholesky-based inversion is insensitive to it, van der Sluis.)
// `ws` must hold bddc_spd_inverse_workspace(n, batch, b) bytes; `info` (device
// int) counts non-positive pivots.
extern "C" int bddc_spd_inverse_batched_ex(double* Mat, int n, int ld, long long sM, int batch, int b, void* ws,
                                           int* info, int flags, void* stream);

extern "C" int bddc_spd_inverse_batched(double* Mat, int n, int ld, long long sM, int batch, int b, void* ws,
                                        int* info, void* stream) {
  return bddc_spd_inverse_batched_ex(Mat, n, ld, sM, batch, b, ws, info, 0, stream);
}

// In-situ timing log of every batched SPD inverse (bench: the setup's own
// factorisation roofline).  Off by default; when on, each call records a pair of
// events on its own stream (no synchronisation) and bddc_spd_log_read resolves them.
namespace {
struct SpdLogEntry {
  int n, batch, flags;
  cudaEvent_t e0, e1;
};
constexpr int SPD_LOG_MAX = 256;
SpdLogEntry g_spd_log[SPD_LOG_MAX];
int g_spd_log_n = 0;
bool g_spd_log_on = false;
}  // namespace

extern "C" void bddc_spd_log_enable(int on) {
  for (int k = 0; k < g_spd_log_n; ++k) {
    cudaEventDestroy(g_spd_log[k].e0);
    cudaEventDestroy(g_spd_log[k].e1);
  }
  g_spd_log_n = 0;
  g_spd_log_on = on != 0;
}

// out[4k..4k+3] = {n, batch, flags, milliseconds}; returns the number of entries
// (synchronises on each entry's end event).
extern "C" int bddc_spd_log_read(double* out, int max_entries) {
  int k = 0;
  for (; k < g_spd_log_n && k < max_entries; ++k) {
    float ms = 0.f;
    CUDA_OK(cudaEventSynchronize(g_spd_log[k].e1));
    CUDA_OK(cudaEventElapsedTime(&ms, g_spd_log[k].e0, g_spd_log[k].e1));
    out[4 * k] = g_spd_log[k].n;
    out[4 * k + 1] = g_spd_log[k].batch;
    out[4 * k + 2] = g_spd_log[k].flags;
    out[4 * k + 3] = ms;
  }
  return k;
}

static int spd_inverse_impl(double* Mat, int n, int ld, long long sM, int batch, int b, void* ws, int* info,
                            int flags, cudaStream_t s);

// flags & 1: only the upper triangle of the result is wanted (no lower mirror;
// the strict lower triangle is left undefined).
extern "C" int bddc_spd_inverse_batched_ex(double* Mat, int n, int ld, long long sM, int batch, int b, void* ws,
                                           int* info, int flags, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!g_spd_log_on || g_spd_log_n >= SPD_LOG_MAX || n <= 0 || batch <= 0)
    return spd_inverse_impl(Mat, n, ld, sM, batch, b, ws, info, flags, s);
  SpdLogEntry& e = g_spd_log[g_spd_log_n++];
  e.n = n;
  e.batch = batch;
  e.flags = flags;
  CUDA_OK(cudaEventCreate(&e.e0));
  CUDA_OK(cudaEventCreate(&e.e1));
  CUDA_OK(cudaEventRecord(e.e0, s));
  const int r = spd_inverse_impl(Mat, n, ld, sM, batch, b, ws, info, flags, s);
  CUDA_OK(cudaEventRecord(e.e1, s));
  return r;
}

static int spd_inverse_impl(double* Mat, int n, int ld, long long sM, int batch, int b, void* ws, int* info,
                            int flags, cudaStream_t s) {
  if (n <= 0 || batch <= 0) return 0;
  if (b <= 0 || b > 64) return bddc_set_error(BDDC_ERR_ARG, "spd_inverse: leaf size must be in 1..64");
  double* rest = (double*)ws;
  int r;
  if (n <= b) {
    if ((r = leaf_launch(Mat, n, ld, sM, batch, info, 3, s))) return r;
  } else {
    if ((r = chol_inv_rec(Mat, n, ld, sM, batch, b, rest, info, s, true))) return r;
    if ((r = lauum_rec(Mat, n, ld, sM, batch, b, rest, info, s))) return r;
    if (flags & 1) return 0;
    const int nt = (n + 63) / 64;
    CUDA_OK(launch_pdl(lower_from_upper_kernel, dim3(nt * (nt + 1) / 2, batch), dim3(256), 0, s, Mat, n, ld, sM));
    LAUNCH_OK();
  }
  return 0;
}
