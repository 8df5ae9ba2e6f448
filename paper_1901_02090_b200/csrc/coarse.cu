// Coarse space (coarse.py:121-245) on the device.
//
// Local pieces per subdomain, via the interface Schur complement S_i:
//   constrained KKT solve with interface load  <=>  [[S, C^T],[C, 0]]
//   Kc   = (C S^-1 C^T)^-1            (= Psi^T A Psi, coarse.py:179)
//   Psi  = S^-1 C^T Kc                (Gamma rows of the coarse basis, coarse.py:166-171),
//          stored transposed: PsiT = Kc (S^-1 C^T)^T, maxC x maxG per subdomain
//   T    = Gamma block of the constrained inverse (coarse.py:237-245) = Z (Z^T S Z)^-1 Z^T,
//          Z = null(C).  Computed without cancellation as
//          T = (P S P + g Q Q^T)^-1 - Q Q^T / g,  P = I - Q Q^T,  g = tr(S)/n,
//          Q = per-face orthonormal bases of the constraint rows (from the pair kernel).
//   b0   = 1^T B_loc psi = -D_i sum_q sign_q Psi[q]   (coarse.py:184-185)
// The global coarse problem (S_Pi and the pinned pressure block) is handled
// by the nested-dissection multifrontal solver in nd.cu / coarse_nd.py.
#include "common.cuh"

extern "C" int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha, const double* A,
                                  int lda, long long sA, const double* B, int ldb, long long sB, double beta,
                                  double* C, int ldc, long long sC, int batch, int upper, void* stream);
extern "C" int bddc_dgemm_batched_dims(int transA, int transB, int M, int N, int K, double alpha,
                                       const double* A, int lda, long long sA, const double* B, int ldb,
                                       long long sB, double beta, double* C, int ldc, long long sC,
                                       int batch, int upper, const int* dims, int dstride, void* stream);
extern "C" int bddc_spd_inverse_batched_ex(double* M, int n, int ld, long long sM, int batch, int b, void* ws,
                                           int* info, int flags, void* stream);
extern "C" int bddc_spd_inverse_batched(double* M, int n, int ld, long long sM, int batch, int b, void* ws,
                                        int* info, void* stream);

#define PAIR_MMAX 112
#ifndef KC_LEAF
#define KC_LEAF 64   // leaf order of the Kc inverses (maxC = 160: 128 + 32 instead of five 32-leaves)
#endif

namespace {

// C^T (maxG x maxC) per subdomain.  sub_rows[i][r] = {g, face, k, sigma}.
__global__ void coarse_ct_kernel(bddc_geom G, const int* __restrict__ sub_rows, const int* __restrict__ faces,
                                 const int* __restrict__ fslot, const double* __restrict__ rows, int maxsel,
                                 int maxC, double* __restrict__ Ct) {
  const int i = blockIdx.x;
  const int mg = G.maxG;
  double* C = Ct + (size_t)i * mg * maxC;
  for (size_t e = threadIdx.x; e < (size_t)mg * maxC; e += blockDim.x) C[e] = 0.0;
  __syncthreads();
  for (int r = 0; r < maxC; ++r) {
    const int* sr = sub_rows + ((size_t)i * maxC + r) * 4;
    if (sr[0] < 0) continue;
    int f = sr[1], k = sr[2];
    double sg = (double)sr[3];
    int a = faces[4 * f + 2], m = faces[4 * f + 3];
    int side = (sg > 0) ? 1 : 0;  // lower subdomain: face on its high side
    for (int s = threadIdx.x; s < m; s += blockDim.x) {
      int q = fslot[((size_t)i * 6 + a * 2 + side) * G.maxF + s];
      double v = (k == 0) ? 1.0 : rows[((size_t)f * maxsel + (k - 1)) * PAIR_MMAX + s];
      C[(size_t)q * maxC + r] = sg * v;
    }
  }
}

// Identity on the padding of Kinv (rows/cols r >= nc_i).
__global__ void pad_identity_kernel(int maxC, const int* __restrict__ sub_rows, double* __restrict__ K) {
  const int i = blockIdx.x;
  double* Ki = K + (size_t)i * maxC * maxC;
  for (int e = threadIdx.x; e < maxC * maxC; e += blockDim.x) {
    int r = e / maxC, c = e % maxC;
    bool lr = sub_rows[((size_t)i * maxC + r) * 4] >= 0;
    bool lc = sub_rows[((size_t)i * maxC + c) * 4] >= 0;
    if (!lr || !lc) Ki[e] = (r == c) ? 1.0 : 0.0;
  }
}

// b0[i][r] = sigma_r * D_i * sum_q (side_q ? -1 : +1) Psi[q][r]   (warp per row r)
__global__ void b0_kernel(bddc_geom G, const int* __restrict__ gcode, const int* __restrict__ sub_rows,
                          const double* __restrict__ PsiT, const double* __restrict__ Dsub, int maxC,
                          double* __restrict__ b0) {
  const int i = blockIdx.x;
  const int mg = G.maxG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < maxC; r += nw) {
    const int* sr = sub_rows + ((size_t)i * maxC + r) * 4;
    double v = 0.0;
    if (sr[0] >= 0) {
      const double* row = PsiT + ((size_t)i * maxC + r) * mg;
      for (int q = lane; q < mg; q += 32) {
        int code = gcode[(size_t)i * mg + q];
        if (code < 0) continue;
        double p = row[q];
        v += ((code >> 2) & 1) ? -p : p;
      }
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      v *= Dsub[i] * (double)sr[3];
    }
    if (lane == 0) b0[(size_t)i * maxC + r] = v;
  }
}

// Qc (maxG x maxC): orthonormal basis of range(C^T) from the per-face bases
// (qbasis[f][k], or 1/sqrt(m) for the initial row when qbasis is NULL).
__global__ void qc_kernel(bddc_geom G, const int* __restrict__ sub_rows, const int* __restrict__ faces,
                          const int* __restrict__ fslot, const double* __restrict__ qbasis, int maxsel, int maxC,
                          double* __restrict__ Qc) {
  const int i = blockIdx.x;
  const int mg = G.maxG;
  double* Q = Qc + (size_t)i * mg * maxC;
  for (size_t e = threadIdx.x; e < (size_t)mg * maxC; e += blockDim.x) Q[e] = 0.0;
  __syncthreads();
  for (int r = 0; r < maxC; ++r) {
    const int* sr = sub_rows + ((size_t)i * maxC + r) * 4;
    if (sr[0] < 0) continue;
    int f = sr[1], k = sr[2];
    int a = faces[4 * f + 2], m = faces[4 * f + 3];
    int side = (sr[3] > 0) ? 1 : 0;
    for (int s = threadIdx.x; s < m; s += blockDim.x) {
      int q = fslot[((size_t)i * 6 + a * 2 + side) * G.maxF + s];
      double v = qbasis ? qbasis[((size_t)f * (maxsel + 1) + k) * PAIR_MMAX + s] : rsqrt((double)m);
      Q[(size_t)q * maxC + r] = v;
    }
  }
}

// gamma_i = tr(S_i)/n_i ; QtSQ[i] += gamma_i I (live rows)
__global__ void gamma_kernel(int mg, int maxC, const int* __restrict__ nG, const int* __restrict__ sub_rows,
                             const double* __restrict__ S, double* __restrict__ gamma, double* __restrict__ QtSQ) {
  __shared__ double red[32];
  const int i = blockIdx.x;
  const int n = nG[i];
  double acc = 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x) acc += S[((size_t)i * mg + q) * mg + q];
  acc = block_sum(acc, red);
  const double g = (n > 0 && acc > 0.0) ? acc / n : 1.0;
  if (threadIdx.x == 0) gamma[i] = g;
  for (int r = threadIdx.x; r < maxC; r += blockDim.x)
    if (sub_rows[((size_t)i * maxC + r) * 4] >= 0) QtSQ[((size_t)i * maxC + r) * maxC + r] += g;
}

__global__ void scale_rows_kernel(long long per, const double* __restrict__ gamma, double* __restrict__ X) {
  const int i = blockIdx.y;
  const double sc = rsqrt(gamma[i]);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (long long)gridDim.x * blockDim.x)
    X[(size_t)i * per + e] *= sc;
}

// Per-subdomain live GEMM sizes (stride 16): nG_i and nC_i (= live coarse rows).
//  0: (nG, nC, nG)  3: (nC, nC, nG)  6: (nC, nG, nC)  9: (nG, nG, nC)  12: (nG, nC, nC)
__global__ void coarse_dims_kernel(int N, int maxC, const int* __restrict__ nG, const int* __restrict__ sub_rows,
                                   int* __restrict__ dims) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int nc = 0;
  while (nc < maxC && sub_rows[((size_t)i * maxC + nc) * 4] >= 0) ++nc;
  const int ng = nG[i];
  int* d = dims + (size_t)i * 16;
  const int v[15] = {ng, nc, ng, nc, nc, ng, nc, ng, nc, ng, ng, nc, ng, nc, nc};
  for (int k = 0; k < 15; ++k) d[k] = v[k];
  d[15] = 0;
}

// Identity padding for a dense matrix beyond n.
__global__ void pad_tail_identity_kernel(double* M, int n, int npad) {
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long tot = (long long)npad * npad;
  if (e >= tot) return;
  int r = (int)(e / npad), c = (int)(e % npad);
  if (r >= n || c >= n) M[e] = (r == c) ? 1.0 : 0.0;
}

__global__ void copy_kernel(const double* __restrict__ a, double* __restrict__ b, long long n) {
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) b[e] = a[e];
}

}  // namespace

// Per-subdomain coarse pieces (part 1: Kc, Psi, b0 and the live-size table dims;
// part 2: T, independent of part 1 when given its own Ct, Y, inv_ws and dims;
// 3: both).  Workspaces: Ct, Y, E (N*maxG*maxC each),
// inv_ws (bddc_spd_inverse_workspace(max(maxC, maxG), N, 32|64)), gamma (N).
extern "C" int bddc_coarse_local(const bddc_geom* g, const int* sub_rows, const int* faces, const int* fslot,
                                 const int* gcode, const int* nG, const double* rows, const double* qbasis,
                                 int maxsel, const double* S, const double* Sinv, const double* Dsub, int maxC,
                                 double* Ct, double* Y, double* E, double* gamma, double* Kc, double* Psi, double* T,
                                 double* b0, void* inv_ws, int* dims, int* info, int part, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int N = g->N, mg = g->maxG;
  const long long sG = (long long)mg * mg, sGC = (long long)mg * maxC, sCC = (long long)maxC * maxC;
  if (maxC % 32) return bddc_set_error(BDDC_ERR_ARG, "coarse_local: maxC must be a multiple of 32");
  const int* dGCG = dims;
  const int* dCCG = dims + 3;
  const int* dCGC = dims + 6;
  const int* dGGC = dims + 9;
  const int* dGCC = dims + 12;
  int r;
  if (part & 1) {
  coarse_ct_kernel<<<N, 128, 0, s>>>(*g, sub_rows, faces, fslot, rows, maxsel, maxC, Ct);
  LAUNCH_OK();
  // every product below runs on the live nG_i x nC_i blocks only (maxC pads to the
  // largest subdomain's coarse count; the mean is ~5x smaller)
  coarse_dims_kernel<<<(N + 127) / 128, 128, 0, s>>>(N, maxC, nG, sub_rows, dims);
  LAUNCH_OK();
  // Y = Sinv C^T ; Kinv = C Y ; Kc = Kinv^-1 ; PsiT = Kc Y^T ; b0
  if ((r = bddc_dgemm_batched_dims(0, 0, mg, maxC, mg, 1.0, Sinv, mg, sG, Ct, maxC, sGC, 0.0, Y, maxC, sGC, N, 0, dGCG, 16, stream)))
    return r;
  if ((r = bddc_dgemm_batched_dims(1, 0, maxC, maxC, mg, 1.0, Ct, maxC, sGC, Y, maxC, sGC, 0.0, Kc, maxC, sCC, N, 0, dCCG,
                                   16, stream)))
    return r;
  pad_identity_kernel<<<N, 256, 0, s>>>(maxC, sub_rows, Kc);
  LAUNCH_OK();
  if ((r = bddc_spd_inverse_batched(Kc, maxC, maxC, sCC, N, KC_LEAF, inv_ws, info, stream))) return r;
  if ((r = bddc_dgemm_batched_dims(0, 1, maxC, mg, maxC, 1.0, Kc, maxC, sCC, Y, maxC, sGC, 0.0, Psi, mg, sGC, N, 0, dCGC,
                                   16, stream)))
    return r;
  b0_kernel<<<N, 256, 0, s>>>(*g, gcode, sub_rows, Psi, Dsub, maxC, b0);
  LAUNCH_OK();
  }
  if (!(part & 2)) return 0;
  if (!(part & 1)) {
    // part 2 alone (concurrently with part 1 on another stream, with its own Ct, Y,
    // workspace and dims): the live-size table first
    coarse_dims_kernel<<<(N + 127) / 128, 128, 0, s>>>(N, maxC, nG, sub_rows, dims);
    LAUNCH_OK();
  }
  // ---- T = (P S P + g Q Q^T)^-1 - Q Q^T / g   (Q in Ct, S Q in Y, Q^T S Q in E[..maxC^2])
  qc_kernel<<<N, 128, 0, s>>>(*g, sub_rows, faces, fslot, qbasis, maxsel, maxC, Ct);
  LAUNCH_OK();
  if ((r = bddc_dgemm_batched_dims(0, 0, mg, maxC, mg, 1.0, S, mg, sG, Ct, maxC, sGC, 0.0, Y, maxC, sGC, N, 0, dGCG, 16, stream)))
    return r;
  double* QtSQ = Kc;  // Kc is kept: use the tail of E for Q^T S Q instead
  QtSQ = E + (size_t)N * sGC - (size_t)N * sCC;
  if ((r = bddc_dgemm_batched_dims(1, 0, maxC, maxC, mg, 1.0, Ct, maxC, sGC, Y, maxC, sGC, 0.0, QtSQ, maxC, sCC, N, 0, dCCG,
                                   16, stream)))
    return r;
  gamma_kernel<<<N, 128, 0, s>>>(mg, maxC, nG, sub_rows, S, gamma, QtSQ);
  LAUNCH_OK();
  // M = S - Q (SQ)^T - (SQ) Q^T + Q (Q^T S Q + g I) Q^T, built in T
  long long tot = (long long)N * sG;
  copy_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(S, T, tot);
  LAUNCH_OK();
  if ((r = bddc_dgemm_batched_dims(0, 1, mg, mg, maxC, -1.0, Ct, maxC, sGC, Y, maxC, sGC, 1.0, T, mg, sG, N, 1, dGGC, 16, stream)))
    return r;
  if ((r = bddc_dgemm_batched_dims(0, 1, mg, mg, maxC, -1.0, Y, maxC, sGC, Ct, maxC, sGC, 1.0, T, mg, sG, N, 1, dGGC, 16, stream)))
    return r;
  // Y <- Q (Q^T S Q + g I)   (reuse Y)
  if ((r = bddc_dgemm_batched_dims(0, 0, mg, maxC, maxC, 1.0, Ct, maxC, sGC, QtSQ, maxC, sCC, 0.0, Y, maxC, sGC, N, 0, dGCC,
                                   16, stream)))
    return r;
  if ((r = bddc_dgemm_batched_dims(0, 1, mg, mg, maxC, 1.0, Y, maxC, sGC, Ct, maxC, sGC, 1.0, T, mg, sG, N, 1, dGGC, 16, stream)))
    return r;
  // T is consumed through its upper tiles only (bddc_pack_sym): every product
  // on it and its inverse skip the lower triangle
  if ((r = bddc_spd_inverse_batched_ex(T, mg, mg, sG, N, 64, inv_ws, info, 1, stream))) return r;
  // T -= (Q/sqrt g)(Q/sqrt g)^T
  dim3 gsc(64, N);
  scale_rows_kernel<<<gsc, 256, 0, s>>>(sGC, gamma, Ct);
  LAUNCH_OK();
  if ((r = bddc_dgemm_batched_dims(0, 1, mg, mg, maxC, -1.0, Ct, maxC, sGC, Ct, maxC, sGC, 1.0, T, mg, sG, N, 1, dGGC, 16, stream)))
    return r;
  return 0;
}

// Identity on rows/columns >= n of a dense npad x npad matrix.
extern "C" int bddc_pad_identity(double* M, int n, int npad, void* stream) {
  long long tot = (long long)npad * npad;
  pad_tail_identity_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(M, n, npad);
  LAUNCH_OK();
  return 0;
}
