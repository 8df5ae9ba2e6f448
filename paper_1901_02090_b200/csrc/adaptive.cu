// Adaptive constraint selection: one CTA per subdomain pair (face).
//
// Reference (adaptive.py:63-173) solves, per pair, the dense n x n pencil
//   Pi (I-E)^T S (I-E) Pi w = lambda Pi S Pi w,  S = blockdiag(S_i, S_j)
// (n = |Gamma_i| + |Gamma_j|, up to 800 at config 3) with two eigh calls.
// (I - E) = U V^T has rank m (= shared dofs of the face), u_s = dj_s e_a - di_s e_b,
// v_s = e_a - e_b, and the face constraint rows act on V^T w only, so the
// nonzero spectrum equals that of the m x m pencil
//   A y = lambda M^{-1} y,  y in null(C_f),
//   A = U^T S U = Dj S_i[sh,sh] Dj + Di S_j[sh,sh] Di,
//   M = V^T S^{-1} V = S_i^{-1}[sh,sh] + S_j^{-1}[sh,sh].
// With M = R R^T (Cholesky) and y = R z:  R^T A R z = lambda z, z in null(C_f R).
// Before adaptivity each face carries only its initial row C_f = 1^T
// (coarse.py:111-118), so null(C_f R) is the complement of q = R^T 1/|R^T 1|.
// The harvested row (adaptive.py:400-416) is L w restricted to the i side,
// which reduces to  c = (I - 11^T/m) (A R) z,  normalised to unit max.
// Rows then pass the reference's Gram-Schmidt dependence test per face
// (coarse.py:61-100; rows on other faces have disjoint support).
#include "common.cuh"

#define PAIR_MMAX 112

namespace {

__device__ __forceinline__ void jacobi_pair(int round, int k, int n, int& p, int& q) {
  // circle method over n (even) players, player n-1 fixed
  if (k == 0) {
    p = round;
    q = n - 1;
  } else {
    p = (round + k) % (n - 1);
    q = (round - k + (n - 1)) % (n - 1);
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// Symmetric eigen-decomposition of X (m x m, leading dim ld) by parallel
// cyclic Jacobi; eigenvectors accumulate in V.  Uses rot (3 * mpad/2).
__device__ void jacobi_eig(double* X, double* V, int m, int ld, double* rot, double* red) {
  const int mp = m + (m & 1);
  for (int e = threadIdx.x; e < m * ld; e += blockDim.x) {
    int r = e / ld, c = e % ld;
    if (c < m) V[e] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    // convergence: off-diagonal mass relative to the diagonal
    double off = 0.0, dia = 0.0;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      int r = e / m, c = e % m;
      double v = X[r * ld + c];
      if (r == c) dia += v * v;
      else off += v * v;
    }
    off = block_sum(off, red);
    dia = block_sum(dia, red);
    if (off <= 1e-30 * dia || off == 0.0) break;
    for (int round = 0; round < mp - 1; ++round) {
      for (int k = threadIdx.x; k < mp / 2; k += blockDim.x) {
        int p, q;
        jacobi_pair(round, k, mp, p, q);
        double c = 1.0, s = 0.0;
        if (q < m) {
          double apq = X[p * ld + q];
          double app = X[p * ld + p], aqq = X[q * ld + q];
          if (fabs(apq) > 1e-300 && fabs(apq) > 1e-18 * sqrt(fabs(app * aqq))) {
            double th = (aqq - app) / (2.0 * apq);
            double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        }
        rot[3 * k] = c;
        rot[3 * k + 1] = s;
      }
      __syncthreads();
      // columns: X <- X J, V <- V J
      const int npair = mp / 2;
      for (int e = threadIdx.x; e < npair * m; e += blockDim.x) {
        int k = e / m, r = e % m;
        double c = rot[3 * k], s = rot[3 * k + 1];
        if (s == 0.0) continue;
        int p, q;
        jacobi_pair(round, k, mp, p, q);
        double xp = X[r * ld + p], xq = X[r * ld + q];
        X[r * ld + p] = c * xp - s * xq;
        X[r * ld + q] = s * xp + c * xq;
        double vp = V[r * ld + p], vq = V[r * ld + q];
        V[r * ld + p] = c * vp - s * vq;
        V[r * ld + q] = s * vp + c * vq;
      }
      __syncthreads();
      // rows: X <- J^T X
      for (int e = threadIdx.x; e < npair * m; e += blockDim.x) {
        int k = e / m, cidx = e % m;
        double c = rot[3 * k], s = rot[3 * k + 1];
        if (s == 0.0) continue;
        int p, q;
        jacobi_pair(round, k, mp, p, q);
        double xp = X[p * ld + cidx], xq = X[q * ld + cidx];
        X[p * ld + cidx] = c * xp - s * xq;
        X[q * ld + cidx] = s * xp + c * xq;
      }
      __syncthreads();
    }
  }
}

__global__ void pair_eig_kernel(bddc_geom G, const int* __restrict__ faces, const int* __restrict__ fslot,
                                const double* __restrict__ S, const double* __restrict__ Sinv,
                                const double* __restrict__ delta, double tau, int maxsel,
                                double* __restrict__ lam_out, int lam_ld, int* __restrict__ nsel,
                                int* __restrict__ nadd, double* __restrict__ rows, double* __restrict__ omega,
                                double* __restrict__ scratch, int* __restrict__ err) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ int bad;
  const int f = blockIdx.x;
  const int i = faces[4 * f], j = faces[4 * f + 1], a = faces[4 * f + 2], m = faces[4 * f + 3];
  const int ld = m + ((m & 1) ? 0 : 1);
  const int mg = G.maxG;
  double* X = sm;                 // m x ld
  double* Y = X + m * ld;         // m x ld
  double* vec = Y + m * ld;       // 4 * m
  double* rot = vec + 4 * m;      // 3 * (m/2 + 1)
  int* qi = (int*)(rot + 3 * (m / 2 + 1));
  int* qj = qi + m;
  double* T1 = scratch + (size_t)f * PAIR_MMAX * PAIR_MMAX;  // A R, m x m
  if (threadIdx.x == 0) bad = 0;
  for (int s = threadIdx.x; s < m; s += blockDim.x) {
    qi[s] = fslot[((size_t)i * 6 + a * 2 + 1) * G.maxF + s];
    qj[s] = fslot[((size_t)j * 6 + a * 2 + 0) * G.maxF + s];
  }
  __syncthreads();
  const double* Si = S + (size_t)i * mg * mg;
  const double* Sj = S + (size_t)j * mg * mg;
  const double* Ii = Sinv + (size_t)i * mg * mg;
  const double* Ij = Sinv + (size_t)j * mg * mg;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    int s = e / m, t = e % m;
    int as = qi[s], at = qi[t], bs = qj[s], bt = qj[t];
    double dis = delta[(size_t)i * mg + as], dit = delta[(size_t)i * mg + at];
    double djs = delta[(size_t)j * mg + bs], djt = delta[(size_t)j * mg + bt];
    // u_s = dj_s e_a - di_s e_b with di/dj the weights of i/j at shared dof s
    X[s * ld + t] = djs * djt * Si[(size_t)as * mg + at] + dis * dit * Sj[(size_t)bs * mg + bt];
    Y[s * ld + t] = Ii[(size_t)as * mg + at] + Ij[(size_t)bs * mg + bt];
  }
  __syncthreads();
  // Cholesky Y = R R^T (lower), symmetrised input
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      double d = Y[k * ld + k];
      if (!(d > 0.0)) {
        bad = 1;
        d = 1.0;
      }
      Y[k * ld + k] = sqrt(d);
    }
    __syncthreads();
    double dk = Y[k * ld + k];
    for (int r = k + 1 + threadIdx.x; r < m; r += blockDim.x) Y[r * ld + k] /= dk;
    __syncthreads();
    for (int e = threadIdx.x; e < (m - k - 1) * (m - k - 1); e += blockDim.x) {
      int r = k + 1 + e / (m - k - 1), c = k + 1 + e % (m - k - 1);
      if (c <= r) Y[r * ld + c] -= Y[r * ld + k] * Y[c * ld + k];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    int r = e / m, c = e % m;
    if (c > r) Y[r * ld + c] = 0.0;
  }
  __syncthreads();
  // X <- X R  (row by row through vec), save T1 = A R
  for (int r = 0; r < m; ++r) {
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      double acc = 0.0;
      for (int k = c; k < m; ++k) acc += X[r * ld + k] * Y[k * ld + c];
      vec[c] = acc;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      X[r * ld + c] = vec[c];
      T1[(size_t)r * m + c] = vec[c];
    }
    __syncthreads();
  }
  // X <- R^T X (column by column)
  for (int c = 0; c < m; ++c) {
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double acc = 0.0;
      for (int k = r; k < m; ++k) acc += Y[k * ld + r] * X[k * ld + c];
      vec[r] = acc;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < m; r += blockDim.x) X[r * ld + c] = vec[r];
    __syncthreads();
  }
  // symmetrise and project out q = R^T 1 / |R^T 1|
  double* qv = vec;       // m
  double* bq = vec + m;   // m
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double acc = 0.0;
    for (int k = r; k < m; ++k) acc += Y[k * ld + r];
    qv[r] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    int r = e / m, c = e % m;
    if (c > r) {
      double v = 0.5 * (X[r * ld + c] + X[c * ld + r]);
      X[r * ld + c] = v;
      X[c * ld + r] = v;
    }
  }
  double nq = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) nq += qv[r] * qv[r];
  nq = sqrt(block_sum(nq, red));
  for (int r = threadIdx.x; r < m; r += blockDim.x) qv[r] /= nq;
  __syncthreads();
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc += X[r * ld + k] * qv[k];
    bq[r] = acc;
  }
  __syncthreads();
  double sq = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) sq += qv[r] * bq[r];
  sq = block_sum(sq, red);
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    int r = e / m, c = e % m;
    X[r * ld + c] += -qv[r] * bq[c] - bq[r] * qv[c] + sq * qv[r] * qv[c];
  }
  __syncthreads();
  jacobi_eig(X, Y, m, ld, rot, red);
  // sort eigenvalues descending (rank by value, ties by index)
  double* lam = vec;            // m
  int* order = (int*)(vec + m); // m ints
  for (int r = threadIdx.x; r < m; r += blockDim.x) lam[r] = fmax(X[r * ld + r], 0.0);
  __syncthreads();
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    int rank = 0;
    for (int k = 0; k < m; ++k) rank += (lam[k] > lam[r]) || (lam[k] == lam[r] && k < r);
    order[rank] = r;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < lam_ld; r += blockDim.x)
    lam_out[(size_t)f * lam_ld + r] = (r < m) ? lam[order[r]] : 0.0;
  if (threadIdx.x == 0) {
    int k = 0;
    while (k < m && lam[order[k]] > tau) ++k;
    // omega = max(first eigenvalue <= tau, 1); the full pencil always has zeros
    omega[f] = (k < m) ? fmax(lam[order[k]], 1.0) : 1.0;
    nsel[f] = k;
    if (k > maxsel) bad |= 2;
  }
  __syncthreads();
  int k = nsel[f];
  if (k > maxsel) k = maxsel;
  // candidate rows: c = (I - 11^T/m) T1 z, normalised to unit max;
  // Gram-Schmidt dependence filter against 1/sqrt(m) and accepted rows.
  double* cv = vec + 2 * m;      // m
  double* basis = X;             // reuse X rows as orthonormal basis (<= m rows)
  for (int c = threadIdx.x; c < m; c += blockDim.x) basis[c] = rsqrt((double)m);
  __syncthreads();
  int nb = 1, added = 0;
  for (int l = 0; l < k; ++l) {
    int col = order[l];
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double acc = 0.0;
      for (int t = 0; t < m; ++t) acc += T1[(size_t)r * m + t] * Y[t * ld + col];
      cv[r] = acc;
    }
    __syncthreads();
    double mean = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) mean += cv[r];
    mean = block_sum(mean, red) / m;
    double mx = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      cv[r] -= mean;
      mx = fmax(mx, fabs(cv[r]));
    }
    mx = block_max(mx, red);
    if (mx == 0.0) continue;
    for (int r = threadIdx.x; r < m; r += blockDim.x) cv[r] /= mx;
    __syncthreads();
    // residual after one projection (independence test) then two-pass GS
    double nv = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) nv += cv[r] * cv[r];
    nv = sqrt(block_sum(nv, red));
    double* w = vec + 3 * m;
    for (int r = threadIdx.x; r < m; r += blockDim.x) w[r] = cv[r];
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      // classical GS: w -= B^T (B w)
      double* coefs = rot;  // nb <= m entries (rot holds >= 3*(m/2+1) >= m doubles)
      for (int bidx = 0; bidx < nb; ++bidx) {
        double d = 0.0;
        for (int r = threadIdx.x; r < m; r += blockDim.x) d += basis[bidx * ld + r] * w[r];
        d = block_sum(d, red);
        if (threadIdx.x == 0) coefs[bidx] = d;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < m; r += blockDim.x) {
        double acc = w[r];
        for (int bidx = 0; bidx < nb; ++bidx) acc -= coefs[bidx] * basis[bidx * ld + r];
        w[r] = acc;
      }
      __syncthreads();
      if (pass == 0) {
        double nr = 0.0;
        for (int r = threadIdx.x; r < m; r += blockDim.x) nr += w[r] * w[r];
        nr = sqrt(block_sum(nr, red));
        if (!(nr > 1e-10 * fmax(nv, 1.0))) {
          nv = -1.0;  // dependent: drop
          break;
        }
      }
    }
    if (nv < 0.0) continue;
    double nw = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) nw += w[r] * w[r];
    nw = sqrt(block_sum(nw, red));
    if (nb < m) {
      for (int r = threadIdx.x; r < m; r += blockDim.x) basis[nb * ld + r] = w[r] / nw;
      for (int r = threadIdx.x; r < m; r += blockDim.x)
        rows[((size_t)f * maxsel + added) * PAIR_MMAX + r] = cv[r];
    }
    __syncthreads();
    ++nb;
    ++added;
  }
  if (threadIdx.x == 0) {
    nadd[f] = added;
    if (bad) atomicOr(err, bad);
  }
}

}  // namespace

extern "C" size_t bddc_pair_scratch_bytes(int n_faces) {
  return (size_t)n_faces * PAIR_MMAX * PAIR_MMAX * sizeof(double);
}

extern "C" int bddc_pair_eigs(const bddc_geom* g, const int* faces, const int* fslot, const double* S,
                              const double* Sinv, const double* delta, double tau, int maxsel, double* lam_out,
                              int lam_ld, int* nsel, int* nadd, double* rows, double* omega, double* scratch,
                              int* err, void* stream) {
  if (g->maxF > PAIR_MMAX) return bddc_set_error(BDDC_ERR_ARG, "pair face larger than PAIR_MMAX=112 dofs");
  int m = g->maxF;
  int ld = m + ((m & 1) ? 0 : 1);
  size_t shm = (size_t)(2 * m * ld + 4 * m + 3 * (m / 2 + 1)) * sizeof(double) + 2 * m * sizeof(int) + 16;
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(pair_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  pair_eig_kernel<<<g->n_faces, 256, shm, (cudaStream_t)stream>>>(*g, faces, fslot, S, Sinv, delta, tau, maxsel,
                                                                  lam_out, lam_ld, nsel, nadd, rows, omega,
                                                                  scratch, err);
  LAUNCH_OK();
  return 0;
}
