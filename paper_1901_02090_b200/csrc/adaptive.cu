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
// Eigen-solve: Householder tridiagonalisation, bisection for every eigenvalue
// (Sturm counts), inverse iteration with full reorthogonalisation for the
// eigenvalues above tau, back-transformation by the reflectors.
// Rows then pass the reference's Gram-Schmidt dependence test per face
// (coarse.py:61-100; rows on other faces have disjoint support).
#include "common.cuh"

#define PAIR_MMAX 112

namespace {

// Sturm count: number of eigenvalues of the symmetric tridiagonal (d, e) below x.
__device__ int sturm_below(const double* d, const double* e, int m, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) ++cnt;
  for (int k = 1; k < m; ++k) {
    q = d[k] - x - e[k - 1] * e[k - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) ++cnt;
  }
  return cnt;
}

// Inverse iteration on (T - lam I) for a symmetric tridiagonal with partial
// pivoting (LAPACK dgttrf/dgtts2 pattern): tri_shift_factor once per shift,
// tri_shift_apply per iteration (b overwritten by the solution).
__device__ void tri_shift_factor(const double* d0, const double* e0, int m, double lam, double tiny, double* dd,
                                 double* du, double* du2, double* dl, unsigned char* piv) {
  for (int i = 0; i < m; ++i) {
    dd[i] = d0[i] - lam;
    if (i < m - 1) {
      du[i] = e0[i];
      dl[i] = e0[i];
    }
    du2[i] = 0.0;
    piv[i] = 0;
  }
  for (int i = 0; i < m - 1; ++i) {
    if (fabs(dd[i]) >= fabs(dl[i])) {
      if (dd[i] == 0.0) dd[i] = tiny;
      double f = dl[i] / dd[i];
      dl[i] = f;
      dd[i + 1] -= f * du[i];
    } else {
      double f = dd[i] / dl[i];
      dd[i] = dl[i];
      dl[i] = f;
      double t = du[i];
      du[i] = dd[i + 1];
      dd[i + 1] = t - f * dd[i + 1];
      if (i < m - 2) {
        du2[i] = du[i + 1];
        du[i + 1] = -f * du[i + 1];
      }
      piv[i] = 1;
    }
  }
  if (dd[m - 1] == 0.0) dd[m - 1] = tiny;
}

__device__ void tri_shift_apply(int m, const double* dd, const double* du, const double* du2, const double* dl,
                                const unsigned char* piv, double* b) {
  for (int i = 0; i < m - 1; ++i) {
    if (!piv[i]) {
      b[i + 1] -= dl[i] * b[i];
    } else {
      double t = b[i];
      b[i] = b[i + 1];
      b[i + 1] = t - dl[i] * b[i];
    }
  }
  b[m - 1] /= dd[m - 1];
  if (m > 1) b[m - 2] = (b[m - 2] - du[m - 2] * b[m - 1]) / dd[m - 2];
  for (int i = m - 3; i >= 0; --i) b[i] = (b[i] - du[i] * b[i + 1] - du2[i] * b[i + 2]) / dd[i];
}

__global__ void pair_eig_kernel(bddc_geom G, const int* __restrict__ faces, const int* __restrict__ fslot,
                                const double* __restrict__ S, const double* __restrict__ Sinv,
                                const double* __restrict__ delta, double tau, int maxsel,
                                double* __restrict__ lam_out, int lam_ld, int* __restrict__ nsel,
                                int* __restrict__ nadd, double* __restrict__ rows, double* __restrict__ omega,
                                double* __restrict__ scratch, double* __restrict__ qbasis, int* __restrict__ err,
                                const int* __restrict__ flist, int full) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ int bad;
  const int f = flist ? flist[blockIdx.x] : blockIdx.x;
  const int i = faces[4 * f], j = faces[4 * f + 1], a = faces[4 * f + 2], m = faces[4 * f + 3];
  const int ld = m + ((m & 1) ? 0 : 1);
  const int mg = G.maxG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* X = sm;                 // m x ld
  double* Y = X + m * ld;         // m x ld
  double* vec = Y + m * ld;       // 4 m
  double* aux = vec + 4 * m;      // 3 (m/2 + 1) >= m
  int* qi = (int*)(aux + 3 * (m / 2 + 1));
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
  // ---- Cholesky M = R R^T (lower, in Y): every thread takes the pivot itself
  // (two barriers per column), trailing update warp per row, lanes over columns
  for (int k = 0; k < m; ++k) {
    double d = Y[k * ld + k];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) bad = 1;
      d = 1.0;
    }
    const double dk = sqrt(d);
    for (int r = k + 1 + threadIdx.x; r < m; r += blockDim.x) Y[r * ld + k] /= dk;
    __syncthreads();
    if (threadIdx.x == 0) Y[k * ld + k] = dk;   // read again only after the next barrier
    for (int r = k + 1 + warp; r < m; r += nw) {
      const double yrk = Y[r * ld + k];
      for (int c = k + 1 + lane; c <= r; c += 32) Y[r * ld + c] -= yrk * Y[c * ld + k];
    }
    __syncthreads();
  }
  for (int r = warp; r < m; r += nw)
    for (int c = r + 1 + lane; c < m; c += 32) Y[r * ld + c] = 0.0;
  __syncthreads();
  // ---- T1 = A R (global scratch), then X = R^T T1, both one-shot (warp per row)
  for (int r = warp; r < m; r += nw)
    for (int c = lane; c < m; c += 32) {
      double acc = 0.0;
      for (int k = c; k < m; ++k) acc += X[r * ld + k] * Y[k * ld + c];
      T1[(size_t)r * m + c] = acc;
    }
  __syncthreads();
  for (int r = warp; r < m; r += nw)
    for (int c = lane; c < m; c += 32) {
      double acc = 0.0;
      for (int k = r; k < m; ++k) acc += Y[k * ld + r] * T1[(size_t)k * m + c];
      X[r * ld + c] = acc;
    }
  __syncthreads();
  // ---- symmetrise and project out q = R^T 1 / |R^T 1|
  double* qv = vec;       // m
  double* bq = vec + m;   // m
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double acc = 0.0;
    for (int k = r; k < m; ++k) acc += Y[k * ld + r];
    qv[r] = acc;
  }
  __syncthreads();
  for (int r = warp; r < m; r += nw)
    for (int c = r + 1 + lane; c < m; c += 32) {
      double v = 0.5 * (X[r * ld + c] + X[c * ld + r]);
      X[r * ld + c] = v;
      X[c * ld + r] = v;
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
  for (int r = warp; r < m; r += nw) {
    const double qr = qv[r], br = bq[r];
    for (int c = lane; c < m; c += 32) X[r * ld + c] += -qr * bq[c] - br * qv[c] + sq * qr * qv[c];
  }
  __syncthreads();
  // ---- Householder tridiagonalisation of X (Y rows hold the reflectors v_j).
  // Three barriers per column: the column norm and v.p are reduced by every warp
  // itself (same lane partition and shuffle tree in every warp: identical values),
  // and q = p - K v is formed inside the rank-2 update.
  double* pv = vec;       // m
  for (int jj = 0; jj + 2 < m; ++jj) {
    const int n1 = m - jj - 1;   // length of the column below the diagonal
    double sx = 0.0;
    for (int r = lane; r < n1; r += 32) {
      const double t = X[(jj + 1 + r) * ld + jj];
      sx += t * t;
    }
    for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
    const double x0 = X[(jj + 1) * ld + jj];
    const double nrm = sqrt(sx);
    const double alpha = (x0 >= 0.0) ? -nrm : nrm;
    const double vn2 = sx - x0 * x0 + (x0 - alpha) * (x0 - alpha);
    const bool skip = !(vn2 > 0.0) || nrm == 0.0;
    const double inv = skip ? 0.0 : 1.0 / sqrt(vn2);
    double* v = Y + jj * ld;   // reflector j stored in row jj (entries jj+1..m-1)
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double val = 0.0;
      if (r > jj) val = (r == jj + 1 ? x0 - alpha : X[r * ld + jj]) * inv;
      v[r] = val;
    }
    __syncthreads();
    if (!skip) {
      // p = A22 v  (rows/cols jj+1..m-1)
      for (int r = jj + 1 + warp; r < m; r += nw) {
        double acc = 0.0;
        for (int c = jj + 1 + lane; c < m; c += 32) acc += X[r * ld + c] * v[c];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) pv[r] = acc;
      }
      __syncthreads();
      double K = 0.0;
      for (int r = jj + 1 + lane; r < m; r += 32) K += v[r] * pv[r];
      for (int o = 16; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
      for (int r = jj + 1 + warp; r < m; r += nw) {
        const double vr = v[r], qr = pv[r] - K * vr;
        for (int c = jj + 1 + lane; c < m; c += 32)
          X[r * ld + c] -= 2.0 * (vr * (pv[c] - K * v[c]) + qr * v[c]);
      }
      if (threadIdx.x == 0) {
        X[(jj + 1) * ld + jj] = alpha;
        X[jj * ld + jj + 1] = alpha;
      }
    }
    __syncthreads();
  }
  // ---- eigenvalues of the tridiagonal by bisection (thread per eigenvalue)
  double* dg = vec;          // m
  double* eo = vec + m;      // m
  double* lam = vec + 2 * m; // m, ascending
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    dg[r] = X[r * ld + r];
    eo[r] = (r + 1 < m) ? X[(r + 1) * ld + r] : 0.0;
  }
  __syncthreads();
  double tnorm = 0.0, gl = 1e308, gu = -1e308;
  for (int r = 0; r < m; ++r) {
    double rad = fabs(eo[r]) + (r > 0 ? fabs(eo[r - 1]) : 0.0);
    gl = fmin(gl, dg[r] - rad);
    gu = fmax(gu, dg[r] + rad);
  }
  tnorm = fmax(fabs(gl), fabs(gu));
  const double pivmin = fmax(1e-300, tnorm * 1e-300);
  // only the eigenvalues the selection uses are resolved: those above tau (one
  // Sturm count at tau gives how many) and the next one (omega, adaptive.py:56-60)
  __shared__ int nabove;
  if (threadIdx.x == 0) nabove = (tau < gu) ? m - sturm_below(dg, eo, m, tau, pivmin) : 0;
  __syncthreads();
  const int ntop = full ? m : imin(nabove + 1, m);
  // multisection: a warp per eigenvalue, 32 Sturm counts per round (interval / 33)
  for (int r = warp; r < ntop; r += nw) {
    const int kk = m - 1 - r;
    double lo = gl - 1e-14 * tnorm, hi = gu + 1e-14 * tnorm;
    for (int it = 0; it < 64; ++it) {
      if (hi - lo <= 2e-16 * fmax(fabs(lo), fabs(hi))) break;
      const double w = hi - lo;
      const double x = lo + w * (double)(lane + 1) / 33.0;
      const bool above = sturm_below(dg, eo, m, x, pivmin) > kk;
      const unsigned msk = __ballot_sync(0xffffffffu, above);
      const int fl = msk ? __ffs(msk) - 1 : 32;
      const double nhi = (fl < 32) ? lo + w * (double)(fl + 1) / 33.0 : hi;
      const double nlo = (fl > 0) ? lo + w * (double)fl / 33.0 : lo;
      if (nlo == lo && nhi == hi) break;
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) lam[kk] = 0.5 * (lo + hi);
  }
  __syncthreads();
  // descending order: lam_desc[t] = lam[m-1-t], clipped at 0 (adaptive.py:381);
  // entries beyond the resolved ones are NaN
  for (int r = threadIdx.x; r < lam_ld; r += blockDim.x)
    lam_out[(size_t)f * lam_ld + r] = (r < ntop) ? fmax(lam[m - 1 - r], 0.0) : __longlong_as_double(0x7ff8000000000000LL);
  __shared__ int ksel;
  if (threadIdx.x == 0) {
    int k = 0;
    while (k < ntop && fmax(lam[m - 1 - k], 0.0) > tau) ++k;
    // omega = max(first eigenvalue <= tau, 1); the full pencil always has zeros
    omega[f] = (k < m) ? fmax(fmax(lam[m - 1 - k], 0.0), 1.0) : 1.0;
    nsel[f] = k;
    if (k > maxsel) bad |= 2;
    ksel = k < maxsel ? k : maxsel;
  }
  __syncthreads();
  const int k = ksel;
  // ---- inverse iteration, one thread per selected eigenvalue; vectors -> X rows
  // (one factorisation per shift; the factor arrays live in the rows of X behind
  // the k vectors when they fit, in local memory otherwise)
  if (threadIdx.x < k) {
    const int l = threadIdx.x;
    const double lv = lam[m - 1 - l];
    double loc[4 * PAIR_MMAX];
    double* fac = (5 * k <= m) ? X + (size_t)(k + 4 * l) * ld : loc;
    const int fs = (5 * k <= m) ? ld : PAIR_MMAX;
    double *dd = fac, *du = fac + fs, *du2 = fac + 2 * fs, *dl = fac + 3 * fs;
    double* b = X + (size_t)l * ld;
    unsigned char pvt[PAIR_MMAX];
    for (int r = 0; r < m; ++r) b[r] = 1.0 + 0.5 * sin(1.7 * (r + 1) + 0.61 * (l + 1));
    const double tiny = fmax(2.2e-16 * tnorm, 1e-300);
    tri_shift_factor(dg, eo, m, lv, tiny, dd, du, du2, dl, pvt);
    for (int it = 0; it < 3; ++it) {
      tri_shift_apply(m, dd, du, du2, dl, pvt, b);
      double nb = 0.0;
      for (int r = 0; r < m; ++r) nb += b[r] * b[r];
      nb = 1.0 / sqrt(nb);
      for (int r = 0; r < m; ++r) b[r] *= nb;
    }
  }
  __syncthreads();
  // full reorthogonalisation in descending-eigenvalue order (fixes near-degenerate clusters)
  for (int l = 1; l < k; ++l) {
    for (int pidx = warp; pidx < l; pidx += nw) {
      double dsum = 0.0;
      for (int r = lane; r < m; r += 32) dsum += X[pidx * ld + r] * X[l * ld + r];
      for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
      if (lane == 0) aux[pidx] = dsum;
    }
    __syncthreads();
    double nn = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double v = X[l * ld + r];
      for (int pidx = 0; pidx < l; ++pidx) v -= aux[pidx] * X[pidx * ld + r];
      X[l * ld + r] = v;
      nn += v * v;
    }
    nn = block_sum(nn, red);
    nn = 1.0 / sqrt(nn);
    for (int r = threadIdx.x; r < m; r += blockDim.x) X[l * ld + r] *= nn;
    __syncthreads();
  }
  // ---- back-transform z = H_0 ... H_{m-3} y  (apply H_{m-3} first)
  for (int jj = m - 3; jj >= 0; --jj) {
    const double* v = Y + jj * ld;
    for (int l = warp; l < k; l += nw) {
      double dsum = 0.0;
      for (int r = jj + 1 + lane; r < m; r += 32) dsum += v[r] * X[l * ld + r];
      for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
      if (lane == 0) aux[l] = dsum;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) {
      int l = e / m, r = e % m;
      if (r > jj) X[l * ld + r] -= 2.0 * aux[l] * v[r];
    }
    __syncthreads();
  }
  // ---- candidate rows c = (I - 11^T/m) T1 z, unit max; dependence filter
  // against 1/sqrt(m) and the accepted rows (coarse.py:61-100), basis in Y rows.
  double* cv = vec + 2 * m;      // m (lam no longer needed)
  double* w = vec + 3 * m;       // m
  double* basis = Y;
  for (int c = threadIdx.x; c < m; c += blockDim.x) basis[c] = rsqrt((double)m);
  __syncthreads();
  int nb = 1, added = 0;
  for (int l = 0; l < k; ++l) {
    for (int r = warp; r < m; r += nw) {
      double acc = 0.0;
      for (int t = lane; t < m; t += 32) acc += T1[(size_t)r * m + t] * X[l * ld + t];
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) cv[r] = acc;
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
    double nv = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) nv += cv[r] * cv[r];
    nv = sqrt(block_sum(nv, red));
    for (int r = threadIdx.x; r < m; r += blockDim.x) w[r] = cv[r];
    __syncthreads();
    bool dep = false;
    for (int pass = 0; pass < 2 && !dep; ++pass) {
      // classical GS: w -= B^T (B w), coefficients by one warp each
      for (int bidx = warp; bidx < nb; bidx += nw) {
        double dsum = 0.0;
        for (int r = lane; r < m; r += 32) dsum += basis[bidx * ld + r] * w[r];
        for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        if (lane == 0) aux[bidx] = dsum;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < m; r += blockDim.x) {
        double acc = w[r];
        for (int bidx = 0; bidx < nb; ++bidx) acc -= aux[bidx] * basis[bidx * ld + r];
        w[r] = acc;
      }
      __syncthreads();
      if (pass == 0) {
        double nr = 0.0;
        for (int r = threadIdx.x; r < m; r += blockDim.x) nr += w[r] * w[r];
        nr = sqrt(block_sum(nr, red));
        dep = !(nr > 1e-10 * fmax(nv, 1.0));
      }
    }
    if (dep) continue;
    double nwn = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) nwn += w[r] * w[r];
    nwn = sqrt(block_sum(nwn, red));
    if (nb < m) {
      for (int r = threadIdx.x; r < m; r += blockDim.x) basis[nb * ld + r] = w[r] / nwn;
      for (int r = threadIdx.x; r < m; r += blockDim.x)
        rows[((size_t)f * maxsel + added) * PAIR_MMAX + r] = cv[r];
    }
    __syncthreads();
    ++nb;
    ++added;
  }
  // orthonormal basis of the face's constraint span (initial row + accepted rows), used
  // for the projected Delta-solve operator T (coarse.cu)
  for (int e = threadIdx.x; e < nb * m; e += blockDim.x) {
    int bidx = e / m, r = e % m;
    if (bidx <= maxsel) qbasis[((size_t)f * (maxsel + 1) + bidx) * PAIR_MMAX + r] = basis[bidx * ld + r];
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

// MsMFEM baseline rows (adaptive.py:207-262), one CTA per face (i low, j high),
// in Schur form: the pair-local Darcy problem with a unit source transfer
// (-1 spread over i, +1 over j) and no flow on the pair's other boundaries
// reduces to its shared-face fluxes x:
//   min 1/2 x^T M x - b^T x  s.t.  1^T x = 1   (net outflow of i = its sink)
//   M = S_i[sh,sh] + S_j[sh,sh],  b = rg_i[sh] - rg_j[sh]
// where rg_k is the interface residual of subdomain k's interior solution for
// its unit source distribution (local_solve condense output); the Lagrange
// multiplier is the pair's pressure-constant jump.  The row (outward from i)
// passes the reference's dependence test against the initial row
// (coarse.py:61-100) and is stored raw, with the orthonormal face basis.
__global__ void multiscale_kernel(bddc_geom G, const int* __restrict__ faces, const int* __restrict__ fslot,
                                  const double* __restrict__ S, const double* __restrict__ rg, int maxsel,
                                  double* __restrict__ rows, double* __restrict__ qbasis, int* __restrict__ nadd,
                                  int* __restrict__ err) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ int bad;
  const int f = blockIdx.x;
  const int i = faces[4 * f], j = faces[4 * f + 1], a = faces[4 * f + 2], m = faces[4 * f + 3];
  const int ld = m + ((m & 1) ? 0 : 1);
  const int mg = G.maxG;
  double* M = sm;            // m x ld, Cholesky in place (lower)
  double* y1 = M + m * ld;   // m: M^-1 b
  double* y2 = y1 + m;       // m: M^-1 1
  double* x = y2 + m;        // m
  int* qi = (int*)(x + m);
  int* qj = qi + m;
  if (threadIdx.x == 0) bad = 0;
  for (int s = threadIdx.x; s < m; s += blockDim.x) {
    qi[s] = fslot[((size_t)i * 6 + a * 2 + 1) * G.maxF + s];
    qj[s] = fslot[((size_t)j * 6 + a * 2 + 0) * G.maxF + s];
  }
  __syncthreads();
  const double* Si = S + (size_t)i * mg * mg;
  const double* Sj = S + (size_t)j * mg * mg;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int r = e / m, c = e % m;
    M[r * ld + c] = Si[(size_t)qi[r] * mg + qi[c]] + Sj[(size_t)qj[r] * mg + qj[c]];
  }
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    y1[r] = rg[(size_t)i * mg + qi[r]] - rg[(size_t)j * mg + qj[r]];
    y2[r] = 1.0;
  }
  __syncthreads();
  // Cholesky M = L L^T (lower, in place)
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      double d = M[k * ld + k];
      if (!(d > 0.0)) {
        bad = 1;
        d = 1.0;
      }
      M[k * ld + k] = sqrt(d);
    }
    __syncthreads();
    const double dk = M[k * ld + k];
    for (int r = k + 1 + threadIdx.x; r < m; r += blockDim.x) M[r * ld + k] /= dk;
    __syncthreads();
    const int w = m - k - 1;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int r = k + 1 + e / w, c = k + 1 + e % w;
      if (c <= r) M[r * ld + c] -= M[r * ld + k] * M[c * ld + k];
    }
    __syncthreads();
  }
  // two right-hand sides: forward L z = [b, 1], then back L^T y = z
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      y1[k] /= M[k * ld + k];
      y2[k] /= M[k * ld + k];
    }
    __syncthreads();
    for (int r = k + 1 + threadIdx.x; r < m; r += blockDim.x) {
      y1[r] -= M[r * ld + k] * y1[k];
      y2[r] -= M[r * ld + k] * y2[k];
    }
    __syncthreads();
  }
  for (int k = m - 1; k >= 0; --k) {
    if (threadIdx.x == 0) {
      y1[k] /= M[k * ld + k];
      y2[k] /= M[k * ld + k];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
      y1[r] -= M[k * ld + r] * y1[k];
      y2[r] -= M[k * ld + r] * y2[k];
    }
    __syncthreads();
  }
  double s1 = 0.0, s2 = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    s1 += y1[r];
    s2 += y2[r];
  }
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  const double mu = (1.0 - s1) / s2;
  for (int r = threadIdx.x; r < m; r += blockDim.x) x[r] = y1[r] + mu * y2[r];
  __syncthreads();
  // dependence test against the initial row's basis q0 = 1/sqrt(m), two GS passes
  const double q0 = rsqrt((double)m);
  double nx = 0.0, d1 = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    nx += x[r] * x[r];
    d1 += x[r] * q0;
  }
  nx = sqrt(block_sum(nx, red));
  d1 = block_sum(d1, red);
  double d2 = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) d2 += (x[r] - d1 * q0) * q0;
  d2 = block_sum(d2, red);
  double nr = 0.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    const double v = x[r] - (d1 + d2) * q0;
    nr += v * v;
  }
  nr = sqrt(block_sum(nr, red));
  const bool keep = nr > 1e-10 * fmax(nx, 1.0);
  for (int r = threadIdx.x; r < PAIR_MMAX; r += blockDim.x) {
    qbasis[((size_t)f * (maxsel + 1)) * PAIR_MMAX + r] = (r < m) ? q0 : 0.0;
    if (keep) {
      rows[((size_t)f * maxsel) * PAIR_MMAX + r] = (r < m) ? x[r] : 0.0;
      qbasis[((size_t)f * (maxsel + 1) + 1) * PAIR_MMAX + r] = (r < m) ? (x[r] - (d1 + d2) * q0) / nr : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    nadd[f] = keep ? 1 : 0;
    if (bad) atomicOr(err, 1);
  }
}

extern "C" int bddc_multiscale_rows(const bddc_geom* g, const int* faces, const int* fslot, const double* S,
                                    const double* rg, int maxsel, double* rows, double* qbasis, int* nadd, int* err,
                                    void* stream) {
  if (g->n_faces <= 0) return 0;
  if (g->maxF > PAIR_MMAX) return bddc_set_error(BDDC_ERR_ARG, "pair face larger than PAIR_MMAX=112 dofs");
  if (maxsel < 1) return bddc_set_error(BDDC_ERR_ARG, "multiscale: maxsel must be >= 1");
  const int m = g->maxF;
  const int ld = m + ((m & 1) ? 0 : 1);
  size_t shm = (size_t)(m * ld + 3 * m) * sizeof(double) + 2 * m * sizeof(int) + 16;
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(multiscale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  multiscale_kernel<<<g->n_faces, 256, shm, (cudaStream_t)stream>>>(*g, faces, fslot, S, rg, maxsel, rows, qbasis,
                                                                    nadd, err);
  LAUNCH_OK();
  return 0;
}

static int g_pair_threads_big = 512;
extern "C" void bddc_set_pair_threads(int t) { g_pair_threads_big = (t == 512) ? 512 : 256; }

extern "C" int bddc_pair_eigs(const bddc_geom* g, const int* faces, const int* fslot, const double* S,
                              const double* Sinv, const double* delta, double tau, int maxsel, double* lam_out,
                              int lam_ld, int* nsel, int* nadd, double* rows, double* omega, double* scratch,
                              double* qbasis, int* err, const int* flist, int nlist, int mmax, int full,
                              void* stream) {
  if (g->maxF > PAIR_MMAX) return bddc_set_error(BDDC_ERR_ARG, "pair face larger than PAIR_MMAX=112 dofs");
  // flist == NULL: every face (shared memory sized for maxF); else the nlist faces
  // listed, all with at most mmax shared dofs (smaller faces -> more CTAs per SM)
  const int nblk = flist ? nlist : g->n_faces;
  if (nblk <= 0) return 0;
  const int m = flist ? imin(mmax, g->maxF) : g->maxF;
  const int ld = m + ((m & 1) ? 0 : 1);
  size_t shm = (size_t)(2 * m * ld + 4 * m + 3 * (m / 2 + 1)) * sizeof(double) + 2 * m * sizeof(int) + 16;
  // one CTA per face; faces whose two m x m blocks leave room for one CTA per SM
  // only get 512 threads (latency hiding of the shared-memory sweeps)
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(pair_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  const int threads = (shm > 113 * 1024) ? g_pair_threads_big : 256;
  pair_eig_kernel<<<nblk, threads, shm, (cudaStream_t)stream>>>(*g, faces, fslot, S, Sinv, delta, tau, maxsel, lam_out,
                                                            lam_ld, nsel, nadd, rows, omega, scratch, qbasis, err,
                                                            flist, full);
  LAUNCH_OK();
  return 0;
}
