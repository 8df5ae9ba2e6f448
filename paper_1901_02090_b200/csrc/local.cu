// Per-subdomain (local) operators for box subdomains, batched one CTA per
// subdomain.  Replaces SubdomainOperator (substructure.py:24-119): instead of
// a SuperLU factorisation of the interior KKT [[A_II,B_I^T,0],[B_I,0,V^T],
// [0,V,0]] we use that A_II is block-diagonal by axis and tridiagonal along
// grid lines, so
//     P   = B_I A_II^{-1} B_I^T        (pressure Schur, summed line blocks)
//     G   = B_G - B_I A_II^{-1} A_IG    (supported on one grid line per slot)
//     S_A = A_GG - A_GI A_II^{-1} A_IG  (diagonal + opposite-end partner)
//     S   = S_A + G^T P^+ G             (Schur complement on Gamma_i)
// with P^+ from the inverse of the Jacobi-scaled, rank-one-regularised P.  D-scaling of B
// (grid.py:344-357) cancels in S and enters only the pressure rhs/solution.
#include "common.cuh"

#define MAXL 32

namespace {

struct SlotLine {
  int a, side, line, L, base, stride;
};

__device__ __forceinline__ int axis_stride(const Box& b, int a) {
  return a == 0 ? 1 : (a == 1 ? b.L[0] : b.L[0] * b.L[1]);
}

__device__ __forceinline__ int line_base(const Box& b, int a, int line) {
  int c[3];
  line_coords(b, a, line, c);
  return local_cell(b, c[0], c[1], c[2]);
}

__device__ __forceinline__ SlotLine decode_slot(const Box& b, int code) {
  SlotLine s;
  s.a = code & 3;
  s.side = (code >> 2) & 1;
  s.line = code >> 3;
  s.L = b.L[s.a];
  s.base = line_base(b, s.a, s.line);
  s.stride = axis_stride(b, s.a);
  return s;
}

// Global cell id of local cell k along line `line` of axis a.
__device__ __forceinline__ int line_cell_global(const bddc_geom& G, const Box& b, int a, int line, int k) {
  int c[3];
  line_coords(b, a, line, c);
  c[a] = k;
  return cell_id(G, b.o[0] + c[0], b.o[1] + c[1], b.o[2] + c[2]);
}

// Interior dofs of a line of L cells: the faces at positions p = 1-lo .. L-1+hi
// (position p separates cells p-1 and p; lo / hi = 1 when that end is a mode-B
// Dirichlet face, which is then an interior dof too), m = L-1+lo+hi of them,
// dof j <-> position p = j+1-lo.  Cell k has low face j = k-1+lo, high k+lo.

// Global dof of line dof j.
__device__ __forceinline__ int line_face_dof(const bddc_geom& G, const Box& b, int a, int line, int j, int lo) {
  int c[3];
  line_coords(b, a, line, c);
  const int p = j + 1 - lo;
  int gc[3] = {b.o[0] + c[0], b.o[1] + c[1], b.o[2] + c[2]};
  if (p == 0) return bnd_dof(G, 0, gc);
  if (p == b.L[a]) return bnd_dof(G, 1, gc);
  gc[a] += p;
  return face_dof(G, a, gc[0], gc[1], gc[2]);
}

// Thomas factorisation of the line tridiagonal T (order m = L-1+lo+hi):
// T[j][j] = dg (c_{p-1} + c_p) (cells that exist), T[j][j+1] = of c_p, p = j+1-lo,
// with the element block c [[dg, of], [of, dg]]: (2, 1) consistent RT0, (3, 0)
// lumped (grid.py:220-225).  Stores the modified super-diagonal cp and the reciprocal
// pivots piv (one division per dof here, none in the solves).
__device__ __forceinline__ void line_factor(const double* c, int L, int lo, int hi, double* cp, double* piv,
                                            double dg, double of) {
  const int m = L - 1 + lo + hi;
  for (int j = 0; j < m; ++j) {
    const int p = j + 1 - lo;
    double d = (p >= 1 ? dg * c[p - 1] : 0.0) + (p <= L - 1 ? dg * c[p] : 0.0);
    double pv = d - ((j > 0) ? of * c[p - 1] * cp[j - 1] : 0.0);  // T[j][j-1] = of c_{p-1}
    const double rp = 1.0 / pv;
    piv[j] = rp;
    cp[j] = (j + 1 < m) ? of * c[p] * rp : 0.0;
  }
}

// Solve T x = r in place with a factored line.
__device__ __forceinline__ void line_solve(const double* c, int L, int lo, int hi, const double* cp,
                                           const double* piv, double* r, double of) {
  const int m = L - 1 + lo + hi;
  for (int j = 0; j < m; ++j) r[j] = (r[j] - ((j > 0) ? of * c[j - lo] * r[j - 1] : 0.0)) * piv[j];
  for (int j = m - 2; j >= 0; --j) r[j] -= cp[j] * r[j + 1];
}

// The same solve from the factor alone (T symmetric: T[j][j-1] = cp[j-1] / piv[j-1]):
// z_j = r_j - cp[j-1] z_{j-1}, y_j = z_j piv_j, x_j = y_j - cp_j x_{j+1}.  cp / piv may
// live in shared memory (factor kept from an earlier phase), element stride 1.
__device__ __forceinline__ void line_solve_sym(int m, const double* cp, const double* piv, double* r) {
  double z = 0.0;
  for (int j = 0; j < m; ++j) {
    z = r[j] - ((j > 0) ? cp[j - 1] * z : 0.0);
    r[j] = z * piv[j];
  }
  for (int j = m - 2; j >= 0; --j) r[j] -= cp[j] * r[j + 1];
}

__global__ void cell_coeff_kernel(bddc_geom G, const double* __restrict__ k, double* __restrict__ coef) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= G.n_cells) return;
  for (int a = 0; a < 3; ++a) {
    double v = 0.0;
    if (a < G.dim) v = G.h[a] * G.h[a] / (6.0 * G.vol) / k[(size_t)c * G.dim + a];
    coef[(size_t)(a) * G.n_cells + (c)] = v;
  }
}

// delta per slot: 0.5 (multiplicity) or d_own/(d_own+d_other) with
// d = h^2/(3 V k) = 2 c (stiffness, decomposition.py:212-239).
__global__ void weights_kernel(bddc_geom G, int stiffness, const double* __restrict__ coef,
                               const int* __restrict__ gcode, double* __restrict__ delta) {
  int i = blockIdx.x;
  Box b = sub_box(G, i);
  for (int q = threadIdx.x; q < G.maxG; q += blockDim.x) {
    int code = gcode[(size_t)i * G.maxG + q];
    double w = 0.0;
    if (code >= 0) {
      w = 0.5;
      if (stiffness) {
        SlotLine s = decode_slot(b, code);
        int k_own = s.side ? s.L - 1 : 0;
        int own = line_cell_global(G, b, s.a, s.line, k_own);
        int stride_g = s.a == 0 ? 1 : (s.a == 1 ? G.n[0] : G.n[0] * G.n[1]);
        int oth = s.side ? own + stride_g : own - stride_g;
        double d_own = 2.0 * coef[(size_t)(s.a) * G.n_cells + (own)];
        double d_oth = 2.0 * coef[(size_t)(s.a) * G.n_cells + (oth)];
        w = d_own / (d_own + d_oth);
      }
    }
    delta[(size_t)i * G.maxG + q] = w;
  }
}

// D_i = mean of diag(A) over the interior dofs on faces of subdomain i
// (grid.py:344-357).  diag(A) at a dof = 2 c_lo + 2 c_hi (both neighbours).
__global__ void rescale_kernel(bddc_geom G, const double* __restrict__ coef, double* __restrict__ Dsub) {
  __shared__ double red[32];
  int i = blockIdx.x;
  Box b = sub_box(G, i);
  double acc = 0.0;
  int cnt = 0;
  for (int a = 0; a < G.dim; ++a) {
    int nl = n_lines(b, a);
    int L = b.L[a];
    int nf = (L + 1) * nl;  // faces j = 0..L along every line
    int stride_g = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
    for (int e = threadIdx.x; e < nf; e += blockDim.x) {
      int line = e / (L + 1), j = e % (L + 1);
      int fc = b.o[a] + j;  // global face coordinate along a
      const bool dir = (a == G.dir_axis);  // mode B: the boundary faces are dofs too
      if (!dir && (fc < 1 || fc > G.n[a] - 1)) continue;
      int c[3];
      line_coords(b, a, line, c);
      int gc[3] = {b.o[0] + c[0], b.o[1] + c[1], b.o[2] + c[2]};
      gc[a] = fc;  // the cell above the face
      int hi = cell_id(G, gc[0], gc[1], gc[2]);
      int lo = hi - stride_g;
      if (fc <= G.n[a] - 1) acc += G.a_diag * coef[(size_t)(a) * G.n_cells + (hi)];
      if (fc >= 1) acc += G.a_diag * coef[(size_t)(a) * G.n_cells + (lo)];
      cnt += 1;
    }
  }
  double tot = block_sum(acc, red);
  double cn = block_sum((double)cnt, red);
  if (threadIdx.x == 0) Dsub[i] = tot / cn;
}

// Build P (+alpha 11^T, identity padding), line-compact G and S_A.
// Gc layout: [i][q][k] (maxG x maxL per subdomain).
__global__ void local_build_kernel(bddc_geom G, const double* __restrict__ coef, const int* __restrict__ fslot,
                                   double* __restrict__ P, double* __restrict__ Gc, double* __restrict__ SAd,
                                   int* __restrict__ SApart, double* __restrict__ SAoff, double* __restrict__ scl) {
  __shared__ double red[32];
  const int i = blockIdx.x;
  const Box b = sub_box(G, i);
  const int np = b.L[0] * b.L[1] * b.L[2];
  const int mp = G.maxP;
  double* Pi = P + (size_t)i * mp * mp;
  for (size_t e = threadIdx.x; e < (size_t)mp * mp; e += blockDim.x) Pi[e] = 0.0;
  for (size_t e = threadIdx.x; e < (size_t)G.maxG * G.maxL; e += blockDim.x) Gc[(size_t)i * G.maxG * G.maxL + e] = 0.0;
  for (int q = threadIdx.x; q < G.maxG; q += blockDim.x) {
    SAd[(size_t)i * G.maxG + q] = 1.0;
    SApart[(size_t)i * G.maxG + q] = -1;
    SAoff[(size_t)i * G.maxG + q] = 0.0;
  }
  __syncthreads();
  for (int a = 0; a < G.dim; ++a) {
    const int L = b.L[a];
    const int nl = n_lines(b, a);
    const int st = axis_stride(b, a);
    const bool has_lo = b.o[a] > 0, has_hi = b.o[a] + L < G.n[a];
    int lo, hi;
    line_open(G, b, a, lo, hi);
    for (int line = threadIdx.x; line < nl; line += blockDim.x) {
      double c[MAXL], cp[MAXL + 1], piv[MAXL + 1], col[MAXL + 1], colp[MAXL + 1];
      for (int k = 0; k < L; ++k) c[k] = coef[(size_t)(a) * G.n_cells + (line_cell_global(G, b, a, line, k))];
      const int base = line_base(b, a, line);
      const int m = L - 1 + lo + hi;
      if (m > 0) line_factor(c, L, lo, hi, cp, piv, G.a_diag, G.a_off);
      // P_line = B Ainv B^T with B[k][k-1+lo] = +1 (low face), B[k][k+lo] = -1:
      // walk the cells kq, keeping the Ainv columns of kq's low face (colp) and
      // high face (col); the high face of kq is the low face of kq+1.
      for (int j = 0; j < m; ++j) colp[j] = (lo && j == 0) ? 1.0 : 0.0;
      if (lo) line_solve(c, L, lo, hi, cp, piv, colp, G.a_off);
      for (int kq = 0; kq < L; ++kq) {
        const int jh = kq + lo;
        for (int j = 0; j < m; ++j) col[j] = (j == jh) ? 1.0 : 0.0;
        if (jh < m) line_solve(c, L, lo, hi, cp, piv, col, G.a_off);
        for (int k = 0; k < L; ++k) {
          const int kl = k - 1 + lo, kh = k + lo;
          double v = 0.0;
          if (kl >= 0) v += colp[kl] - col[kl];
          if (kh < m) v += -colp[kh] + col[kh];
          if (v != 0.0) Pi[(size_t)(base + k * st) * mp + base + kq * st] += v;
        }
        for (int j = 0; j < m; ++j) colp[j] = col[j];
      }
      // Ainv corner entries for the interface ends (Gamma ends are never Dirichlet ends)
      double a00 = 0.0, aEE = 0.0, a0E = 0.0;
      if (m > 0 && (has_lo || has_hi)) {
        for (int j = 0; j < m; ++j) col[j] = (j == 0) ? 1.0 : 0.0;
        line_solve(c, L, lo, hi, cp, piv, col, G.a_off);
        a00 = col[0];
        a0E = col[m - 1];
        for (int j = 0; j < m; ++j) col[j] = (j == m - 1) ? 1.0 : 0.0;
        line_solve(c, L, lo, hi, cp, piv, col, G.a_off);
        aEE = col[m - 1];
      }
      // interface slots at the two ends of the line
      for (int side = 0; side < 2; ++side) {
        if (side == 0 && !has_lo) continue;
        if (side == 1 && !has_hi) continue;
        int q = fslot[((size_t)i * 6 + a * 2 + side) * G.maxF + line];
        double* g = Gc + ((size_t)i * G.maxG + q) * G.maxL;
        int kend = side ? L - 1 : 0;
        double cend = c[kend];
        // v = Ainv * (c_end e_jend), jend = 0 (low) or m-1 (high)
        for (int k = 0; k < L; ++k) g[k] = 0.0;
        g[kend] = side ? -1.0 : 1.0;
        if (m > 0) {
          int jend = side ? m - 1 : 0;
          for (int j = 0; j < m; ++j) col[j] = (j == jend) ? G.a_off * cend : 0.0;
          line_solve(c, L, lo, hi, cp, piv, col, G.a_off);
          for (int k = 0; k < L; ++k) {
            const int kl = k - 1 + lo, kh = k + lo;
            double bv = 0.0;
            if (kl >= 0) bv += col[kl];
            if (kh < m) bv -= col[kh];
            g[k] -= bv;
          }
        }
        double d = G.a_diag * cend;
        if (m > 0) d -= G.a_off * G.a_off * cend * cend * (side ? aEE : a00);
        SAd[(size_t)i * G.maxG + q] = d;
        int other = side ? 0 : 1;
        bool has_other = other ? has_hi : has_lo;
        if (has_other) {
          int q2 = fslot[((size_t)i * 6 + a * 2 + other) * G.maxF + line];
          SApart[(size_t)i * G.maxG + q] = q2;
          SAoff[(size_t)i * G.maxG + q] =
              (m > 0) ? -G.a_off * G.a_off * c[0] * c[L - 1] * a0E : G.a_off * c[0];
        }
      }
    }
    __syncthreads();
  }
  // Jacobi scaling + rank-one regularisation of the null space (P 1 = 0):
  //   Ps = D^-1/2 P D^-1/2 + v v^T,  D = diag(P),  v = D^1/2 1 / |D^1/2 1|.
  // Scaling removes the coefficient-contrast part of cond(P) (1e7 -> 1e3 on
  // 6-decade fields), which keeps S_i accurate to ~1e-15.  scl = [dsq (maxP) | |D^1/2 1|].
  // Mode B subdomains touching a Dirichlet end have a nonsingular P: no v v^T,
  // and the stored norm is 0 (pinv_fix then inverts without projecting).
  const bool flt = sub_floating(G, b);
  double* dsq = scl + (size_t)i * (mp + 1);
  double sd = 0.0;
  for (int r = threadIdx.x; r < np; r += blockDim.x) {
    double dr = Pi[(size_t)r * mp + r];
    if (!(dr > 0.0)) dr = 1.0;
    dsq[r] = rsqrt(dr);
    sd += dr;
  }
  sd = block_sum(sd, red);
  const double vn = sqrt(sd);
  if (threadIdx.x == 0) dsq[mp] = flt ? vn : 0.0;
  __syncthreads();
  for (size_t e = threadIdx.x; e < (size_t)mp * mp; e += blockDim.x) {
    int r = (int)(e / mp), cc = (int)(e % mp);
    if (r < np && cc < np) {
      const double vr = 1.0 / (dsq[r] * vn), vc = 1.0 / (dsq[cc] * vn);
      Pi[e] = Pi[e] * dsq[r] * dsq[cc] + (flt ? vr * vc : 0.0);
    } else {
      Pi[e] = (r == cc) ? 1.0 : 0.0;
    }
  }
}

// Q = P^+ = Pi D^-1/2 (Ps^-1 - v v^T) D^-1/2 Pi,  Pi = I - 11^T/np (zero padding).
__global__ void pinv_fix_kernel(bddc_geom G, double* __restrict__ P, const double* __restrict__ scl) {
  extern __shared__ double rm[];   // maxP column means, then dsq and 1/(dsq vn)
  __shared__ double red[32];
  const int i = blockIdx.x;
  const Box b = sub_box(G, i);
  const int np = b.L[0] * b.L[1] * b.L[2];
  const int mp = G.maxP;
  const double* dsq = scl + (size_t)i * (mp + 1);
  const double vn = dsq[mp];
  double* Pi = P + (size_t)i * mp * mp;
  if (vn == 0.0) {  // mode B, not floating: Q = P^-1 = D^-1/2 Ps^-1 D^-1/2
    for (size_t e = threadIdx.x; e < (size_t)mp * mp; e += blockDim.x) {
      int r = (int)(e / mp), c = (int)(e % mp);
      Pi[e] = (r < np && c < np) ? dsq[r] * Pi[e] * dsq[c] : 0.0;
    }
    return;
  }
  // per-row factors once (no division in the sweeps), column sums with four
  // independent partial sums (loads in flight), coalesced over columns
  double* sd = rm + mp;   // dsq
  double* wv = sd + mp;   // 1 / (dsq vn)
  for (int r = threadIdx.x; r < np; r += blockDim.x) {
    sd[r] = dsq[r];
    wv[r] = 1.0 / (dsq[r] * vn);
  }
  __syncthreads();
  double part = 0.0;
  for (int c = threadIdx.x; c < np; c += blockDim.x) {
    const double vc = wv[c];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int r = 0;
    for (; r + 4 <= np; r += 4) {
      a0 += sd[r] * (Pi[(size_t)r * mp + c] - wv[r] * vc);
      a1 += sd[r + 1] * (Pi[(size_t)(r + 1) * mp + c] - wv[r + 1] * vc);
      a2 += sd[r + 2] * (Pi[(size_t)(r + 2) * mp + c] - wv[r + 2] * vc);
      a3 += sd[r + 3] * (Pi[(size_t)(r + 3) * mp + c] - wv[r + 3] * vc);
    }
    for (; r < np; ++r) a0 += sd[r] * (Pi[(size_t)r * mp + c] - wv[r] * vc);
    const double acc = ((a0 + a1) + (a2 + a3)) * sd[c];
    rm[c] = acc / np;
    part += acc;
  }
  const double tm = block_sum(part, red) / ((double)np * np);
  __syncthreads();
  for (size_t e = threadIdx.x; e < (size_t)mp * mp; e += blockDim.x) {
    int r = (int)(e / mp), c = (int)(e % mp);
    double v = 0.0;
    if (r < np && c < np) v = sd[r] * (Pi[e] - wv[r] * wv[c]) * sd[c] - rm[r] - rm[c] + tm;
    Pi[e] = v;
  }
}

// Wt[i][q][r] = sum_k Q[cell(q,k)][r] * Gc[q][k]   (W = Q G, stored transposed)
__global__ void schur_w_kernel(bddc_geom G, const int* __restrict__ gcode, const double* __restrict__ Q,
                               const double* __restrict__ Gc, double* __restrict__ Wt, int qchunk) {
  const int i = blockIdx.y;
  const Box b = sub_box(G, i);
  const int mp = G.maxP;
  const double* Qi = Q + (size_t)i * mp * mp;
  const int q0 = blockIdx.x * qchunk;
  for (int q = q0; q < imin(q0 + qchunk, G.maxG); ++q) {
    int code = gcode[(size_t)i * G.maxG + q];
    double* w = Wt + ((size_t)i * G.maxG + q) * mp;
    if (code < 0) {
      for (int r = threadIdx.x; r < mp; r += blockDim.x) w[r] = 0.0;
      continue;
    }
    SlotLine s = decode_slot(b, code);
    const double* g = Gc + ((size_t)i * G.maxG + q) * G.maxL;
    for (int r = threadIdx.x; r < mp; r += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < s.L; ++k) acc += Qi[(size_t)(s.base + k * s.stride) * mp + r] * g[k];
      w[r] = acc;
    }
  }
}

// S[i][q][q'] = S_A[q][q'] + sum_k Gc[q'][k] Wt[q][cell(q',k)]
__global__ void schur_s_kernel(bddc_geom G, const int* __restrict__ gcode, const double* __restrict__ Gc,
                               const double* __restrict__ Wt, const double* __restrict__ SAd,
                               const int* __restrict__ SApart, const double* __restrict__ SAoff,
                               double* __restrict__ S, int qchunk) {
  extern __shared__ double wrow[];
  const int i = blockIdx.y;
  const Box b = sub_box(G, i);
  const int mp = G.maxP, mg = G.maxG;
  const int q0 = blockIdx.x * qchunk;
  for (int q = q0; q < imin(q0 + qchunk, mg); ++q) {
    __syncthreads();
    for (int r = threadIdx.x; r < mp; r += blockDim.x) wrow[r] = Wt[((size_t)i * mg + q) * mp + r];
    __syncthreads();
    int codeq = gcode[(size_t)i * mg + q];
    int partner = SApart[(size_t)i * mg + q];
    for (int q2 = threadIdx.x; q2 < mg; q2 += blockDim.x) {
      int code = gcode[(size_t)i * mg + q2];
      double v;
      if (codeq < 0 || code < 0) {
        v = (q == q2) ? 1.0 : 0.0;
      } else {
        SlotLine s = decode_slot(b, code);
        const double* g = Gc + ((size_t)i * mg + q2) * G.maxL;
        double acc = 0.0;
        for (int k = 0; k < s.L; ++k) acc += g[k] * wrow[s.base + k * s.stride];
        if (q2 == q) acc += SAd[(size_t)i * mg + q];
        if (q2 == partner) acc += SAoff[(size_t)i * mg + q];
        v = acc;
      }
      S[((size_t)i * mg + q) * mg + q2] = v;
    }
  }
}

// S <- (S + S^T)/2 (substructure.py:99), tile-wise through shared memory.
__global__ void symmetrize_kernel(double* __restrict__ S, int n, long long stride) {
  __shared__ double t1[32][33], t2[32][33];
  const int i = blockIdx.z;
  const int bx = blockIdx.x, by = blockIdx.y;
  if (by > bx) return;
  double* Si = S + i * stride;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    int gr = by * 32 + r, gc = bx * 32 + tx;
    t1[r][tx] = (gr < n && gc < n) ? Si[(size_t)gr * n + gc] : 0.0;
    int gr2 = bx * 32 + r, gc2 = by * 32 + tx;
    t2[r][tx] = (gr2 < n && gc2 < n) ? Si[(size_t)gr2 * n + gc2] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    int gr = by * 32 + r, gc = bx * 32 + tx;
    double v = 0.5 * (t1[r][tx] + t2[tx][r]);
    if (gr < n && gc < n) Si[(size_t)gr * n + gc] = v;
    int gr2 = bx * 32 + r, gc2 = by * 32 + tx;
    double v2 = 0.5 * (t2[r][tx] + t1[tx][r]);
    if (gr2 < n && gc2 < n) Si[(size_t)gr2 * n + gc2] = v2;
  }
}

// Batched interior solve, one CTA per subdomain (see bddc.h).  With
// B_loc = D B_u (grid.py:250):  p' = Q (B_u A^{-1} f - g/D),
// u_I = A^{-1}(f - B_u^T p'), p = p'/D  where f = f_flux - A_IG x and
// g = g_cell - D B_uG x (substructure.py:72-116).
#ifndef LS_CTAS
#define LS_CTAS 2
#endif
#ifdef LS_TIMING
__device__ unsigned long long g_ls_t[8];
#define LS_T(k)                                                                  \
  do {                                                                           \
    __syncthreads();                                                             \
    if (threadIdx.x == 0) {                                                      \
      long long t_ = clock64();                                                  \
      atomicAdd(&g_ls_t[k], (unsigned long long)(t_ - t0_));                     \
      t0_ = t_;                                                                  \
    }                                                                            \
  } while (0)
#else
#define LS_T(k)
#endif
template <bool TWO>
__global__ void __launch_bounds__(256, LS_CTAS) local_solve_kernel(bddc_geom G, const double* __restrict__ coef, const int* __restrict__ gcode,
                                   const int* __restrict__ gpos, const int* __restrict__ fslot,
                                   const double* __restrict__ Q, const double* __restrict__ Dsub,
                                   bddc_local_solve_args A, int stash) {
  extern __shared__ double sm[];
  const int i = blockIdx.x;
  const Box b = sub_box(G, i);
  const int np = b.L[0] * b.L[1] * b.L[2];
  const int mp = G.maxP, mg = G.maxG;
  double* xg = sm;            // mg
  double* rhs = xg + mg;      // mp
  double* pp = rhs + mp;      // mp
  double* tI = pp + mp;       // 3 mp + 2 maxF (interior faces, per axis blocks)
  double* yw = tI + 3 * mp + 2 * G.maxF;   // (blockDim/32) x mp symv partials (x2 with two rhs)
  constexpr bool two = TWO;
  double* rhs2 = yw + (two ? 16 : 8) * mp;   // second right-hand side (two only)
  double* pp2 = rhs2 + mp;
  // line factors kept from the first line phase for the second (when they fit)
  double* sCp = (two ? pp2 + mp : rhs2);
  double* sRp = sCp + 3 * mp + 2 * G.maxF;
  int off[3], lo3[3] = {0, 0, 0}, hi3[3] = {0, 0, 0};
  {
    int o = 0;
    for (int a = 0; a < 3; ++a) {
      off[a] = o;
      if (a < G.dim) {
        line_open(G, b, a, lo3[a], hi3[a]);
        o += (b.L[a] - 1 + lo3[a] + hi3[a]) * n_lines(b, a);
      }
    }
  }
  const double Di = Dsub[i];
#ifdef LS_TIMING
  long long t0_ = clock64();
#endif
  for (int q = threadIdx.x; q < mg; q += blockDim.x) {
    int gp = gpos[(size_t)i * mg + q];
    xg[q] = (A.x_gamma && gp >= 0) ? A.x_scale * A.x_gamma[gp] : 0.0;
  }
  for (int c = threadIdx.x; c < mp; c += blockDim.x) {
    double v = 0.0;
    if (c < np && A.g_cell) {
      int lx = c % b.L[0], ly = (c / b.L[0]) % b.L[1], lz = c / (b.L[0] * b.L[1]);
      v = A.g_scale * A.g_cell[cell_id(G, b.o[0] + lx, b.o[1] + ly, b.o[2] + lz)] / Di;
    }
    rhs[c] = -v;
  }
  __syncthreads();
  // rhs += B_uG x, one (axis, side) at a time (corner cells are shared)
  if (A.x_gamma) {
    for (int a = 0; a < G.dim; ++a) {
      const int nl = n_lines(b, a), L = b.L[a], st = axis_stride(b, a);
      for (int side = 0; side < 2; ++side) {
        for (int line = threadIdx.x; line < nl; line += blockDim.x) {
          int q = fslot[((size_t)i * 6 + a * 2 + side) * G.maxF + line];
          if (q < 0) continue;
          int cell = line_base(b, a, line) + (side ? (L - 1) * st : 0);
          rhs[cell] += side ? -xg[q] : xg[q];
        }
        __syncthreads();
      }
    }
  }
  // t = A^{-1}(f - A_IG x) per line, the lines of all axes at once (thread per
  // line); rhs += B_u t through per-axis buffers (lines of one axis are
  // cell-disjoint, different axes are not), summed after the barrier
  LS_T(0);
  int nla[3] = {0, 0, 0};
  for (int a = 0; a < G.dim; ++a) nla[a] = n_lines(b, a);
  double* radd = yw;   // 3 x mp, free until the symv
  for (int c = threadIdx.x; c < 3 * mp; c += blockDim.x) radd[c] = 0.0;
  __syncthreads();
  if (stash) {
    // every operand of the line phase staged in shared memory by the whole CTA
    // (coalesced, all loads in flight at once): the per-axis coefficients of the
    // box and the flux load; the factor / forward / backward sweeps then run out of
    // shared memory and registers (no per-thread local arrays)
    double* cs = yw + 3 * mp;   // 3 x mp, free until the symv
    for (int a = 0; a < G.dim; ++a)
      for (int c = threadIdx.x; c < np; c += blockDim.x) {
        const int lx = c % b.L[0], ly = (c / b.L[0]) % b.L[1], lz = c / (b.L[0] * b.L[1]);
        cs[a * mp + c] = coef[(size_t)a * G.n_cells + cell_id(G, b.o[0] + lx, b.o[1] + ly, b.o[2] + lz)];
      }
    for (int a = 0; a < G.dim; ++a) {
      const int m = b.L[a] - 1 + lo3[a] + hi3[a];
      if (m <= 0) continue;
      const int tot = nla[a] * m;
      for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int line = e / m, j = e - line * m;
        tI[off[a] + e] = A.f_flux ? A.f_scale * A.f_flux[line_face_dof(G, b, a, line, j, lo3[a])] : 0.0;
      }
    }
    __syncthreads();
    const double dg = G.a_diag, of = G.a_off;
    for (int gl = threadIdx.x; gl < nla[0] + nla[1] + nla[2]; gl += blockDim.x) {
      const int a = gl < nla[0] ? 0 : (gl < nla[0] + nla[1] ? 1 : 2);
      const int line = gl - (a > 0 ? nla[0] : 0) - (a > 1 ? nla[1] : 0);
      const int L = b.L[a], lo = lo3[a], hi = hi3[a], m = L - 1 + lo + hi, st = axis_stride(b, a);
      if (m <= 0) continue;
      const int base = line_base(b, a, line);
      const double* cl = cs + a * mp + base;   // c[k] = cl[k st]
      double* t = tI + off[a] + line * m;
      double* scp = sCp + off[a] + line * m;
      double* srp = sRp + off[a] + line * m;
      if (A.x_gamma) {
        const int qlo = fslot[((size_t)i * 6 + a * 2 + 0) * G.maxF + line];
        const int qhi = fslot[((size_t)i * 6 + a * 2 + 1) * G.maxF + line];
        if (qlo >= 0) t[0] -= of * cl[0] * xg[qlo];
        if (qhi >= 0) t[m - 1] -= of * cl[(L - 1) * st] * xg[qhi];
      }
      double cpp = 0.0, rprev = 0.0;
      for (int j = 0; j < m; ++j) {   // Thomas factor and forward sweep (see line_factor)
        const int p = j + 1 - lo;
        const double c_lo = p >= 1 ? cl[(p - 1) * st] : 0.0;
        const double c_hi = p <= L - 1 ? cl[p * st] : 0.0;
        const double pv = (dg * c_lo + dg * c_hi) - of * c_lo * cpp;
        const double rp = 1.0 / pv;
        cpp = (j + 1 < m) ? of * c_hi * rp : 0.0;
        rprev = (t[j] - of * c_lo * rprev) * rp;
        scp[j] = cpp;
        srp[j] = rp;
        t[j] = rprev;
      }
      for (int j = m - 2; j >= 0; --j) {
        rprev = t[j] - scp[j] * rprev;
        t[j] = rprev;
      }
      double* ra = radd + a * mp;
      for (int k = 0; k < L; ++k) {
        double v = 0.0;
        if (k - 1 + lo >= 0) v += t[k - 1 + lo];
        if (k + lo < m) v -= t[k + lo];
        ra[base + k * st] = v;
      }
    }
  } else {
    for (int gl = threadIdx.x; gl < nla[0] + nla[1] + nla[2]; gl += blockDim.x) {
      const int a = gl < nla[0] ? 0 : (gl < nla[0] + nla[1] ? 1 : 2);
      const int line = gl - (a > 0 ? nla[0] : 0) - (a > 1 ? nla[1] : 0);
      const int L = b.L[a], lo = lo3[a], hi = hi3[a], m = L - 1 + lo + hi, st = axis_stride(b, a);
      if (m <= 0) continue;
      double c[MAXL], cp[MAXL + 1], piv[MAXL + 1], r[MAXL + 1];
      for (int k = 0; k < L; ++k) c[k] = coef[(size_t)(a) * G.n_cells + (line_cell_global(G, b, a, line, k))];
      line_factor(c, L, lo, hi, cp, piv, G.a_diag, G.a_off);
      for (int j = 0; j < m; ++j)
        r[j] = A.f_flux ? A.f_scale * A.f_flux[line_face_dof(G, b, a, line, j, lo)] : 0.0;
      if (A.x_gamma) {
        int qlo = fslot[((size_t)i * 6 + a * 2 + 0) * G.maxF + line];
        int qhi = fslot[((size_t)i * 6 + a * 2 + 1) * G.maxF + line];
        if (qlo >= 0) r[0] -= G.a_off * c[0] * xg[qlo];
        if (qhi >= 0) r[m - 1] -= G.a_off * c[L - 1] * xg[qhi];
      }
      line_solve(c, L, lo, hi, cp, piv, r, G.a_off);
      double* t = tI + off[a] + line * m;
      const int base = line_base(b, a, line);
      double* ra = radd + a * mp;
      for (int j = 0; j < m; ++j) t[j] = r[j];
      for (int k = 0; k < L; ++k) {
        double v = 0.0;
        if (k - 1 + lo >= 0) v += r[k - 1 + lo];
        if (k + lo < m) v -= r[k + lo];
        ra[base + k * st] = v;
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < mp; c += blockDim.x) {
    const double v = (radd[c] + radd[mp + c]) + radd[2 * mp + c];
    if (two) {
      double g2 = 0.0;
      if (c < np && A.g_cell2) {
        int lx = c % b.L[0], ly = (c / b.L[0]) % b.L[1], lz = c / (b.L[0] * b.L[1]);
        g2 = A.g_scale2 * A.g_cell2[cell_id(G, b.o[0] + lx, b.o[1] + ly, b.o[2] + lz)] / Di;
      }
      // the second system differs from the first only in its cell load
      rhs2[c] = rhs[c] + v - g2;
    }
    rhs[c] += v;
  }
  __syncthreads();
  LS_T(1);
  // p' = Q rhs, Q tile-packed symmetric (half the bytes of full storage)
  {
    const int nt = mp / 32, ntl = (np + 31) / 32;
    const double* Qi = Q + (size_t)i * (nt * (nt + 1) / 2) * 1024;
    if (two) cta_symv_packed2(Qi, nt, ntl, rhs, rhs2, pp, pp2, yw);
    else cta_symv_packed(Qi, nt, ntl, rhs, pp, yw);
    for (int r = ntl * 32 + threadIdx.x; r < mp; r += blockDim.x) {
      pp[r] = 0.0;
      if (two) pp2[r] = 0.0;
    }
    __syncthreads();
  }
  LS_T(2);
  // u_I = t - A^{-1} B_u^T p' (lines of all axes at once: disjoint outputs)
  for (int gl = threadIdx.x; gl < nla[0] + nla[1] + nla[2]; gl += blockDim.x) {
    const int a = gl < nla[0] ? 0 : (gl < nla[0] + nla[1] ? 1 : 2);
    const int line = gl - (a > 0 ? nla[0] : 0) - (a > 1 ? nla[1] : 0);
    const int L = b.L[a], lo = lo3[a], hi = hi3[a], m = L - 1 + lo + hi, st = axis_stride(b, a);
    {
      if (m <= 0) continue;
      double cpl[MAXL + 1], pivl[MAXL + 1], r[MAXL + 1];
      const double* cp = sCp + off[a] + line * m;
      const double* piv = sRp + off[a] + line * m;
      if (!stash) {
        double c[MAXL];
        for (int k = 0; k < L; ++k) c[k] = coef[(size_t)(a) * G.n_cells + (line_cell_global(G, b, a, line, k))];
        line_factor(c, L, lo, hi, cpl, pivl, G.a_diag, G.a_off);
        cp = cpl;
        piv = pivl;
      }
      const int base = line_base(b, a, line);
      double* t = tI + off[a] + line * m;
      if (two) {   // second system first: t is still the shared A^{-1} f
        for (int j = 0; j < m; ++j) {
          const int p = j + 1 - lo;
          r[j] = (p <= L - 1 ? pp2[base + p * st] : 0.0) - (p >= 1 ? pp2[base + (p - 1) * st] : 0.0);
        }
        line_solve_sym(m, cp, piv, r);
        for (int j = 0; j < m; ++j)
          A.u_out2[(size_t)line_face_dof(G, b, a, line, j, lo)] = t[j] - r[j];
      }
      for (int j = 0; j < m; ++j) {
        const int p = j + 1 - lo;  // (B_u^T p')_j = p'(cell above) - p'(cell below)
        r[j] = (p <= L - 1 ? pp[base + p * st] : 0.0) - (p >= 1 ? pp[base + (p - 1) * st] : 0.0);
      }
      line_solve_sym(m, cp, piv, r);
      for (int j = 0; j < m; ++j) {
        double u = t[j] - r[j];
        t[j] = u;
        if (A.u_out) {
          size_t d = (size_t)line_face_dof(G, b, a, line, j, lo);
          if (A.u_mode) A.u_out[d] += u;
          else A.u_out[d] = u;
        }
      }
    }
  }
  __syncthreads();
  LS_T(3);
  if (A.p_out) {
    for (int c = threadIdx.x; c < np; c += blockDim.x) {
      int lx = c % b.L[0], ly = (c / b.L[0]) % b.L[1], lz = c / (b.L[0] * b.L[1]);
      A.p_out[cell_id(G, b.o[0] + lx, b.o[1] + ly, b.o[2] + lz)] = pp[c] / Di;
    }
  }
  if (A.rg_broken) {
    for (int q = threadIdx.x; q < mg; q += blockDim.x) {
      int code = gcode[(size_t)i * mg + q];
      double v = 0.0;
      if (code >= 0) {
        SlotLine s = decode_slot(b, code);
        int m = s.L - 1 + lo3[s.a] + hi3[s.a];
        int kend = s.side ? s.L - 1 : 0;
        if (m > 0) {
          double cend = coef[(size_t)(s.a) * G.n_cells + (line_cell_global(G, b, s.a, s.line, kend))];
          int jend = s.side ? m - 1 : 0;
          v += G.a_off * cend * tI[off[s.a] + s.line * m + jend];
        }
        double pc = pp[s.base + kend * s.stride];
        v += s.side ? -pc : pc;
      }
      A.rg_broken[(size_t)i * mg + q] = v;
    }
  }
  LS_T(4);
}

}  // namespace

extern "C" int bddc_cell_coeffs(const bddc_geom* g, const double* k, double* coef, void* stream) {
  cell_coeff_kernel<<<(g->n_cells + 255) / 256, 256, 0, (cudaStream_t)stream>>>(*g, k, coef);
  LAUNCH_OK();
  return 0;
}

#ifdef LS_TIMING
extern "C" int bddc_ls_timing_read(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_ls_t, sizeof(g_ls_t));
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_ls_t, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" int bddc_weights(const bddc_geom* g, int stiffness, const double* coef, const int* gcode, double* delta,
                            void* stream) {
  weights_kernel<<<g->N, 128, 0, (cudaStream_t)stream>>>(*g, stiffness, coef, gcode, delta);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_rescale(const bddc_geom* g, const double* coef, double* Dsub, void* stream) {
  rescale_kernel<<<g->N, 256, 0, (cudaStream_t)stream>>>(*g, coef, Dsub);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_local_build(const bddc_geom* g, const double* coef, const int* fslot, double* P, double* Gc,
                                double* SAd, int* SApart, double* SAoff, double* scl, void* stream) {
  if (g->maxL > MAXL) return bddc_set_error(BDDC_ERR_ARG, "subdomain strip wider than MAXL=32 cells");
  local_build_kernel<<<g->N, 128, 0, (cudaStream_t)stream>>>(*g, coef, fslot, P, Gc, SAd, SApart, SAoff, scl);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_local_pinv_fix(const bddc_geom* g, double* P, const double* scl, void* stream) {
  pinv_fix_kernel<<<g->N, 512, 3 * g->maxP * sizeof(double), (cudaStream_t)stream>>>(*g, P, scl);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_local_schur(const bddc_geom* g, const int* gcode, const double* Q, const double* Gc,
                                const double* SAd, const int* SApart, const double* SAoff, double* Wt, double* S,
                                void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int qchunk = 8;
  dim3 gw((g->maxG + qchunk - 1) / qchunk, g->N);
  schur_w_kernel<<<gw, 256, 0, s>>>(*g, gcode, Q, Gc, Wt, qchunk);
  LAUNCH_OK();
  size_t shm = (size_t)g->maxP * sizeof(double);
  schur_s_kernel<<<gw, 256, shm, s>>>(*g, gcode, Gc, Wt, SAd, SApart, SAoff, S, qchunk);
  LAUNCH_OK();
  dim3 gs((g->maxG + 31) / 32, (g->maxG + 31) / 32, g->N);
  symmetrize_kernel<<<gs, dim3(32, 8), 0, s>>>(S, g->maxG, (long long)g->maxG * g->maxG);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_local_solve(const bddc_geom* g, const double* coef, const int* gcode, const int* gpos,
                                const int* fslot, const double* Q, const double* Dsub,
                                const bddc_local_solve_args* a, void* stream) {
  if (g->maxP % 32) return bddc_set_error(BDDC_ERR_ARG, "local_solve: maxP must be a multiple of 32");
  const bool two = a->u_out2 != nullptr;
  size_t shm = (size_t)(g->maxG + 5 * g->maxP + 2 * g->maxF + (two ? 18 : 8) * g->maxP) * sizeof(double);
  // the line factors of the first phase stay in shared memory for the second while
  // two CTAs still fit on an SM; larger subdomains refactor their lines
  const size_t shm_stash = shm + 2 * (size_t)(3 * g->maxP + 2 * g->maxF) * sizeof(double);
  const int stash = shm_stash <= 113 * 1024;
  if (stash) shm = shm_stash;
  if (shm > 227 * 1024) return bddc_set_error(BDDC_ERR_ARG, "local_solve: subdomain too large for shared memory");
  if (shm > 48 * 1024) {
    CUDA_OK(cudaFuncSetAttribute(local_solve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    CUDA_OK(cudaFuncSetAttribute(local_solve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  }
  if (two) local_solve_kernel<true><<<g->N, 256, shm, (cudaStream_t)stream>>>(*g, coef, gcode, gpos, fslot, Q, Dsub, *a, stash);
  else local_solve_kernel<false><<<g->N, 256, shm, (cudaStream_t)stream>>>(*g, coef, gcode, gpos, fslot, Q, Dsub, *a, stash);
  LAUNCH_OK();
  return 0;
}
