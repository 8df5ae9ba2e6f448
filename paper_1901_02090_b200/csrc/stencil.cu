// Matrix-free RT0/P0 operators on the structured grid and the fast pressure
// recovery (grid.py:270-341, solver.py:254-274, 337-342).
//
//  (A u)_d  = 2(c_lo + c_hi) u_d + c_lo u_{d-} + c_hi u_{d+}   (lines of axis a)
//  (B u)_c  = sum_a u_{low face} - u_{high face}                 (boundary faces = 0)
//  (B^T p)_d = p_hi - p_lo
// Pressure recovery solves the D-free Neumann problem B B^T p = B(-A u)
// (equivalent to the reference's pinned (Bs Bs^T) solve after unscaling and
// re-centring) by an orthonormal DCT-II eigenbasis: three mode products with
// dense cosine matrices on DMMA, a diagonal scale, and three more products.
// Mode B (G.dir_axis >= 0): the boundary faces of that axis are dofs numbered
// after the interior ones (bnd_dof), B B^T p = B(g - A u) has Dirichlet ends
// along it (a DST-I basis there) and no null space.
#include "common.cuh"

extern "C" int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha, const double* A,
                                  int lda, long long sA, const double* B, int ldb, long long sB, double beta,
                                  double* C, int ldc, long long sC, int batch, int upper, void* stream);

namespace {

__device__ __forceinline__ void decode_dof(const bddc_geom& G, int d, int& a, int f[3]) {
  a = (d >= G.fam_off[1]) + (d >= G.fam_off[2]);
  int r = d - G.fam_off[a];
  int e0 = G.n[0] - (a == 0), e1 = G.n[1] - (a == 1);
  f[0] = r % e0;
  f[1] = (r / e0) % e1;
  f[2] = r / (e0 * e1);
  f[a] += 1;  // face coordinate along a in 1..n_a-1
}

// Mode B boundary dof d >= n_flux_int -> end (side) and the adjacent cell's coordinates.
__device__ __forceinline__ void decode_bnd(const bddc_geom& G, int d, int& side, int gc[3]) {
  int r = d - G.n_flux_int;
  side = r >= G.n_bt;
  r -= side * G.n_bt;
  int t1, t2;
  trans_axes(G.dir_axis, t1, t2);
  gc[t1] = r % G.n[t1];
  gc[t2] = r / G.n[t1];
  gc[G.dir_axis] = side ? G.n[G.dir_axis] - 1 : 0;
}

// Row-structured operators: consecutive lanes touch consecutive dofs, cells and
// (structure-of-arrays) coefficients of one grid row.

// Row (f1, f2) of family a (interior faces, face coordinates): x-extent e0 and
// the first dof d0; false outside the family.
__device__ __forceinline__ bool fam_row(const bddc_geom& G, int a, int r1, int r2, int& e0, int f[3], int& d0) {
  e0 = G.n[0] - (a == 0);
  const int e1 = G.n[1] - (a == 1), e2 = (G.dim > 2) ? G.n[2] - (a == 2) : 1;
  if (r1 >= e1 || r2 >= e2) return false;
  f[0] = (a == 0);
  f[1] = r1 + (a == 1);
  f[2] = r2 + (a == 2);
  d0 = G.fam_off[a] + e0 * (r1 + e1 * r2);
  return true;
}

// Flat row index R over the families' rows (family a: (n1 - [a==1]) x (n2 - [a==2])
// rows, row-major in (r1, r2)); the launches are persistent-style grid-stride
// loops over rows (a few CTAs per SM, ~10 rows per thread row) instead of one
// short-lived CTA per four rows.
__device__ __forceinline__ void flat_row(const bddc_geom& G, int R, int& a, int& r1, int& r2) {
  for (a = 0; a < G.dim - 1; ++a) {
    const int e1 = G.n[1] - (a == 1), e2 = (G.dim > 2) ? G.n[2] - (a == 2) : 1;
    if (R < e1 * e2) break;
    R -= e1 * e2;
  }
  const int e1 = G.n[1] - (a == 1);
  r1 = R % e1;
  r2 = R / e1;
}

// Warp-per-row launches: a warp takes one grid row at a time (row parameters are
// warp-uniform: computed once per ~60 elements), its lanes cover x in steps of 32
// with SX elements per lane whose loads are all issued before any is used; warps
// stride over the rows of a grid that fills every SM (a few CTAs per SM).
constexpr int ST = 256, SX = 2, RW = 2;   // threads, x per lane, rows per warp pass

struct FluxRow {
  int a, e0, d0, st, h0, fx, fy, fz;
  bool lo_in, hi_in;
};

// row R of the flattened interior-face families
__device__ __forceinline__ FluxRow flux_row(const bddc_geom& G, int R) {
  FluxRow w;
  int r1, r2, a;
  flat_row(G, R, a, r1, r2);
  w.a = a;
  w.e0 = G.n[0] - (a == 0);
  const int e1 = G.n[1] - (a == 1);
  w.fx = (a == 0);
  w.fy = r1 + (a == 1);
  w.fz = r2 + (a == 2);
  w.d0 = G.fam_off[a] + w.e0 * (r1 + e1 * r2);
  w.st = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
  w.h0 = cell_id(G, w.fx, w.fy, w.fz);
  const int fa = a == 1 ? w.fy : w.fz, na = a == 1 ? G.n[1] : G.n[2];
  w.lo_in = a == 0 || fa > 1;
  w.hi_in = a == 0 || fa < na - 1;
  return w;
}

// y = alpha * A u + beta * y on the interior faces (dof stride along a inside
// family a equals the cell stride st; partners outside the family are predicated
// off or, in mode B, the Dirichlet face)
__global__ void __launch_bounds__(ST) flux_A_kernel(bddc_geom G, const double* __restrict__ coef,
                                                    const double* __restrict__ u, double alpha, double beta,
                                                    double* __restrict__ y, int nrows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * ST) >> 5;
  for (int R0 = ((blockIdx.x * ST + threadIdx.x) >> 5) * RW; R0 < nrows; R0 += nw * RW) {
    FluxRow r[RW];
    int emax = 0;
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      r[j] = flux_row(G, imin(R0 + j, nrows - 1));
      if (R0 + j >= nrows) r[j].e0 = 0;
      emax = imax(emax, r[j].e0);
    }
    for (int x0 = 0; x0 < emax; x0 += 32 * SX) {
      double clo[RW][SX], chi[RW][SX], u0[RW][SX], ul[RW][SX], uh[RW][SX];
      int dd[RW][SX];
#pragma unroll
      for (int j = 0; j < RW; ++j)
#pragma unroll
        for (int k = 0; k < SX; ++k) {
          const FluxRow& w = r[j];
          const int x = x0 + lane + 32 * k;
          const bool act = x < w.e0;
          const int d = w.d0 + x, hi = w.h0 + x;
          dd[j][k] = act ? d : -1;
          const bool l = w.a == 0 ? x > 0 : w.lo_in, h = w.a == 0 ? x < w.e0 - 1 : w.hi_in;
          int dl = l ? d - w.st : -1, dh = h ? d + w.st : -1;
          if (w.a == G.dir_axis && act && (!l || !h)) {
            const int g[3] = {w.fx + x, w.fy, w.fz};
            if (!l) dl = bnd_dof(G, 0, g);
            if (!h) dh = bnd_dof(G, 1, g);
          }
          const double* ca = coef + (size_t)w.a * G.n_cells;
          clo[j][k] = act ? __ldg(ca + hi - w.st) : 0.0;
          chi[j][k] = act ? __ldg(ca + hi) : 0.0;
          u0[j][k] = act ? __ldg(u + d) : 0.0;
          ul[j][k] = (act && dl >= 0) ? __ldg(u + dl) : 0.0;
          uh[j][k] = (act && dh >= 0) ? __ldg(u + dh) : 0.0;
        }
#pragma unroll
      for (int j = 0; j < RW; ++j)
#pragma unroll
        for (int k = 0; k < SX; ++k) {
          if (dd[j][k] < 0) continue;
          const double v = G.a_diag * (clo[j][k] + chi[j][k]) * u0[j][k] +
                           G.a_off * (clo[j][k] * ul[j][k] + chi[j][k] * uh[j][k]);
          y[dd[j][k]] = alpha * v + (beta == 0.0 ? 0.0 : beta * y[dd[j][k]]);
        }
    }
  }
}

// Mode B Dirichlet faces (dofs n_flux_int..n_flux-1): one cell each, partner =
// that cell's other face along the drop axis
__global__ void flux_A_bnd_kernel(bddc_geom G, const double* __restrict__ coef, const double* __restrict__ u,
                                  double alpha, double beta, double* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 2 * G.n_bt) return;
  const int d = G.n_flux_int + r;
  int side, gc[3];
  decode_bnd(G, d, side, gc);
  const int a = G.dir_axis;
  const double c = coef[(size_t)a * G.n_cells + cell_id(G, gc[0], gc[1], gc[2])];
  int other;
  if (G.n[a] == 1) {
    other = bnd_dof(G, 1 - side, gc);
  } else {
    gc[a] = side ? G.n[a] - 1 : 1;
    other = face_dof(G, a, gc[0], gc[1], gc[2]);
  }
  const double v = G.a_diag * c * u[d] + G.a_off * c * u[other];
  y[d] = alpha * v + (beta == 0.0 ? 0.0 : beta * y[d]);
}

// out_c = s_f * fvec_c + s_b * Dcell_c * (B u)_c   (Dcell = D of the cell's subdomain, or 1);
// warp per cell row, the 2 dim face loads of each cell predicated and issued first
__global__ void __launch_bounds__(ST) cell_div_kernel(bddc_geom G, const double* __restrict__ u,
                                                      const double* __restrict__ fvec, double s_f, double s_b,
                                                      const int* __restrict__ cell_sub,
                                                      const double* __restrict__ Dsub, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * ST) >> 5;
  const int nrows = G.n[1] * G.n[2];
  const int ex = G.n[0] - 1;
  for (int R0 = ((blockIdx.x * ST + threadIdx.x) >> 5) * RW; R0 < nrows; R0 += nw * RW) {
    for (int x0 = 0; x0 < G.n[0]; x0 += 32 * SX) {
      double b[RW][SX], fv[RW][SX], D[RW][SX];
      int cc[RW][SX];
#pragma unroll
      for (int j = 0; j < RW; ++j) {
        const int R = imin(R0 + j, nrows - 1);
        const int yy = R % G.n[1], z = R / G.n[1];
        const int c0 = G.n[0] * (yy + G.n[1] * z);
        const int dx0 = G.fam_off[0] + ex * (yy + G.n[1] * z) - 1;
        const int dyl0 = G.fam_off[1] + G.n[0] * (yy - 1 + (G.n[1] - 1) * z);
        const int dzl0 = G.fam_off[2] + G.n[0] * (yy + G.n[1] * (z - 1));
#pragma unroll
        for (int k = 0; k < SX; ++k) {
          const int x = x0 + lane + 32 * k;
          const bool act = x < G.n[0] && R0 + j < nrows;
          const int c3[3] = {x, yy, z};
          cc[j][k] = act ? c0 + x : -1;
          int dlo[3] = {-1, -1, -1}, dhi[3] = {-1, -1, -1};
          dlo[0] = x > 0 ? dx0 + x : (G.dir_axis == 0 ? bnd_dof(G, 0, c3) : -1);
          dhi[0] = x < G.n[0] - 1 ? dx0 + x + 1 : (G.dir_axis == 0 ? bnd_dof(G, 1, c3) : -1);
          if (G.dim > 1) {
            dlo[1] = yy > 0 ? dyl0 + x : (G.dir_axis == 1 ? bnd_dof(G, 0, c3) : -1);
            dhi[1] = yy < G.n[1] - 1 ? dyl0 + G.n[0] + x : (G.dir_axis == 1 ? bnd_dof(G, 1, c3) : -1);
          }
          if (G.dim > 2) {
            dlo[2] = z > 0 ? dzl0 + x : (G.dir_axis == 2 ? bnd_dof(G, 0, c3) : -1);
            dhi[2] = z < G.n[2] - 1 ? dzl0 + G.n[0] * G.n[1] + x : (G.dir_axis == 2 ? bnd_dof(G, 1, c3) : -1);
          }
          double sacc = 0.0;
#pragma unroll
          for (int a2 = 0; a2 < 3; ++a2) {
            const double vl = (act && dlo[a2] >= 0) ? __ldg(u + dlo[a2]) : 0.0;
            const double vh = (act && dhi[a2] >= 0) ? __ldg(u + dhi[a2]) : 0.0;
            sacc += vl - vh;
          }
          b[j][k] = sacc;
          fv[j][k] = (act && fvec) ? __ldg(fvec + c0 + x) : 0.0;
          D[j][k] = (act && Dsub) ? __ldg(Dsub + __ldg(cell_sub + c0 + x)) : 1.0;
        }
      }
#pragma unroll
      for (int j = 0; j < RW; ++j)
#pragma unroll
        for (int k = 0; k < SX; ++k) {
          if (cc[j][k] < 0) continue;
          double v = s_b * D[j][k] * b[j][k];
          if (fvec) v += s_f * fv[j][k];
          out[cc[j][k]] = v;
        }
    }
  }
}

// y_d = alpha (p_hi - p_lo) + beta y_d on the interior faces (warp per row)
__global__ void __launch_bounds__(ST) grad_kernel(bddc_geom G, const double* __restrict__ p, double alpha,
                                                  double beta, double* __restrict__ y, int nrows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * ST) >> 5;
  for (int R0 = ((blockIdx.x * ST + threadIdx.x) >> 5) * RW; R0 < nrows; R0 += nw * RW) {
    FluxRow r[RW];
    int emax = 0;
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      r[j] = flux_row(G, imin(R0 + j, nrows - 1));
      if (R0 + j >= nrows) r[j].e0 = 0;
      emax = imax(emax, r[j].e0);
    }
    for (int x0 = 0; x0 < emax; x0 += 32 * SX) {
      double ph[RW][SX], pl[RW][SX];
#pragma unroll
      for (int j = 0; j < RW; ++j)
#pragma unroll
        for (int k = 0; k < SX; ++k) {
          const int x = x0 + lane + 32 * k;
          const bool act = x < r[j].e0;
          ph[j][k] = act ? __ldg(p + r[j].h0 + x) : 0.0;
          pl[j][k] = act ? __ldg(p + r[j].h0 + x - r[j].st) : 0.0;
        }
#pragma unroll
      for (int j = 0; j < RW; ++j)
#pragma unroll
        for (int k = 0; k < SX; ++k) {
          const int x = x0 + lane + 32 * k;
          if (x >= r[j].e0) continue;
          const int d = r[j].d0 + x;
          y[d] = alpha * (ph[j][k] - pl[j][k]) + (beta == 0.0 ? 0.0 : beta * y[d]);
        }
    }
  }
}

// Mode B Dirichlet faces: +p of the cell above (low end), -p below (high end)
__global__ void grad_bnd_kernel(bddc_geom G, const double* __restrict__ p, double alpha, double beta,
                                double* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 2 * G.n_bt) return;
  const int d = G.n_flux_int + r;
  int side, gc[3];
  decode_bnd(G, d, side, gc);
  const double pc = p[cell_id(G, gc[0], gc[1], gc[2])];
  y[d] = alpha * (side ? -pc : pc) + (beta == 0.0 ? 0.0 : beta * y[d]);
}

// Orthonormal DCT-II matrix C[k][x] = s_k cos(pi k (x+1/2)/n) and eigenvalues 4 sin^2(pi k/(2n))
// of the 1-D Neumann cell Laplacian; with `dir` the DST-I pair sqrt(2/(n+1)) sin(pi (k+1)(x+1)/(n+1)),
// 4 sin^2(pi (k+1)/(2(n+1))) of tridiag(-1, 2, -1) (both ends on a Dirichlet face).
__global__ void dct_matrix_kernel(int n, int dir, double* __restrict__ C, double* __restrict__ lam) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n * n) {
    int k = e / n, x = e % n;
    if (dir) {
      C[e] = sqrt(2.0 / (n + 1)) * sinpi((double)(k + 1) * (x + 1) / (n + 1));
    } else {
      double s = (k == 0) ? sqrt(1.0 / n) : sqrt(2.0 / n);
      C[e] = s * cospi((double)k * (x + 0.5) / n);
    }
  }
  if (e < n) {
    double sn = dir ? sinpi((double)(e + 1) / (2.0 * (n + 1))) : sinpi((double)e / (2.0 * n));
    lam[e] = 4.0 * sn * sn;
  }
}

__global__ void dct_scale_kernel(int nx, int ny, int nz, const double* __restrict__ lx, const double* __restrict__ ly,
                                 const double* __restrict__ lz, double* __restrict__ v) {
  long long n = (long long)nx * ny * nz;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    int x = (int)(e % nx), y = (int)((e / nx) % ny), z = (int)(e / ((long long)nx * ny));
    double l = lx[x] + ly[y] + lz[z];
    v[e] = (l == 0.0) ? 0.0 : v[e] / l;   // the Neumann null mode (k = 0 on every axis: l is exactly 0)
  }
}

__global__ void sub_mean_kernel(long long n, const double* __restrict__ sum, double* __restrict__ v) {
  const double m = sum[0] / (double)n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    v[e] -= m;
}

}  // namespace

namespace {
// rows of the interior-face families (flux operators) or of the cells
int flux_rows(const bddc_geom* g) {
  int t = 0;
  for (int a = 0; a < g->dim; ++a) t += (g->n[1] - (a == 1)) * ((g->dim > 2) ? g->n[2] - (a == 2) : 1);
  return t;
}
// grid-stride launch: exactly the CTAs that are co-resident (one wave), never more
// than the rows need
template <typename K>
dim3 row_grid(K kernel, int nrows) {
  int dev = 0, nsm = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, ST, 0);
  const int need = (nrows + RW * ST / 32 - 1) / (RW * ST / 32);
  return dim3((unsigned)imax(1, imin(need, nsm * imax(occ, 1))));
}
}  // namespace

extern "C" int bddc_flux_A(const bddc_geom* g, const double* coef, const double* u, double alpha, double beta,
                           double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int nr = flux_rows(g);
  flux_A_kernel<<<row_grid(flux_A_kernel, nr), ST, 0, s>>>(*g, coef, u, alpha, beta, y, nr);
  LAUNCH_OK();
  if (g->dir_axis >= 0 && g->n_bt > 0) {
    flux_A_bnd_kernel<<<(2 * g->n_bt + 255) / 256, 256, 0, s>>>(*g, coef, u, alpha, beta, y);
    LAUNCH_OK();
  }
  return 0;
}

extern "C" int bddc_cell_div(const bddc_geom* g, const double* u, const double* fvec, double s_f, double s_b,
                             const int* cell_sub, const double* Dsub, double* out, void* stream) {
  cell_div_kernel<<<row_grid(cell_div_kernel, g->n[1] * g->n[2]), ST, 0, (cudaStream_t)stream>>>(*g, u, fvec, s_f, s_b,
                                                                                           cell_sub,
                                                                              Dsub, out);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_grad(const bddc_geom* g, const double* p, double alpha, double beta, double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int nr = flux_rows(g);
  grad_kernel<<<row_grid(grad_kernel, nr), ST, 0, s>>>(*g, p, alpha, beta, y, nr);
  LAUNCH_OK();
  if (g->dir_axis >= 0 && g->n_bt > 0) {
    grad_bnd_kernel<<<(2 * g->n_bt + 255) / 256, 256, 0, s>>>(*g, p, alpha, beta, y);
    LAUNCH_OK();
  }
  return 0;
}

// dct: workspace with C_x, C_y, C_z (n_a^2) and eigenvalues (n_a), built once.
extern "C" int bddc_dct_init(const bddc_geom* g, double* dct, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* p = dct;
  for (int a = 0; a < 3; ++a) {
    int n = g->n[a];
    dct_matrix_kernel<<<(n * n + 255) / 256, 256, 0, s>>>(n, a == g->dir_axis, p, p + n * n);
    LAUNCH_OK();
    p += n * n + n;
  }
  return 0;
}

// Solve (B B^T) p = rhs for the zero-mean p, in place on rhs (n_cells).
// tmp: n_cells doubles.
extern "C" int bddc_neumann_solve(const bddc_geom* g, const double* dct, double* rhs, double* tmp, void* stream) {
  const int nx = g->n[0], ny = g->n[1], nz = g->n[2];
  const double* Cx = dct;
  const double* lx = Cx + nx * nx;
  const double* Cy = lx + nx;
  const double* ly = Cy + ny * ny;
  const double* Cz = ly + ny;
  const double* lz = Cz + nz * nz;
  int r;
  // forward: v1 = rhs . Cx^T  (rows = (z,y), cols = x)
  if ((r = bddc_dgemm_batched(0, 1, ny * nz, nx, nx, 1.0, rhs, nx, 0, Cx, nx, 0, 0.0, tmp, nx, 0, 1, 0, stream)))
    return r;
  // v2[z] = Cy . v1[z]
  if ((r = bddc_dgemm_batched(0, 0, ny, nx, ny, 1.0, Cy, ny, 0, tmp, nx, (long long)nx * ny, 0.0, rhs, nx,
                              (long long)nx * ny, nz, 0, stream)))
    return r;
  // v3 = Cz . v2  (rows z, cols (y,x))
  if ((r = bddc_dgemm_batched(0, 0, nz, nx * ny, nz, 1.0, Cz, nz, 0, rhs, nx * ny, 0, 0.0, tmp, nx * ny, 0, 1, 0,
                              stream)))
    return r;
  dct_scale_kernel<<<592, 256, 0, (cudaStream_t)stream>>>(nx, ny, nz, lx, ly, lz, tmp);
  LAUNCH_OK();
  // inverse: v2 = Cz^T v3
  if ((r = bddc_dgemm_batched(1, 0, nz, nx * ny, nz, 1.0, Cz, nz, 0, tmp, nx * ny, 0, 0.0, rhs, nx * ny, 0, 1, 0,
                              stream)))
    return r;
  // v1[z] = Cy^T v2[z]
  if ((r = bddc_dgemm_batched(1, 0, ny, nx, ny, 1.0, Cy, ny, 0, rhs, nx, (long long)nx * ny, 0.0, tmp, nx,
                              (long long)nx * ny, nz, 0, stream)))
    return r;
  // p = v1 . Cx
  if ((r = bddc_dgemm_batched(0, 0, ny * nz, nx, nx, 1.0, tmp, nx, 0, Cx, nx, 0, 0.0, rhs, nx, 0, 1, 0, stream)))
    return r;
  return 0;
}

extern "C" int bddc_sub_mean(long long n, const double* sum, double* v, void* stream) {
  sub_mean_kernel<<<592, 256, 0, (cudaStream_t)stream>>>(n, sum, v);
  LAUNCH_OK();
  return 0;
}

namespace {

// out[i] = scale * sum_{cells of i} v[c] / (Dsub ? Dsub[i] : 1)
__global__ void sub_sum_kernel(bddc_geom G, const double* __restrict__ v, double* __restrict__ out, double scale,
                               const double* __restrict__ Dsub) {
  __shared__ double red[32];
  const int i = blockIdx.x;
  const Box b = sub_box(G, i);
  const int np = b.L[0] * b.L[1] * b.L[2];
  double acc = 0.0;
  for (int c = threadIdx.x; c < np; c += blockDim.x) {
    int lx = c % b.L[0], ly = (c / b.L[0]) % b.L[1], lz = c / (b.L[0] * b.L[1]);
    acc += v[cell_id(G, b.o[0] + lx, b.o[1] + ly, b.o[2] + lz)];
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) out[i] = scale * acc / (Dsub ? Dsub[i] : 1.0);
}

__global__ void gamma_flux_kernel(int n, const int* __restrict__ gamma, double* __restrict__ gv,
                                  double* __restrict__ flux, int mode) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  if (mode == 0) flux[gamma[d]] = gv[d];
  else if (mode == 1) flux[gamma[d]] += gv[d];
  else gv[d] = flux[gamma[d]];
}

// balanced_shift (solver.py:146-164): w[d] = (z[i_f] - z[j_f]) / m_f
__global__ void face_shift_kernel(int n, const int* __restrict__ gface, const int* __restrict__ faces,
                                  const double* __restrict__ z, double* __restrict__ w) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  int f = gface[d];
  w[d] = (z[faces[4 * f]] - z[faces[4 * f + 1]]) / (double)faces[4 * f + 3];
}

}  // namespace

extern "C" int bddc_sub_sum(const bddc_geom* g, const double* v, double* out, double scale, const double* Dsub,
                            void* stream) {
  sub_sum_kernel<<<g->N, 256, 0, (cudaStream_t)stream>>>(*g, v, out, scale, Dsub);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_gamma_flux(int n, const int* gamma, double* gv, double* flux, int mode, void* stream) {
  if (n <= 0) return 0;
  gamma_flux_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, gamma, gv, flux, mode);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_face_shift(int n, int n_faces, const int* gface, const int* faces, const double* z, double* w,
                               void* stream) {
  if (n <= 0) return 0;
  face_shift_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, gface, faces, z, w);
  LAUNCH_OK();
  return 0;
}

namespace {
__global__ void scale_cells_kernel(int n, const double* __restrict__ f, const int* __restrict__ cell_sub,
                                   const double* __restrict__ Dsub, double* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) out[c] = Dsub[cell_sub[c]] * f[c];
}
}  // namespace

// fs = D f (grid.py:250-251)
extern "C" int bddc_scale_cells(const bddc_geom* g, const double* f, const int* cell_sub, const double* Dsub,
                                double* out, void* stream) {
  scale_cells_kernel<<<(g->n_cells + 255) / 256, 256, 0, (cudaStream_t)stream>>>(g->n_cells, f, cell_sub, Dsub, out);
  LAUNCH_OK();
  return 0;
}
