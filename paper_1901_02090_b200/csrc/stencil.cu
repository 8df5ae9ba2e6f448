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

// Row-structured launches, no integer division: thread (x, ty) of CTA
// (bx, by, bz) handles element x (+ RX k) of grid row (f1, f2) = (RY bx + ty, by)
// of family bz (flux operators; cells: bz = 0).  Consecutive threads touch
// consecutive dofs, cells and (structure-of-arrays) coefficients.
constexpr int RX = 64, RY = 4;

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

// y = alpha * A u + beta * y on the interior faces
__global__ void __launch_bounds__(RX* RY) flux_A_kernel(bddc_geom G, const double* __restrict__ coef,
                                                        const double* __restrict__ u, double alpha, double beta,
                                                        double* __restrict__ y) {
  const int a = blockIdx.z;
  int e0, f[3], d0;
  if (!fam_row(G, a, blockIdx.x * RY + threadIdx.y, blockIdx.y, e0, f, d0)) return;
  const int st = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
  const double* ca = coef + (size_t)a * G.n_cells;
  const int h0 = cell_id(G, f[0], f[1], f[2]);
  const bool lo_in = f[a] > 1 || a == 0, hi_in = f[a] < G.n[a] - 1 || a == 0;   // along a (x: per element)
  for (int x = threadIdx.x; x < e0; x += RX) {
    const int d = d0 + x, hi = h0 + x, lo = hi - st;
    const double clo = ca[lo], chi = ca[hi];
    double v = G.a_diag * (clo + chi) * u[d];
    const bool l = a == 0 ? x > 0 : lo_in, h = a == 0 ? x < e0 - 1 : hi_in;
    // dof stride along a inside family a equals the cell stride st
    double w = 0.0;
    if (l) w += clo * u[d - st];
    else if (a == G.dir_axis) {
      int g[3] = {f[0] + x, f[1], f[2]};
      w += clo * u[bnd_dof(G, 0, g)];
    }
    if (h) w += chi * u[d + st];
    else if (a == G.dir_axis) {
      int g[3] = {f[0] + x, f[1], f[2]};
      w += chi * u[bnd_dof(G, 1, g)];
    }
    v += G.a_off * w;
    y[d] = alpha * v + (beta == 0.0 ? 0.0 : beta * y[d]);
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

// out_c = s_f * fvec_c + s_b * Dcell_c * (B u)_c   (Dcell = D of the cell's subdomain, or 1)
__global__ void __launch_bounds__(RX* RY) cell_div_kernel(bddc_geom G, const double* __restrict__ u,
                                                          const double* __restrict__ fvec, double s_f, double s_b,
                                                          const int* __restrict__ cell_sub,
                                                          const double* __restrict__ Dsub, double* __restrict__ out) {
  const int y = blockIdx.x * RY + threadIdx.y, z = blockIdx.y;
  if (y >= G.n[1] || z >= G.n[2]) return;
  const int c0 = G.n[0] * (y + G.n[1] * z);
  // first dofs of this row's faces: x-faces (x-1, y, z) and the y / z faces (x, ., .)
  const int ex = G.n[0] - 1;
  const int dx = G.fam_off[0] + ex * (y + G.n[1] * z) - 1;
  const int dyl = G.fam_off[1] + G.n[0] * (y - 1 + (G.n[1] - 1) * z), dyh = dyl + G.n[0];
  const int dzl = G.fam_off[2] + G.n[0] * (y + G.n[1] * (z - 1)), dzh = dzl + G.n[0] * G.n[1];
  for (int x = threadIdx.x; x < G.n[0]; x += RX) {
    const int c3[3] = {x, y, z};
    double b = 0.0;
    if (x > 0) b += u[dx + x];
    else if (G.dir_axis == 0) b += u[bnd_dof(G, 0, c3)];
    if (x < G.n[0] - 1) b -= u[dx + x + 1];
    else if (G.dir_axis == 0) b -= u[bnd_dof(G, 1, c3)];
    if (G.dim > 1) {
      if (y > 0) b += u[dyl + x];
      else if (G.dir_axis == 1) b += u[bnd_dof(G, 0, c3)];
      if (y < G.n[1] - 1) b -= u[dyh + x];
      else if (G.dir_axis == 1) b -= u[bnd_dof(G, 1, c3)];
    }
    if (G.dim > 2) {
      if (z > 0) b += u[dzl + x];
      else if (G.dir_axis == 2) b += u[bnd_dof(G, 0, c3)];
      if (z < G.n[2] - 1) b -= u[dzh + x];
      else if (G.dir_axis == 2) b -= u[bnd_dof(G, 1, c3)];
    }
    const int c = c0 + x;
    const double D = Dsub ? Dsub[cell_sub[c]] : 1.0;
    double v = s_b * D * b;
    if (fvec) v += s_f * fvec[c];
    out[c] = v;
  }
}

// y_d = alpha (p_hi - p_lo) + beta y_d on the interior faces
__global__ void __launch_bounds__(RX* RY) grad_kernel(bddc_geom G, const double* __restrict__ p, double alpha,
                                                      double beta, double* __restrict__ y) {
  const int a = blockIdx.z;
  int e0, f[3], d0;
  if (!fam_row(G, a, blockIdx.x * RY + threadIdx.y, blockIdx.y, e0, f, d0)) return;
  const int st = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
  const int h0 = cell_id(G, f[0], f[1], f[2]);
  for (int x = threadIdx.x; x < e0; x += RX) {
    const int hi = h0 + x, d = d0 + x;
    y[d] = alpha * (p[hi] - p[hi - st]) + (beta == 0.0 ? 0.0 : beta * y[d]);
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
// (n1 / RY, n2) covers every family's (e1, e2)
dim3 row_grid(const bddc_geom* g, int fams) {
  return dim3((g->n[1] + RY - 1) / RY, g->n[2], fams);
}
}  // namespace

extern "C" int bddc_flux_A(const bddc_geom* g, const double* coef, const double* u, double alpha, double beta,
                           double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  flux_A_kernel<<<row_grid(g, g->dim), dim3(RX, RY), 0, s>>>(*g, coef, u, alpha, beta, y);
  LAUNCH_OK();
  if (g->dir_axis >= 0 && g->n_bt > 0) {
    flux_A_bnd_kernel<<<(2 * g->n_bt + 255) / 256, 256, 0, s>>>(*g, coef, u, alpha, beta, y);
    LAUNCH_OK();
  }
  return 0;
}

extern "C" int bddc_cell_div(const bddc_geom* g, const double* u, const double* fvec, double s_f, double s_b,
                             const int* cell_sub, const double* Dsub, double* out, void* stream) {
  cell_div_kernel<<<row_grid(g, 1), dim3(RX, RY), 0, (cudaStream_t)stream>>>(*g, u, fvec, s_f, s_b, cell_sub,
                                                                              Dsub, out);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_grad(const bddc_geom* g, const double* p, double alpha, double beta, double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  grad_kernel<<<row_grid(g, g->dim), dim3(RX, RY), 0, s>>>(*g, p, alpha, beta, y);
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
