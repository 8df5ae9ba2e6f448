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
#include <cstdlib>

#include "common.cuh"

extern "C" int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha, const double* A,
                                  int lda, long long sA, const double* B, int ldb, long long sB, double beta,
                                  double* C, int ldc, long long sC, int batch, int upper, void* stream);

namespace {

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

// Flat operators: each family's dofs (and the cells) are one contiguous range;
// a CTA takes a block-uniform family and ST x SV consecutive entries of it, a
// thread SV entries ST apart (every warp access is 32 consecutive doubles), all
// loads of its SV entries issued before any is used.  Coordinates come from
// multiply-high divisions by the grid extents (FDiv, set up on the host).
constexpr int ST = 256;

struct FDiv {
  unsigned d, m, s;   // n / d = (umulhi(n, m) + n) >> s  for n < 2^31
};

FDiv fdiv(unsigned d) {
  unsigned s = 0;
  while ((1ull << s) < d) ++s;
  const unsigned long long m = (((1ull << 32) * ((1ull << s) - d)) / d) + 1;
  return FDiv{d, (unsigned)m, s};
}

__device__ __forceinline__ int fdivu(const FDiv& f, int n) {
  const unsigned t = __umulhi((unsigned)n, f.m);
  return (int)((t + (unsigned)n) >> f.s);
}

struct FlatArgs {
  int nb[3];    // CTAs per family
  FDiv dx0;     // nx - 1
  FDiv dx;      // nx
  FDiv dy0;     // ny - 1
  FDiv dy;      // ny
  FDiv dxy;     // nx * ny
};

// Interior face dof d of family a (r = d - fam_off[a]): its high cell and whether
// the partner faces d -+ st along a are interior faces (else: wall, or in mode B
// on the drop axis the Dirichlet face).
struct FaceAt {
  int hi;
  bool l, h;
};

__device__ __forceinline__ FaceAt face_at(const bddc_geom& G, const FlatArgs& F, int a, int r) {
  FaceAt f;
  if (a == 0) {
    const int q = fdivu(F.dx0, r), x = r - q * (G.n[0] - 1);
    f.hi = r + q + 1;
    f.l = x > 0;
    f.h = x < G.n[0] - 2;
  } else if (a == 1) {
    const int q = fdivu(F.dx, r), z = fdivu(F.dy0, q), y1 = q - z * (G.n[1] - 1);
    f.hi = r + G.n[0] * (1 + z);
    f.l = y1 > 0;
    f.h = y1 < G.n[1] - 2;
  } else {
    const int z1 = fdivu(F.dxy, r);
    f.hi = r + G.n[0] * G.n[1];
    f.l = z1 > 0;
    f.h = z1 < G.n[2] - 2;
  }
  return f;
}

// mode B: the Dirichlet face at end `side` of the line through cell `c` (along dir_axis)
__device__ __forceinline__ int bnd_of_cell(const bddc_geom& G, int side, int c) {
  const int x = c % G.n[0], y = (c / G.n[0]) % G.n[1], z = c / (G.n[0] * G.n[1]);
  // transverse coordinates of the drop axis (bnd_dof without a dynamically indexed array)
  const int g1 = G.dir_axis == 0 ? y : x, g2 = G.dir_axis == 2 ? y : z;
  const int n1 = G.dir_axis == 0 ? G.n[1] : G.n[0];
  return G.n_flux_int + side * G.n_bt + g1 + n1 * g2;
}

__device__ __forceinline__ int block_family(const FlatArgs& F, int& blk) {
  int a = 0;
  blk = blockIdx.x;
  if (blk >= F.nb[0]) { a = 1; blk -= F.nb[0]; }
  if (a == 1 && blk >= F.nb[1]) { a = 2; blk -= F.nb[1]; }
  return a;
}

// y = alpha * A u + beta * y on the interior faces (grid.py:270-307):
//   (A u)_d = a_diag (c_lo + c_hi) u_d + a_off (c_lo u_{d-st} + c_hi u_{d+st})
template <int SV>
__global__ void __launch_bounds__(ST) flux_A_kernel(bddc_geom G, FlatArgs F, const double* __restrict__ coef,
                                                    const double* __restrict__ u, double alpha, double beta,
                                                    double* __restrict__ y) {
  int blk;
  const int a = block_family(F, blk);
  const int off = G.fam_off[a], nfam = G.fam_off[a + 1] - off;
  const int st = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
  const double* __restrict__ ca = coef + (size_t)a * G.n_cells;
  const int r0 = blk * ST * SV + threadIdx.x;
  double clo[SV], chi[SV], u0[SV], ul[SV], uh[SV], yo[SV];
#pragma unroll
  for (int k = 0; k < SV; ++k) {
    const int r = r0 + k * ST;
    const bool act = r < nfam;
    const FaceAt f = face_at(G, F, a, act ? r : 0);
    const int d = off + r;
    int dl = f.l ? d - st : -1, dh = f.h ? d + st : -1;
    if (a == G.dir_axis && act && (!f.l || !f.h)) {
      if (!f.l) dl = bnd_of_cell(G, 0, f.hi);
      if (!f.h) dh = bnd_of_cell(G, 1, f.hi);
    }
    clo[k] = act ? __ldg(ca + f.hi - st) : 0.0;
    chi[k] = act ? __ldg(ca + f.hi) : 0.0;
    u0[k] = act ? __ldg(u + d) : 0.0;
    ul[k] = (act && dl >= 0) ? __ldg(u + dl) : 0.0;
    uh[k] = (act && dh >= 0) ? __ldg(u + dh) : 0.0;
    yo[k] = (act && beta != 0.0) ? y[d] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < SV; ++k) {
    const int r = r0 + k * ST;
    if (r >= nfam) break;
    const double v = G.a_diag * (clo[k] + chi[k]) * u0[k] + G.a_off * (clo[k] * ul[k] + chi[k] * uh[k]);
    y[off + r] = alpha * v + beta * yo[k];
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
// (B u)_c = sum_a u(low a-face) - u(high a-face), wall faces 0 (grid.py:310-324)
template <int SV>
__global__ void __launch_bounds__(ST) cell_div_kernel(bddc_geom G, FlatArgs F, const double* __restrict__ u,
                                                      const double* __restrict__ fvec, double s_f, double s_b,
                                                      const int* __restrict__ cell_sub,
                                                      const double* __restrict__ Dsub, double* __restrict__ out) {
  const int nx = G.n[0], ny = G.n[1], nxy = nx * ny;
  const int c0 = blockIdx.x * ST * SV + threadIdx.x;
  double b[SV], fv[SV], D[SV];
#pragma unroll
  for (int k = 0; k < SV; ++k) {
    const int c = c0 + k * ST;
    const bool act = c < G.n_cells;
    const int q = fdivu(F.dx, c), x = c - q * nx;
    const int z = fdivu(F.dy, q), yy = q - z * ny;
    int l0 = x > 0 ? G.fam_off[0] + c - q - 1 : -1;
    int h0 = x < nx - 1 ? G.fam_off[0] + c - q : -1;
    int l1 = (G.dim > 1 && yy > 0) ? G.fam_off[1] + c - nx * (1 + z) : -1;
    int h1 = (G.dim > 1 && yy < ny - 1) ? G.fam_off[1] + c - nx * z : -1;
    int l2 = (G.dim > 2 && z > 0) ? G.fam_off[2] + c - nxy : -1;
    int h2 = (G.dim > 2 && z < G.n[2] - 1) ? G.fam_off[2] + c : -1;
    if (G.dir_axis >= 0 && act) {   // mode B: the drop axis ends on Dirichlet faces
      const int ad = G.dir_axis;
      if (ad == 0 && l0 < 0) l0 = bnd_of_cell(G, 0, c);
      if (ad == 0 && h0 < 0) h0 = bnd_of_cell(G, 1, c);
      if (ad == 1 && l1 < 0) l1 = bnd_of_cell(G, 0, c);
      if (ad == 1 && h1 < 0) h1 = bnd_of_cell(G, 1, c);
      if (ad == 2 && l2 < 0) l2 = bnd_of_cell(G, 0, c);
      if (ad == 2 && h2 < 0) h2 = bnd_of_cell(G, 1, c);
    }
    const double v0 = (act && l0 >= 0) ? __ldg(u + l0) : 0.0, w0 = (act && h0 >= 0) ? __ldg(u + h0) : 0.0;
    const double v1 = (act && l1 >= 0) ? __ldg(u + l1) : 0.0, w1 = (act && h1 >= 0) ? __ldg(u + h1) : 0.0;
    const double v2 = (act && l2 >= 0) ? __ldg(u + l2) : 0.0, w2 = (act && h2 >= 0) ? __ldg(u + h2) : 0.0;
    const double sacc = ((v0 - w0) + (v1 - w1)) + (v2 - w2);
    b[k] = sacc;
    fv[k] = (act && fvec) ? __ldg(fvec + c) : 0.0;
    D[k] = (act && Dsub) ? __ldg(Dsub + __ldg(cell_sub + c)) : 1.0;
  }
#pragma unroll
  for (int k = 0; k < SV; ++k) {
    const int c = c0 + k * ST;
    if (c >= G.n_cells) break;
    double v = s_b * D[k] * b[k];
    if (fvec) v += s_f * fv[k];
    out[c] = v;
  }
}

// y_d = alpha (p_hi - p_lo) + beta y_d on the interior faces
template <int SV>
__global__ void __launch_bounds__(ST) grad_kernel(bddc_geom G, FlatArgs F, const double* __restrict__ p,
                                                  double alpha, double beta, double* __restrict__ y) {
  int blk;
  const int a = block_family(F, blk);
  const int off = G.fam_off[a], nfam = G.fam_off[a + 1] - off;
  const int st = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
  const int r0 = blk * ST * SV + threadIdx.x;
  double ph[SV], pl[SV], yo[SV];
#pragma unroll
  for (int k = 0; k < SV; ++k) {
    const int r = r0 + k * ST;
    const bool act = r < nfam;
    const FaceAt f = face_at(G, F, a, act ? r : 0);
    ph[k] = act ? __ldg(p + f.hi) : 0.0;
    pl[k] = act ? __ldg(p + f.hi - st) : 0.0;
    yo[k] = (act && beta != 0.0) ? y[off + r] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < SV; ++k) {
    const int r = r0 + k * ST;
    if (r >= nfam) break;
    y[off + r] = alpha * (ph[k] - pl[k]) + beta * yo[k];
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
// entries per thread: BDDC_STENCIL_SV overrides (tuning sweeps), else `def`
// (C3 sweep over 1/2/4/8: A u 3.9/4.4/4.6/3.6 TB/s, B u 3.4/3.4/2.9/2.0, B^T p 2.8/3.4/3.4/3.4)
int stencil_sv(int def) {
  static int ov = -1;
  if (ov < 0) {
    const char* e = getenv("BDDC_STENCIL_SV");
    ov = e ? atoi(e) : 0;
  }
  return (ov == 1 || ov == 2 || ov == 4 || ov == 8) ? ov : def;
}

// one CTA per ST x sv consecutive entries of a family (block-uniform family)
FlatArgs flat_args(const bddc_geom* g, int sv) {
  FlatArgs F;
  for (int a = 0; a < 3; ++a) {
    const int nfam = a < g->dim ? g->fam_off[a + 1] - g->fam_off[a] : 0;
    F.nb[a] = (nfam + ST * sv - 1) / (ST * sv);
  }
  F.dx0 = fdiv((unsigned)imax(1, g->n[0] - 1));
  F.dx = fdiv((unsigned)g->n[0]);
  F.dy0 = fdiv((unsigned)imax(1, g->n[1] - 1));
  F.dy = fdiv((unsigned)g->n[1]);
  F.dxy = fdiv((unsigned)(g->n[0] * g->n[1]));
  return F;
}
int flat_blocks(const FlatArgs& F) { return F.nb[0] + F.nb[1] + F.nb[2]; }

#define STENCIL_DISPATCH(sv, KER, GRID, STREAM, ...)                               \
  switch (sv) {                                                                    \
    case 1: KER<1><<<GRID, ST, 0, STREAM>>>(__VA_ARGS__); break;                   \
    case 2: KER<2><<<GRID, ST, 0, STREAM>>>(__VA_ARGS__); break;                   \
    case 8: KER<8><<<GRID, ST, 0, STREAM>>>(__VA_ARGS__); break;                   \
    default: KER<4><<<GRID, ST, 0, STREAM>>>(__VA_ARGS__); break;                  \
  }
}  // namespace

extern "C" int bddc_flux_A(const bddc_geom* g, const double* coef, const double* u, double alpha, double beta,
                           double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int sv = stencil_sv(4);
  const FlatArgs F = flat_args(g, sv);
  if (flat_blocks(F) > 0) {
    STENCIL_DISPATCH(sv, flux_A_kernel, flat_blocks(F), s, *g, F, coef, u, alpha, beta, y);
    LAUNCH_OK();
  }
  if (g->dir_axis >= 0 && g->n_bt > 0) {
    flux_A_bnd_kernel<<<(2 * g->n_bt + 255) / 256, 256, 0, s>>>(*g, coef, u, alpha, beta, y);
    LAUNCH_OK();
  }
  return 0;
}

extern "C" int bddc_cell_div(const bddc_geom* g, const double* u, const double* fvec, double s_f, double s_b,
                             const int* cell_sub, const double* Dsub, double* out, void* stream) {
  const int sv = stencil_sv(2);   // C3: 2.87 TB/s at 4 entries per thread, 3.43 at 2
  const FlatArgs F = flat_args(g, sv);
  const int nb = (g->n_cells + ST * sv - 1) / (ST * sv);
  STENCIL_DISPATCH(sv, cell_div_kernel, nb, (cudaStream_t)stream, *g, F, u, fvec, s_f, s_b, cell_sub, Dsub, out);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_grad(const bddc_geom* g, const double* p, double alpha, double beta, double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int sv = stencil_sv(4);
  const FlatArgs F = flat_args(g, sv);
  if (flat_blocks(F) > 0) {
    STENCIL_DISPATCH(sv, grad_kernel, flat_blocks(F), s, *g, F, p, alpha, beta, y);
    LAUNCH_OK();
  }
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
