// Multifrontal (nested-dissection) coarse solver kernels, see coarse_nd.py.
// Replaces the dense coarse lu_factor/lu_solve of coarse.py:186-215.
#include "common.cuh"

namespace {

// F = 0 with identity on the padded separator diagonal (slot == -1), or
// extend-add of child `slot` of every node into its front.
__global__ void nd_assemble_kernel(int m, int S, int B, int nf, int slot, int K, const int* __restrict__ cmap,
                                   const int* __restrict__ ckind, const int* __restrict__ sep_idx,
                                   double* __restrict__ F, const double* __restrict__ Fc, int Sc, int nfc,
                                   const double* __restrict__ Kc, const int* __restrict__ sub_rows,
                                   const double* __restrict__ b0, int maxC) {
  const int q = blockIdx.y;
  double* Fq = F + (size_t)q * nf * nf;
  if (slot < 0) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)nf * nf;
         e += (long long)gridDim.x * blockDim.x) {
      int r = (int)(e / nf), c = (int)(e % nf);
      double v = 0.0;
      if (r == c && r < S && sep_idx[(size_t)q * S + r] < 0) v = 1.0;
      Fq[e] = v;
    }
    return;
  }
  const int* mp = cmap + ((size_t)slot * m + q) * K;
  const int* ck = ckind + ((size_t)slot * m + q) * 3;
  const int kind = ck[0], idx = ck[1], npr = ck[2];
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)K * K;
       e += (long long)gridDim.x * blockDim.x) {
    int r = (int)(e / K), c = (int)(e % K);
    int pr = mp[r], pc = mp[c];
    if (pr < 0 || pc < 0) continue;
    double v;
    if (kind == 1) {
      // leaf: [[sigma sigma^T Kc, b0^T],[b0, 0]] over (rows 0..npr-1, pressure npr)
      if (r < npr && c < npr) {
        const int* a = sub_rows + ((size_t)idx * maxC + r) * 4;
        const int* b = sub_rows + ((size_t)idx * maxC + c) * 4;
        v = (double)(a[3] * b[3]) * Kc[((size_t)idx * maxC + r) * maxC + c];
      } else if (r < npr) {
        v = b0[(size_t)idx * maxC + r];
      } else if (c < npr) {
        v = b0[(size_t)idx * maxC + c];
      } else {
        v = 0.0;
      }
    } else {
      v = Fc[(size_t)idx * nfc * nfc + (size_t)(Sc + r) * nfc + Sc + c];
    }
    Fq[(size_t)pr * nf + pc] += v;
  }
}

// Forward (left-looking): r_sep[k] = r[g_k] - sum of the stored descendant
// contributions for g_k (fixed order), then y = F11inv r_sep (rows < S) and
// c = X r_sep (rows S..S+Bf-1) into the level's slice of the global cbuf.
__global__ void nd_fwd_kernel(int m, int S, int Bf, int nf, long long xstride, const int* __restrict__ sep_idx,
                              const int* __restrict__ lptr, const int* __restrict__ lsrc,
                              const double* __restrict__ F, const double* __restrict__ X,
                              const double* __restrict__ r, double* __restrict__ ybuf, double* __restrict__ cbuf,
                              long long coff, int rows_per_cta) {
  extern __shared__ double rs[];  // S
  const int q = blockIdx.x;
  const int row0 = blockIdx.y * rows_per_cta;
  const int Bp = Bf > 0 ? Bf : 1;
  // thread per separator slot; contributions fetched 4 at a time (independent
  // loads) and added strictly in list order (deterministic)
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    int g = sep_idx[(size_t)q * S + k];
    double v = 0.0;
    if (g >= 0) {
      const int t = q * S + k;
      int p = lptr[t];
      const int p1 = lptr[t + 1];
      double acc = 0.0;
      for (; p + 4 <= p1; p += 4) {
        int i0 = lsrc[p], i1 = lsrc[p + 1], i2 = lsrc[p + 2], i3 = lsrc[p + 3];
        double c0 = cbuf[i0], c1 = cbuf[i1], c2 = cbuf[i2], c3 = cbuf[i3];
        acc += c0;
        acc += c1;
        acc += c2;
        acc += c3;
      }
      for (; p < p1; ++p) acc += cbuf[lsrc[p]];
      v = r[g] - acc;
    }
    rs[k] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nrows = S + Bf;
  for (int row = row0 + warp; row < imin(row0 + rows_per_cta, nrows); row += nw) {
    const double* mr = (row < S) ? F + (size_t)q * nf * nf + (size_t)row * nf
                                 : X + (size_t)q * xstride + (size_t)(row - S) * S;
    double acc = 0.0;
    for (int c = lane; c < S; c += 32) acc += mr[c] * rs[c];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (row < S) ybuf[(size_t)q * S + row] = acc;
      else cbuf[coff + (size_t)q * Bp + (row - S)] = acc;
    }
  }
}

// Backward: x_sep = y - X^T x_bnd.  CTA = 32 separator columns; the 8 warps
// split the boundary rows and their partial sums are added in warp order.
__global__ void nd_bwd_kernel(int m, int S, int Bf, long long xstride, const int* __restrict__ sep_idx,
                              const int* __restrict__ bnd_idx, const double* __restrict__ X,
                              const double* __restrict__ ybuf, double* __restrict__ x) {
  extern __shared__ double xb[];  // Bf, then 8 x 32 partials
  const int q = blockIdx.x;
  const int k0 = blockIdx.y * 32;
  const int Bp = Bf > 0 ? Bf : 1;
  double* part = xb + Bp;
  for (int mm = threadIdx.x; mm < Bf; mm += blockDim.x) {
    int g = bnd_idx[(size_t)q * Bp + mm];
    xb[mm] = (g >= 0) ? x[g] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = k0 + lane;
  double acc = 0.0;
  if (k < S) {
    const double* Xq = X + (size_t)q * xstride + k;
    for (int mm = warp; mm < Bf; mm += 8) acc += Xq[(size_t)mm * S] * xb[mm];
  }
  part[warp * 32 + lane] = acc;
  __syncthreads();
  if (warp == 0 && k < S) {
    int g = sep_idx[(size_t)q * S + k];
    if (g >= 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += part[w * 32 + lane];
      x[g] = ybuf[(size_t)q * S + k] - t;
    }
  }
}

// Pc[(i-1),(j-1)] = -U_root[i][j] (i, j >= 1): the pinned pressure Schur complement;
// identity beyond N-1.
__global__ void nd_extract_pc_kernel(const double* __restrict__ F, int nf, int S, int N, double* __restrict__ Pc,
                                     int npc) {
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)npc * npc) return;
  int r = (int)(e / npc), c = (int)(e % npc);
  double v;
  if (r < N - 1 && c < N - 1) v = -F[(size_t)(S + 1 + r) * nf + S + 1 + c];
  else v = (r == c) ? 1.0 : 0.0;
  Pc[e] = v;
}

// out[(i-1) + j*ldo] = sum_r b0[i][r] Y[g_r + j*ldy]   (i >= 1); warp per (i, j)
__global__ void b0_apply_kernel(int N, int maxC, const int* __restrict__ sub_rows, const double* __restrict__ b0,
                                const double* __restrict__ Y, int ldy, int nrhs, double* __restrict__ out, int ldo) {
  long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long long)(N - 1) * nrhs) return;
  int i = 1 + (int)(w % (N - 1)), j = (int)(w / (N - 1));
  double s = 0.0;
  for (int r = lane; r < maxC; r += 32) {
    int g = sub_rows[((size_t)i * maxC + r) * 4];
    if (g >= 0) s += b0[(size_t)i * maxC + r] * Y[(size_t)g + (size_t)j * ldy];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[(size_t)(i - 1) + (size_t)j * ldo] = s;
}

// r[g + j*ldr] += alpha * (b0[lo] z[i_lo-1] + b0[hi] z[i_hi-1])   (owners with i >= 1)
__global__ void b0t_apply_kernel(int nfc, int maxC, const int* __restrict__ cown, const double* __restrict__ b0,
                                 const double* __restrict__ z, int ldz, int nrhs, double alpha, double* __restrict__ r,
                                 int ldr) {
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)nfc * nrhs) return;
  int g = (int)(e % nfc), j = (int)(e / nfc);
  double s = 0.0;
  for (int w = 0; w < 2; ++w) {
    int bi = cown[2 * g + w];
    int i = bi / maxC;
    if (i >= 1) s += b0[bi] * z[(size_t)(i - 1) + (size_t)j * ldz];
  }
  r[(size_t)g + (size_t)j * ldr] += alpha * s;
}

__global__ void fill_kernel(long long n, double v, double* __restrict__ a) {
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) a[e] = v;
}

}  // namespace

extern "C" int bddc_nd_assemble(int m, int S, int B, int nf, int slot, int K, const int* cmap, const int* ckind,
                                const int* sep_idx, double* F, const double* Fc, int Sc, int nfc, const double* Kc,
                                const int* sub_rows, const double* b0, int maxC, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (slot < 0 || slot == 0) {
    long long tot = (long long)nf * nf;
    dim3 g0((unsigned)imin((int)((tot + 255) / 256), 1024), m);
    nd_assemble_kernel<<<g0, 256, 0, s>>>(m, S, B, nf, -1, K, cmap, ckind, sep_idx, F, Fc, Sc, nfc, Kc, sub_rows,
                                          b0, maxC);
    LAUNCH_OK();
  }
  long long tot = (long long)K * K;
  dim3 g((unsigned)imin((int)((tot + 255) / 256), 1024), m);
  nd_assemble_kernel<<<g, 256, 0, s>>>(m, S, B, nf, slot, K, cmap, ckind, sep_idx, F, Fc, Sc, nfc, Kc, sub_rows, b0,
                                       maxC);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_nd_fwd(int m, int S, int Bf, int nf, long long xstride, const int* sep_idx, const int* lptr,
                           const int* lsrc, const double* F, const double* X, const double* r, double* ybuf,
                           double* cbuf, long long coff, void* stream) {
  const int rows_per_cta = 32;
  dim3 g(m, (S + Bf + rows_per_cta - 1) / rows_per_cta);
  size_t shm = (size_t)S * sizeof(double);
  if (shm > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(nd_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  nd_fwd_kernel<<<g, 256, shm, (cudaStream_t)stream>>>(m, S, Bf, nf, xstride, sep_idx, lptr, lsrc, F, X, r, ybuf, cbuf,
                                                       coff, rows_per_cta);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_nd_bwd(int m, int S, int Bf, long long xstride, const int* sep_idx, const int* bnd_idx,
                           const double* X, const double* ybuf, double* x, void* stream) {
  dim3 g(m, (S + 31) / 32);
  size_t shm = ((size_t)(Bf > 0 ? Bf : 1) + 8 * 32) * sizeof(double);
  if (shm > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(nd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  nd_bwd_kernel<<<g, 256, shm, (cudaStream_t)stream>>>(m, S, Bf, xstride, sep_idx, bnd_idx, X, ybuf, x);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_nd_extract_pc(const double* F, int nf, int S, int N, double* Pc, int npc, void* stream) {
  long long tot = (long long)npc * npc;
  nd_extract_pc_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(F, nf, S, N, Pc, npc);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_b0_apply(int N, int maxC, const int* sub_rows, const double* b0, const double* Y, int ldy,
                             int nrhs, double* out, int ldo, void* stream) {
  if (N < 2) return 0;
  long long tot = (long long)(N - 1) * nrhs * 32;
  b0_apply_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(N, maxC, sub_rows, b0, Y, ldy,
                                                                                    nrhs, out, ldo);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_b0t_apply(int nfc, int maxC, const int* cown, const double* b0, const double* z, int ldz, int nrhs,
                              double alpha, double* r, int ldr, void* stream) {
  if (nfc <= 0) return 0;
  long long tot = (long long)nfc * nrhs;
  b0t_apply_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nfc, maxC, cown, b0, z, ldz, nrhs,
                                                                                     alpha, r, ldr);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_fill(long long n, double v, double* a, void* stream) {
  if (n <= 0) return 0;
  fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, v, a);
  LAUNCH_OK();
  return 0;
}

