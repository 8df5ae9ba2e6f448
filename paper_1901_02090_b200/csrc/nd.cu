// Multifrontal (nested-dissection) coarse solver kernels, see coarse_nd.py.
// Replaces the dense coarse lu_factor/lu_solve of coarse.py:186-215.
#include "common.cuh"

namespace {

// F = 0 with identity on the padded separator diagonal (slot == -1), or
// extend-add of child `slot` of every node into its front.
__global__ void nd_assemble_kernel(int m, int S, int Sf, int B, int nf, int slot, int K, const int* __restrict__ cmap,
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
      // padding of the pivot block: +1 on the flux part, -1 on the pressure part
      // (keeps the flux block SPD and the pressure Schur complement negative definite)
      if (r == c && r < S && sep_idx[(size_t)q * S + r] < 0) v = (r < Sf) ? 1.0 : -1.0;
      Fq[e] = v;
    }
    return;
  }
  const int* mp = cmap + ((size_t)slot * m + q) * K;
  const int* ck = ckind + ((size_t)slot * m + q) * 3;
  const int kind = ck[0], idx = ck[1], npr = ck[2];
  if (kind == 2) return;   // no child in this slot
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

// Compact per-node solve layout (see coarse_nd.py): info[q] = {s, b, sep_ptr,
// bnd_ptr, cb_off}; node data at data_off[q]: F11inv (s x s), X (b x s) over the
// whole boundary (flux dofs and pressures, indices into the combined vector),
// then X^T (s x b).

// (Vectors written by the PDL predecessor -- r, v, rs, cbuf, ybuf -- carry no __restrict__:
// their loads follow pdl_wait() inside the kernel's own lifetime and must be ordinary
// global loads, never the non-coherent path.)
// Coarse right-hand side entry g: r[g], or (cown != NULL, the preconditioner's
// restriction) v[own+] - v[own-] for flux dofs and 0 for pressures (coarse.py:225-235
// with a zero pressure load), so no assembled rhs vector is written.
__device__ __forceinline__ double nd_rhs(const double* r, const double* v,
                                         const int* __restrict__ cown, int nfc, int g) {
  if (!cown) return r[g];
  return g < nfc ? v[cown[2 * g]] - v[cown[2 * g + 1]] : 0.0;
}

// Forward gather (left-looking), 8 lanes per separator entry of the level:
// rs[t] = r[g_t] - sum of the descendants' update entries (lane-strided over the
// list, fixed shuffle tree: deterministic).
__global__ void nd_gather_kernel(int n, const int* __restrict__ sep_flat, const int* __restrict__ lptr,
                                 const int* __restrict__ lsrc, const double* cbuf, const double* r, const double* v,
                                 const int* __restrict__ cown, int nfc, double* __restrict__ rs) {
  pdl_trigger();
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = gt >> 3, sub = gt & 7;
  int p = 0, p1 = 0, g = 0;
  if (t < n) {
    p = lptr[t] + sub;
    p1 = lptr[t + 1];
    g = sep_flat[t];
  }
  pdl_wait();
  double acc = 0.0;
  for (; p < p1; p += 8) acc += cbuf[lsrc[p]];
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  if (t < n && sub == 0) rs[t] = nd_rhs(r, v, cown, nfc, g) - acc;
}

// Forward GEMV, task = rows [row0, row1) of one node, 4 rows per warp pass:
// rows < s: y = F11inv r_sep; rows s..s+bf-1: c = X r_sep into cbuf.
// lpe > 0: the task gathers r_sep itself, lpe lanes per separator entry (small
// separators: saves the separate gather launch); lpe == 0: r_sep from rs.
__global__ void nd_fwd_kernel(const int* __restrict__ tasks, const int* __restrict__ info,
                              const long long* __restrict__ data_off, const int* __restrict__ sep_flat,
                              const int* __restrict__ lptr, const int* __restrict__ lsrc,
                              const double* __restrict__ Fc, const double* r,
                              const double* v, const int* __restrict__ cown, int nfc,
                              const double* rs, double* __restrict__ ybuf, double* __restrict__ cbuf,
                              int lpe, double* __restrict__ xdirect) {
  extern __shared__ double rsm[];
  pdl_trigger();
  const int q = tasks[3 * blockIdx.x], row0 = tasks[3 * blockIdx.x + 1], row1 = tasks[3 * blockIdx.x + 2];
  const int s = info[6 * q], sp = info[6 * q + 2], cbo = info[6 * q + 4];
  const double* base = Fc + data_off[q];
  pdl_wait();
  if (lpe > 0) {
    const int per = blockDim.x / lpe, sub = threadIdx.x % lpe;
    for (int tb = 0; tb < s; tb += per) {
      const int t = tb + threadIdx.x / lpe;
      double acc = 0.0;
      if (t < s) {
        const int p1 = lptr[sp + t + 1];
        for (int p = lptr[sp + t] + sub; p < p1; p += lpe) acc += cbuf[lsrc[p]];
      }
      for (int o = lpe >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (t < s && sub == 0) rsm[t] = nd_rhs(r, v, cown, nfc, sep_flat[sp + t]) - acc;
    }
  } else {
    for (int k = threadIdx.x; k < s; k += blockDim.x) rsm[k] = rs[sp + k];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nq = (row1 - row0 + 3) / 4;
  int cs = 1;
  while (cs < 8 && 2 * cs * nq <= nw) cs *= 2;
  if (cs > 1) {
    // short task (long rows, few of them): cs warps split each row quad's columns,
    // partials combined in warp order (deterministic)
    __shared__ double part[8][4];
    const int qd = warp / cs, pc = warp % cs;
    const int chunk = ((s + cs - 1) / cs + 31) & ~31;
    const int c0 = imin(pc * chunk, s), c1 = imin(c0 + chunk, s);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (qd < nq) {
      const int row = row0 + 4 * qd;
      warp_rows4_dot(base + (size_t)row * s + c0, s, imin(4, row1 - row), rsm + c0, c1 - c0, lane, acc);
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) part[warp][k] = acc[k];
    }
    __syncthreads();
    if (threadIdx.x < 4 * nq) {
      const int qd2 = threadIdx.x >> 2, k = threadIdx.x & 3;
      const int rr = row0 + 4 * qd2 + k;
      if (rr < row1) {
        double v = 0.0;
        for (int u = 0; u < cs; ++u) v += part[qd2 * cs + u][k];
        if (rr < s) {
          if (xdirect) xdirect[sep_flat[sp + rr]] = v;
          else ybuf[sp + rr] = v;
        } else {
          cbuf[cbo + rr - s] = v;
        }
      }
    }
    return;
  }
  for (int row = row0 + 4 * warp; row < row1; row += 4 * nw) {
    const int nr = imin(4, row1 - row);
    double acc[4];
    warp_rows4_dot(base + (size_t)row * s, s, nr, rsm, s, lane, acc);
    if (lane < nr) {
      const double v = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
      const int rr = row + lane;
      if (rr < s) {
        // a node without boundary (the root) is final after the forward sweep
        if (xdirect) xdirect[sep_flat[sp + rr]] = v;
        else ybuf[sp + rr] = v;
      } else {
        cbuf[cbo + rr - s] = v;
      }
    }
  }
}

// Backward, task = separator rows [k0, k1) of one node; wpr warps per row
// split the row's columns, partials combined in fixed order:
// x_sep = y - X^T x_bnd with X^T stored row-major (s x b) after X.
__global__ void nd_bwd_kernel(const int* __restrict__ tasks, const int* __restrict__ info,
                              const long long* __restrict__ data_off, const int* __restrict__ sep_flat,
                              const int* __restrict__ bnd_flat, const double* __restrict__ Fc,
                              const double* ybuf, double* __restrict__ x, int wpr) {
  extern __shared__ double xb[];  // bmax
  __shared__ double part[8];
  pdl_trigger();
  const int q = tasks[3 * blockIdx.x], k0 = tasks[3 * blockIdx.x + 1], k1 = tasks[3 * blockIdx.x + 2];
  const int s = info[6 * q], b = info[6 * q + 1], sp = info[6 * q + 2], bp = info[6 * q + 3];
  pdl_wait();
  for (int m = threadIdx.x; m < b; m += blockDim.x) xb[m] = x[bnd_flat[bp + m]];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* XT = Fc + data_off[q] + (size_t)s * s + (size_t)b * s;
  if (wpr == 1) {
    for (int k = k0 + 4 * warp; k < k1; k += 4 * nw) {
      const int nr = imin(4, k1 - k);
      double acc[4];
      warp_rows4_dot(XT + (size_t)k * b, b, nr, xb, b, lane, acc);
      if (lane < nr) {
        const double v = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
        x[sep_flat[sp + k + lane]] = ybuf[sp + k + lane] - v;
      }
    }
    return;
  }
  const int rpc = nw / wpr;                 // rows per pass
  const int rl = warp / wpr, pc = warp % wpr;
  const int chunk = ((b + wpr - 1) / wpr + 31) & ~31;
  const int c0 = imin(pc * chunk, b), c1 = imin(c0 + chunk, b);
  for (int kb = k0; kb < k1; kb += rpc) {
    const int k = kb + rl;
    double acc = 0.0;
    if (k < k1) acc = warp_row_dot(XT + (size_t)k * b + c0, xb + c0, c1 - c0, lane);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (threadIdx.x < rpc && kb + threadIdx.x < k1) {
      double t = 0.0;
      for (int u = 0; u < wpr; ++u) t += part[threadIdx.x * wpr + u];
      const int kk = kb + threadIdx.x;
      x[sep_flat[sp + kk]] = ybuf[sp + kk] - t;
    }
    __syncthreads();
  }
}

// Copy the padded fronts' F11inv and X blocks into the compact layout
// (F11inv s x s, X b x s, X^T s x b); live pivot entry k sits at padded position
// k (flux, k < s_f) or Sf + k - s_f (eliminated pressure).
__global__ void nd_compact_kernel(int S, int Sf, int nf, int B, const double* __restrict__ F,
                                  const double* __restrict__ X, const int* __restrict__ info,
                                  const long long* __restrict__ data_off, double* __restrict__ Fc) {
  const int q = blockIdx.y;
  const int s = info[6 * q], b = info[6 * q + 1], sf = info[6 * q + 5];
  double* out = Fc + data_off[q];
  const long long ss = (long long)s * s, bs = (long long)b * s;
  const long long tot = ss + 2 * bs;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    if (e < ss) {
      int rr = (int)(e / s), cc = (int)(e % s);
      rr = rr < sf ? rr : Sf + rr - sf;
      cc = cc < sf ? cc : Sf + cc - sf;
      out[e] = F[(size_t)q * nf * nf + (size_t)rr * nf + cc];
    } else if (e < ss + bs) {
      long long e2 = e - ss;
      int j = (int)(e2 / s), cc = (int)(e2 % s);
      cc = cc < sf ? cc : Sf + cc - sf;
      out[e] = X[(size_t)q * B * S + (size_t)j * S + cc];
    } else {
      long long e2 = e - ss - bs;
      int k = (int)(e2 / b), j = (int)(e2 % b);
      k = k < sf ? k : Sf + k - sf;
      out[e] = X[(size_t)q * B * S + (size_t)j * S + k];
    }
  }
}

// Quasi-definite pivot block helpers (batched over the m fronts of a level):
// mode 0: C <- -C on the pressure block F[Sf:S, Sf:S];
// mode 1: F[0:Sf, Sf:S] <- F[Sf:S, 0:Sf]^T (mirror the off-diagonal block).
__global__ void nd_qd_kernel(int mode, int Sf, int Sp, int nf, double* __restrict__ F) {
  double* Fq = F + (size_t)blockIdx.y * nf * nf;
  const long long tot = mode == 0 ? (long long)Sp * Sp : (long long)Sf * Sp;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    if (mode == 0) {
      const int r = (int)(e / Sp), c = (int)(e % Sp);
      double* p = Fq + (size_t)(Sf + r) * nf + Sf + c;
      *p = -*p;
    } else {
      const int r = (int)(e / Sp), c = (int)(e % Sp);   // r < Sf, c < Sp
      Fq[(size_t)r * nf + Sf + c] = Fq[(size_t)(Sf + c) * nf + r];
    }
  }
}

__global__ void fill_kernel(long long n, double v, double* __restrict__ a) {
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) a[e] = v;
}

}  // namespace

extern "C" int bddc_nd_assemble(int m, int S, int Sf, int B, int nf, int slot, int K, const int* cmap, const int* ckind,
                                const int* sep_idx, double* F, const double* Fc, int Sc, int nfc, const double* Kc,
                                const int* sub_rows, const double* b0, int maxC, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (slot < 0 || slot == 0) {
    long long tot = (long long)nf * nf;
    dim3 g0((unsigned)imin((int)((tot + 255) / 256), 1024), m);
    nd_assemble_kernel<<<g0, 256, 0, s>>>(m, S, Sf, B, nf, -1, K, cmap, ckind, sep_idx, F, Fc, Sc, nfc, Kc, sub_rows,
                                          b0, maxC);
    LAUNCH_OK();
  }
  long long tot = (long long)K * K;
  dim3 g((unsigned)imin((int)((tot + 255) / 256), 1024), m);
  nd_assemble_kernel<<<g, 256, 0, s>>>(m, S, Sf, B, nf, slot, K, cmap, ckind, sep_idx, F, Fc, Sc, nfc, Kc, sub_rows, b0,
                                       maxC);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_nd_fwd(int ysize, int ntasks, int smax, const int* tasks, const int* info,
                           const long long* data_off, const int* sep_flat, const int* lptr, const int* lsrc,
                           const double* Fc, const double* r, const double* v, const int* cown, int nfc,
                           double* rsbuf, double* ybuf, double* cbuf, double* xdirect, void* stream) {
  if (ntasks <= 0 || ysize <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  // small separators: every task gathers its own r_sep (lanes per entry so one
  // pass covers the separator); large ones: a separate level-wide gather
  const int lpe = (smax <= 32 && ntasks <= 2 * ysize / (smax > 0 ? smax : 1)) ? 8 : 0;
  if (lpe == 0)
    PDL_LAUNCH(nd_gather_kernel, dim3((unsigned)(((long long)ysize * 8 + 255) / 256)), dim3(256), 0, st, ysize,
               sep_flat, lptr, lsrc, (const double*)cbuf, r, v, cown, nfc, rsbuf);
  size_t shm = (size_t)(smax > 0 ? smax : 1) * sizeof(double);
  if (shm > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(nd_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  PDL_LAUNCH(nd_fwd_kernel, dim3(ntasks), dim3(256), shm, st, tasks, info, data_off, sep_flat, lptr, lsrc, Fc, r,
             v, cown, nfc, (const double*)rsbuf, ybuf, cbuf, lpe, xdirect);
  return 0;
}

extern "C" int bddc_nd_bwd(int ntasks, int bfmax, int wpr, const int* tasks, const int* info,
                           const long long* data_off, const int* sep_flat, const int* bnd_flat, const double* Fc,
                           const double* ybuf, double* x, void* stream) {
  if (wpr != 1 && wpr != 2 && wpr != 4 && wpr != 8) return bddc_set_error(BDDC_ERR_ARG, "nd_bwd: wpr must be 1, 2, 4 or 8");
  if (ntasks <= 0) return 0;
  size_t shm = (size_t)(bfmax > 0 ? bfmax : 1) * sizeof(double);
  if (shm > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(nd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  PDL_LAUNCH(nd_bwd_kernel, dim3(ntasks), dim3(256), shm, (cudaStream_t)stream, tasks, info, data_off, sep_flat,
             bnd_flat, Fc, ybuf, x, wpr);
  return 0;
}

extern "C" int bddc_nd_compact(int m, int S, int Sf, int nf, int B, const double* F, const double* X,
                               const int* info, const long long* data_off, double* Fc, void* stream) {
  dim3 g(64, m);
  nd_compact_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(S, Sf, nf, B, F, X, info, data_off, Fc);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_nd_qd(int mode, int m, int Sf, int Sp, int nf, double* F, void* stream) {
  if (m <= 0 || Sp <= 0) return 0;
  dim3 g(64, m);
  nd_qd_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(mode, Sf, Sp, nf, F);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_fill(long long n, double v, double* a, void* stream) {
  if (n <= 0) return 0;
  CUDA_OK(launch_prio(fill_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, n, v, a));
  LAUNCH_OK();
  return 0;
}

