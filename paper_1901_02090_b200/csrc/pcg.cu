// Interface operator, BDDC preconditioner pieces, balanced projection and
// deterministic PCG vector kernels (solver.py:97-251).
//
// Interface vectors are "continuous" (indexed like dec.gamma) or "broken"
// (per subdomain slot, N x maxG).  Scatter = owner reads both copies in the
// fixed order low-subdomain + high-subdomain, which is the reference's
// np.add.at order (solver.py:100-101); every reduction is a fixed-shape tree,
// so repeated solves are bitwise identical (test_solver.py:165-173).
#include "common.cuh"

#define DOT_BLOCKS 296
#define DOT_THREADS 256

namespace {

// y_b[i][q] = sum_c M_i[q][c] * win[i][c] * x[gpos[i][c]]   (c < nG[i])
__global__ void gather_gemv_kernel(int maxG, const int* __restrict__ nG, const int* __restrict__ gpos,
                                   const double* __restrict__ Mats, const double* __restrict__ x,
                                   const double* __restrict__ win, double* __restrict__ yb) {
  extern __shared__ double xs[];
  const int i = blockIdx.x;
  const int n = nG[i];
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double v = x[gpos[(size_t)i * maxG + c]];
    if (win) v *= win[(size_t)i * maxG + c];
    xs[c] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* Mi = Mats + (size_t)i * maxG * maxG;
  for (int q = warp; q < n; q += nw) {
    const double* row = Mi + (size_t)q * maxG;
    double acc = 0.0;
    for (int c = lane; c < n; c += 32) acc += row[c] * xs[c];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) yb[(size_t)i * maxG + q] = acc;
  }
}

// ---------------------------------------------------------------------------
// Symmetric interface matrices (S_i, T_i) in tile-packed upper storage:
// 32x32 row-major tiles (bi <= bj), tile index t(bi,bj) = bi*nt - bi(bi-1)/2 + bj-bi,
// nt = maxG/32.  Only ceil(nG_i/32) block rows are live; this halves the bytes
// streamed per GEMV compared with full storage.


__global__ void pack_sym_kernel(int maxG, const double* __restrict__ full, double* __restrict__ packed) {
  const int i = blockIdx.y;
  const int nt = maxG / 32;
  const int ntiles = nt * (nt + 1) / 2;
  const double* F = full + (size_t)i * maxG * maxG;
  double* Pk = packed + (size_t)i * ntiles * 1024;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)ntiles * 1024;
       e += (long long)gridDim.x * blockDim.x) {
    int t = (int)(e / 1024), w = (int)(e % 1024);
    // invert tile index
    int bi = 0;
    while (bi + 1 < nt && tile_index(bi + 1, bi + 1, nt) <= t) ++bi;
    int bj = bi + (t - tile_index(bi, bi, nt));
    int r = bi * 32 + w / 32, c = bj * 32 + w % 32;
    // the upper triangle defines the matrix (diagonal tiles are stored full:
    // their lower half is mirrored, so callers may leave the lower triangle undefined)
    Pk[e] = (r <= c) ? F[(size_t)r * maxG + c] : F[(size_t)c * maxG + r];
  }
}

// y_b[i][q] = sum_c M_i[q][c] * win[i][c] * x[gpos[i][c]] from tile-packed symmetric M_i.
// Each warp streams whole tiles (coalesced rows), forms the column contribution in
// registers and the row contribution with a 31-shuffle transpose-reduction; per-tile
// partials are combined per output block in a fixed order (deterministic).
template <int MAXT, int G>
__global__ void __launch_bounds__(MAXT) gather_symv_kernel(int N, int maxG, const int* __restrict__ nG,
                                                         const int* __restrict__ gpos,
                                                         const double* __restrict__ packed,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ win, double* __restrict__ yb) {
  extern __shared__ double sm[];
  const int nt = maxG / 32;
  const int ntiles = nt * (nt + 1) / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // G groups of warps take G subdomains at a time (the grid-stride launch beside the
  // coarse chain, one CTA per SM: more subdomains, and loads, in flight per CTA)
  const int gw = (blockDim.x >> 5) / G, grp = warp / gw, wl = warp % gw;
  const int gt = threadIdx.x - grp * gw * 32, gthreads = gw * 32;
  double* xs = sm + (size_t)grp * (maxG + (size_t)ntiles * 64);   // maxG
  double* rowp = xs + maxG;                                        // ntiles x 32
  double* colp = rowp + (size_t)ntiles * 32;                       // ntiles x 32
  for (int i0 = blockIdx.x * G; i0 < N; i0 += gridDim.x * G) {
    const int i = i0 + grp;
    const bool act = i < N;
    const int n = act ? nG[i] : 0;
    const int ntl = (n + 31) / 32;
    __syncthreads();
    for (int c = gt; c < ntl * 32; c += gthreads) {
      double v = 0.0;
      if (c < n) {
        v = x[gpos[(size_t)i * maxG + c]];
        if (win) v *= win[(size_t)i * maxG + c];
      }
      xs[c] = v;
    }
    __syncthreads();
    const double* Pk = packed + (size_t)(act ? i : 0) * ntiles * 1024;
    const int nlive = ntl * (ntl + 1) / 2;
    for (int u = wl; u < nlive; u += gw) {
      // enumerate live tiles (bi <= bj < ntl) in row-major order
      int bi = 0, rem = u;
      while (rem >= ntl - bi) {
        rem -= ntl - bi;
        ++bi;
      }
      const int bj = bi + rem;
      const double* T = Pk + (size_t)tile_index(bi, bj, nt) * 1024;
      const double xl = xs[bj * 32 + lane];
      double v[32];
      double col = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const double a = ldg_stream(T + r * 32 + lane);   // once-read stream: no L1 allocation
        v[r] = a * xl;
        col += a * xs[bi * 32 + r];
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const bool up = lane & off;
#pragma unroll
        for (int k = 0; k < off; ++k) {
          double send = up ? v[k] : v[k + off];
          double recv = __shfl_xor_sync(0xffffffffu, send, off);
          v[k] = (up ? v[k + off] : v[k]) + recv;
        }
      }
      const int t = tile_index(bi, bj, nt);
      rowp[(size_t)t * 32 + lane] = v[0];
      colp[(size_t)t * 32 + lane] = (bi != bj) ? col : 0.0;
    }
    __syncthreads();
    for (int e = gt; e < ntl * 32; e += gthreads) {
      const int b = e / 32, l = e % 32;
      if (e >= n) continue;
      double acc = 0.0;
      for (int bj = b; bj < ntl; ++bj) acc += rowp[(size_t)tile_index(b, bj, nt) * 32 + l];
      for (int bi = 0; bi < b; ++bi) acc += colp[(size_t)tile_index(bi, b, nt) * 32 + l];
      yb[(size_t)i * maxG + e] = acc;
    }
  }
}

// Small subdomains (maxG <= 256, C4: <= 150 live slots): 16 x 16 tiles, so the
// packed bytes follow the live triangle closely (C4: 92 KB vs 123 KB with 32-tiles
// for the 81 KB algorithmic n(n+1)/2).  Each warp takes two tiles at a time, one
// per half-warp (lane = tile column): 16 coalesced 128-byte row loads per half,
// the row contribution by a 15-shuffle transposed reduction inside the half, the
// column contribution in registers; partials combined per output in fixed order.
__device__ __forceinline__ int tile_index16(int bi, int bj, int nt) { return bi * nt - (bi * (bi - 1)) / 2 + (bj - bi); }

__global__ void pack_sym16_kernel(int maxG, const double* __restrict__ full, double* __restrict__ packed) {
  const int i = blockIdx.y;
  const int nt = maxG / 16;
  const int ntiles = nt * (nt + 1) / 2;
  const double* F = full + (size_t)i * maxG * maxG;
  double* Pk = packed + (size_t)i * ntiles * 256;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)ntiles * 256;
       e += (long long)gridDim.x * blockDim.x) {
    int t = (int)(e / 256), w = (int)(e % 256);
    int bi = 0;
    while (bi + 1 < nt && tile_index16(bi + 1, bi + 1, nt) <= t) ++bi;
    int bj = bi + (t - tile_index16(bi, bi, nt));
    int r = bi * 16 + w / 16, c = bj * 16 + w % 16;
    Pk[e] = (r <= c) ? F[(size_t)r * maxG + c] : F[(size_t)c * maxG + r];
  }
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT) gather_symv16_kernel(int N, int maxG, const int* __restrict__ nG,
                                                           const int* __restrict__ gpos,
                                                           const double* __restrict__ packed,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ win, double* __restrict__ yb) {
  extern __shared__ double sm[];
  for (int i = blockIdx.x; i < N; i += gridDim.x) {
    const int n = nG[i];
    const int nt = maxG / 16;
    const int ntl = (n + 15) / 16;
    const int ntiles = nt * (nt + 1) / 2;
    double* xs = sm;                         // maxG
    double* rowp = xs + maxG;                // ntiles x 16
    double* colp = rowp + (size_t)ntiles * 16;
    __syncthreads();
    for (int c = threadIdx.x; c < ntl * 16; c += blockDim.x) {
      double v = 0.0;
      if (c < n) {
        v = x[gpos[(size_t)i * maxG + c]];
        if (win) v *= win[(size_t)i * maxG + c];
      }
      xs[c] = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int h = lane >> 4, l = lane & 15;
    const double* Pk = packed + (size_t)i * ntiles * 256;
    const int nlive = ntl * (ntl + 1) / 2;
    for (int u0 = 2 * warp; u0 < nlive; u0 += 2 * nw) {
      const int u = u0 + h;
      const bool act = u < nlive;
      int bi = 0, rem = act ? u : 0;
      while (rem >= ntl - bi) {
        rem -= ntl - bi;
        ++bi;
      }
      const int bj = bi + rem;
      const double* T = Pk + (size_t)tile_index16(bi, bj, nt) * 256;
      const double xl = xs[bj * 16 + l];
      double v[16];
      double col = 0.0;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const double a = act ? ldg_stream(T + r * 16 + l) : 0.0;
        v[r] = a * xl;
        col += a * xs[bi * 16 + r];
      }
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) {
        const bool up = l & off;
#pragma unroll
        for (int k = 0; k < off; ++k) {
          const double send = up ? v[k] : v[k + off];
          const double recv = __shfl_xor_sync(0xffffffffu, send, off);
          v[k] = (up ? v[k + off] : v[k]) + recv;
        }
      }
      if (act) {
        const int t = tile_index16(bi, bj, nt);
        rowp[(size_t)t * 16 + l] = v[0];
        colp[(size_t)t * 16 + l] = (bi != bj) ? col : 0.0;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ntl * 16; e += blockDim.x) {
      const int b = e / 16, ll = e % 16;
      if (e >= n) continue;
      double acc = 0.0;
      for (int bj = b; bj < ntl; ++bj) acc += rowp[(size_t)tile_index16(b, bj, nt) * 16 + ll];
      for (int bi = 0; bi < b; ++bi) acc += colp[(size_t)tile_index16(bi, b, nt) * 16 + ll];
      yb[(size_t)i * maxG + e] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent bulk-streamed symmetric GEMV (the interface operator S_i and the
// preconditioner's T_i, solver.py:103-107 / coarse.py:237-245).
//
// One CTA per SM; subdomains are handed out by a global ticket counter.  Warp
// roles (mbarrier-synchronised, no CTA-wide barrier after the prologue):
//   gather   takes the ticket, stages win . x of the subdomain's interface
//            slots into one of two x buffers (runs one subdomain ahead) and the
//            subdomain's tile issue order;
//   issuer   streams the subdomain's live packed 32x32 tiles with
//            cp.async.bulk (TMA engine, no register staging) into a ring of
//            SB_NST slots, issue slot j = 8k + c carrying the k-th tile of
//            chunk c (the live tiles in row-major order cut into 8 contiguous
//            chunks);
//   8 consumers: issue slot G (counted across subdomains) goes to warp G % 8
//            through ring slot G % SB_NST, so every ring slot has one consumer
//            warp and its mbarrier phases are consumed in order; a warp walks its
//            chunk keeping the row contributions lane-partial in registers while
//            the chunk stays in one tile row (one transposed reduction per row
//            run), and adds the column contributions of off-diagonal tiles to the
//            chunk's accumulator;
//   epilogue sums the eight chunk accumulators in chunk order, writes y and
//            frees the buffer.
// Consumers never wait at subdomain boundaries; 128 KB of tiles are in flight
// per SM, so a grid of fewer CTAs than SMs still saturates HBM and leaves SMs to
// a concurrent coarse chain.  Results do not depend on which CTA takes which
// subdomain (bitwise reproducible).
#define SB_NCW 8
#define SB_NST 16
#define SB_THREADS (32 * (SB_NCW + 3))
#define SB_ISSUER SB_NCW
#define SB_GATHER (SB_NCW + 1)
#define SB_EPI (SB_NCW + 2)
#define SB_TMAX 136   // live tiles of a 512-slot subdomain (16 * 17 / 2)

// lane l returns sum over lanes of v[l] (31-shuffle transposed reduction; v is consumed)
__device__ __forceinline__ double lane_transpose_sum(double (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = lane & off;
#pragma unroll
    for (int k = 0; k < off; ++k) {
      double send = up ? v[k] : v[k + off];
      double recv = __shfl_xor_sync(0xffffffffu, send, off);
      v[k] = (up ? v[k + off] : v[k]) + recv;
    }
  }
  return v[0];
}

// advance (bi, bj) by `steps` positions in the row-major order of the live upper
// triangle (bi <= bj < ntl)
__device__ __forceinline__ void tri_advance(int& bi, int& bj, int ntl, int steps) {
  for (int s = 0; s < steps; ++s) {
    if (++bj == ntl) {
      ++bi;
      bj = bi;
    }
  }
}

__global__ void __launch_bounds__(SB_THREADS, 1)
symv_bulk_kernel(int N, int maxG, const int* __restrict__ nG, const int* __restrict__ gpos,
                 const double* __restrict__ packed, const double* __restrict__ x,
                 const double* __restrict__ win, double* __restrict__ yb, int* __restrict__ sched) {
  extern __shared__ __align__(128) unsigned char smraw[];
  pdl_trigger();   // the dependent small kernel waits resident instead of paying a launch
  const int nt = maxG / 32;
  const size_t ntiles = (size_t)nt * (nt + 1) / 2;
  double* ring = reinterpret_cast<double*>(smraw);    // SB_NST tiles
  double* xs = ring + SB_NST * 1024;                   // 2 x maxG  (per subdomain buffer b)
  double* yw = xs + 2 * maxG;                          // 2 x SB_NCW x maxG accumulators
  uint64_t* full = reinterpret_cast<uint64_t*>(yw + 2 * SB_NCW * maxG);
  uint64_t* empty = full + SB_NST;
  uint64_t* xfull = empty + SB_NST;   // [2] x staged (gather -> issuer, consumers, epilogue)
  uint64_t* xfree = xfull + 2;        // [2] buffer released (epilogue -> gather)
  uint64_t* ydone = xfree + 2;        // [2] accumulators complete (consumers -> epilogue)
  int* meta = reinterpret_cast<int*>(ydone + 2);
  int* toff = meta + 2;               // [2][SB_TMAX] packed tile index per issue slot
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SB_NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(xfull + b, 32);
      mbar_init(xfree + b, 32);
      mbar_init(ydone + b, SB_NCW);
    }
    mbar_fence_init();
  }
  for (int e = threadIdx.x; e < 2 * SB_NCW * maxG; e += blockDim.x) yw[e] = 0.0;
  __syncthreads();
  if (warp == SB_GATHER) {
    for (int k = 0;; ++k) {
      const int b = k & 1;
      mbar_wait(xfree + b, ((k >> 1) & 1) ^ 1);
      int i = 0;
      if (lane == 0) i = atomicAdd(sched, 1);
      i = __shfl_sync(FULL, i, 0);
      if (i >= N) {
        if (lane == 0) meta[b] = -1;
        __syncwarp();
        mbar_arrive(xfull + b);
        break;
      }
      const int n = nG[i];
      const int ntl = (n + 31) / 32;
      double* xb = xs + b * maxG;
      int gp[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = lane + 32 * u;
        gp[u] = (u < ntl && c < n) ? gpos[(size_t)i * maxG + c] : -1;
      }
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = gp[u] >= 0 ? x[gp[u]] : 0.0;
      if (win) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (gp[u] >= 0) v[u] *= win[(size_t)i * maxG + lane + 32 * u];
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (u < ntl) xb[lane + 32 * u] = v[u];
      // issue order j -> class c = j % 8 (its consumer warp), k = j / 8: the k-th
      // tile of class c's contiguous chunk of the row-major live tiles
      {
        const int T = ntl * (ntl + 1) / 2;
        const int q = T / SB_NCW, rm = T % SB_NCW;
        for (int j = lane; j < T; j += 32) {
          const int c = j % SB_NCW;
          int u = c * q + imin(c, rm) + j / SB_NCW;
          int bi = 0;
          while (u >= ntl - bi) {
            u -= ntl - bi;
            ++bi;
          }
          toff[b * SB_TMAX + j] = tile_index(bi, bi + u, nt);
        }
      }
      if (lane == 0) meta[b] = i;
      __syncwarp();
      mbar_arrive(xfull + b);
    }
    if (lane == 0) {
      // the last CTA to finish re-arms the ticket counter for the next launch
      __threadfence();
      if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
        atomicExch(sched, 0);
        atomicExch(sched + 1, 0);
      }
    }
  } else if (warp == SB_ISSUER) {
    if (lane == 0) {
      unsigned G = 0;
      for (int k = 0;; ++k) {
        const int b = k & 1;
        mbar_wait(xfull + b, (k >> 1) & 1);
        const int i = meta[b];
        if (i < 0) break;
        const int ntl = (nG[i] + 31) / 32;
        const int T = ntl * (ntl + 1) / 2;
        const double* Pk = packed + (size_t)i * ntiles * 1024;
        const int* to = toff + b * SB_TMAX;
        for (int j = 0; j < T; ++j, ++G) {
          const unsigned slot = G % SB_NST;
          mbar_wait(empty + slot, ((G / SB_NST) & 1) ^ 1);
          mbar_arrive_expect_tx(full + slot, 8192u);
          bulk_g2s(ring + slot * 1024, Pk + (size_t)to[j] * 1024, 8192u, full + slot);
        }
      }
    }
  } else if (warp == SB_EPI) {
    for (int k = 0;; ++k) {
      const int b = k & 1;
      mbar_wait(xfull + b, (k >> 1) & 1);
      const int i = meta[b];
      if (i < 0) break;
      const int n = nG[i];
      const int ntl = (n + 31) / 32;
      mbar_wait(ydone + b, (k >> 1) & 1);
      double* yk = yw + (size_t)b * SB_NCW * maxG;
      for (int e = lane; e < ntl * 32; e += 32) {
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < SB_NCW; ++w) {
          acc += yk[w * maxG + e];
          yk[w * maxG + e] = 0.0;
        }
        if (e < n) yb[(size_t)i * maxG + e] = acc;
      }
      __syncwarp();
      mbar_arrive(xfree + b);
    }
  } else {
    // ------------------------------------------------------------ consumers
    unsigned G = 0;   // CTA-wide index of the first tile of the current subdomain
    for (int k = 0;; ++k) {
      const int b = k & 1;
      mbar_wait(xfull + b, (k >> 1) & 1);
      const int i = meta[b];
      if (i < 0) break;
      const int ntl = (nG[i] + 31) / 32;
      const int T = ntl * (ntl + 1) / 2;
      const double* xb = xs + b * maxG;
      const int c = (int)((warp - G % SB_NCW + SB_NCW) % SB_NCW);
      // class c (subdomain-local, not the warp) owns a contiguous chunk of the
      // row-major live tiles and its own accumulator: the summation grouping is
      // independent of the CTA's history (deterministic)
      double* myy = yw + ((size_t)b * SB_NCW + c) * maxG;
      const int q = T / SB_NCW, rm = T % SB_NCW;
      const int len = q + (c < rm ? 1 : 0);
      int bi = 0, bj = 0;
      {
        int u = c * q + imin(c, rm);
        while (u >= ntl - bi) {
          u -= ntl - bi;
          ++bi;
        }
        bj = bi + u;
      }
      // row contributions stay lane-partial (v[r] over this lane's column) while
      // the chunk walks one tile row; one transposed reduction per row run
      double v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = 0.0;
      int cur = bi;
      for (int k = 0; k < len; ++k) {
        if (bi != cur) {
          myy[cur * 32 + lane] += lane_transpose_sum(v, lane);
#pragma unroll
          for (int r = 0; r < 32; ++r) v[r] = 0.0;
          cur = bi;
        }
        const unsigned g = G + (unsigned)(k * SB_NCW + c);
        const unsigned slot = g % SB_NST;
        mbar_wait(full + slot, (g / SB_NST) & 1);
        const double* Tt = ring + slot * 1024;
        const double* xr = xb + bi * 32;
        const double xl = xb[bj * 32 + lane];
        double cs0 = 0.0, cs1 = 0.0, cs2 = 0.0, cs3 = 0.0;
#pragma unroll
        for (int r = 0; r < 32; r += 4) {
          const double a0 = Tt[r * 32 + lane], a1 = Tt[(r + 1) * 32 + lane];
          const double a2 = Tt[(r + 2) * 32 + lane], a3 = Tt[(r + 3) * 32 + lane];
          v[r] = fma(a0, xl, v[r]);
          v[r + 1] = fma(a1, xl, v[r + 1]);
          v[r + 2] = fma(a2, xl, v[r + 2]);
          v[r + 3] = fma(a3, xl, v[r + 3]);
          cs0 = fma(a0, xr[r], cs0);
          cs1 = fma(a1, xr[r + 1], cs1);
          cs2 = fma(a2, xr[r + 2], cs2);
          cs3 = fma(a3, xr[r + 3], cs3);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
        // off the diagonal the tile also acts transposed (diagonal tiles are stored full)
        if (bi != bj) myy[bj * 32 + lane] += (cs0 + cs1) + (cs2 + cs3);
        tri_advance(bi, bj, ntl, 1);
      }
      if (len > 0) myy[cur * 32 + lane] += lane_transpose_sum(v, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(ydone + b);
      G += T;
    }
  }
}

// v[i][r] = sum_q PsiT[i][r][q] * win[i][q] * x[gpos[i][q]]   (warp per coarse row r)
__global__ void gather_gemv_t_kernel(int maxG, int maxC, const int* __restrict__ nG, const int* __restrict__ nC,
                                     const int* __restrict__ gpos, const double* __restrict__ PsiT,
                                     const double* __restrict__ x, const double* __restrict__ win,
                                     double* __restrict__ v) {
  extern __shared__ double xs[];
  const int i = blockIdx.x;
  const int n = nG[i], nc = nC[i];
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double t = x[gpos[(size_t)i * maxG + c]];
    if (win) t *= win[(size_t)i * maxG + c];
    xs[c] = t;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* Pi = PsiT + (size_t)i * maxC * maxG;
  // four coarse rows per warp pass (16 loads per lane in flight)
  for (int r = 4 * warp; r < maxC; r += 4 * nw) {
    const int nr = imax(0, imin(4, nc - r));
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (nr > 0) warp_rows4_dot(Pi + (size_t)r * maxG, maxG, nr, xs, n, lane, acc);
    if (lane < 4 && r + lane < maxC) {
      const double t = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
      v[(size_t)i * maxC + r + lane] = (lane < nr) ? t : 0.0;
    }
  }
}

// rhs[g] = v[lo] - v[hi]  (sigma = +1 lower owner, -1 upper owner)
__global__ void coarse_restrict_kernel(int nfc, const int* __restrict__ cown, const double* __restrict__ v,
                                       double* __restrict__ rhs) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nfc) return;
  rhs[g] = v[cown[2 * g]] - v[cown[2 * g + 1]];
}

// out_b[i][q] = wout[i][q] * (y_b[i][q] + sum_r PsiT[i][r][q] sigma_r xc[g_r]).
// The live rows of PsiT_i stream through shared memory in double-buffered
// chunks of PRO_RB rows by cp.async (all copies of a chunk in flight at once);
// thread per slot q reads its column from shared memory.
#define PRO_RB 8
#define PRO_QPT 4   // slots per thread: maxG <= 4 * blockDim
template <bool al16>
__global__ void __launch_bounds__(256) prolong_kernel(int maxG, int maxC, const int* __restrict__ nG,
                                                      const int* __restrict__ nC, const int* __restrict__ sub_rows,
                                                      const double* __restrict__ PsiT, const double* __restrict__ xc,
                                                      const double* __restrict__ yb, const double* __restrict__ wout,
                                                      double* __restrict__ outb) {
  extern __shared__ __align__(16) double psm[];
  const int i = blockIdx.x;
  const int n = nG[i], nc = nC[i];
  const int cpad = (maxC + 1) & ~1;
  const int ldt = al16 ? ((n + 1) & ~1) : n;
  double* cf = psm;
  double* tile = psm + cpad;
  for (int r = threadIdx.x; r < nc; r += blockDim.x) {
    const int* sr = sub_rows + ((size_t)i * maxC + r) * 4;
    cf[r] = (double)sr[3] * xc[sr[0]];
  }
  const double* Pi = PsiT + (size_t)i * maxC * maxG;
  const int nch = (nc + PRO_RB - 1) / PRO_RB;
  auto issue = [&](int c) {
    const int r0 = c * PRO_RB, rows = imin(PRO_RB, nc - r0);
    double* dst = tile + (size_t)(c & 1) * PRO_RB * ldt;
    if (al16) {
      const int pr = ldt / 2;
      for (int e = threadIdx.x; e < rows * pr; e += blockDim.x) {
        const int rr = e / pr, pp = e - rr * pr;
        cp_async16(dst + rr * ldt + 2 * pp, Pi + (size_t)(r0 + rr) * maxG + 2 * pp, 16);
      }
    } else {
      for (int e = threadIdx.x; e < rows * ldt; e += blockDim.x) {
        const int rr = e / ldt, q = e - rr * ldt;
        cp_async8(dst + rr * ldt + q, Pi + (size_t)(r0 + rr) * maxG + q, 8);
      }
    }
    cp_async_commit();
  };
  double acc[PRO_QPT];
#pragma unroll
  for (int k = 0; k < PRO_QPT; ++k) acc[k] = 0.0;
  if (nch > 0) issue(0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* tb = tile + (size_t)(c & 1) * PRO_RB * ldt;
    const int r0 = c * PRO_RB, rows = imin(PRO_RB, nc - r0);
    for (int rr = 0; rr < rows; ++rr) {
      const double w = cf[r0 + rr];
#pragma unroll
      for (int k = 0; k < PRO_QPT; ++k) {
        const int q = threadIdx.x + k * blockDim.x;
        if (q < n) acc[k] += tb[rr * ldt + q] * w;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < PRO_QPT; ++k) {
    const int q = threadIdx.x + k * blockDim.x;
    if (q < n) {
      const size_t s = (size_t)i * maxG + q;
      const double w = yb ? yb[s] + acc[k] : acc[k];
      outb[s] = wout ? wout[s] * w : w;
    }
  }
}

// Same product without shared-memory staging: thread per slot q (QPT slots per
// thread), the live rows of PsiT_i streamed straight from HBM, 8 rows per batch so
// 8*QPT independent coalesced loads per thread are in flight; only the coarse
// coefficients live in shared memory (more CTAs per SM than the staged variant).
template <int QPT>
__global__ void __launch_bounds__(256) prolong_direct_kernel(int maxG, int maxC, const int* __restrict__ nG,
                                                             const int* __restrict__ nC,
                                                             const int* __restrict__ sub_rows,
                                                             const double* __restrict__ PsiT,
                                                             const double* __restrict__ xc,
                                                             const double* __restrict__ yb,
                                                             const double* __restrict__ wout,
                                                             double* __restrict__ outb) {
  extern __shared__ double cf[];
  pdl_trigger();
  const int i = blockIdx.x;
  const int n = nG[i], nc = nC[i];
  for (int r = threadIdx.x; r < nc; r += blockDim.x) {
    const int* sr = sub_rows + ((size_t)i * maxC + r) * 4;
    cf[r] = (double)sr[3] * xc[sr[0]];
  }
  __syncthreads();
  const double* Pi = PsiT + (size_t)i * maxC * maxG;
  double acc[QPT];
#pragma unroll
  for (int k = 0; k < QPT; ++k) acc[k] = 0.0;
  int r = 0;
  for (; r + 8 <= nc; r += 8) {
    double m[8][QPT];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < QPT; ++k) {
        const int q = threadIdx.x + k * 256;
        m[u][k] = (q < n) ? ldg_stream(Pi + (size_t)(r + u) * maxG + q) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double w = cf[r + u];
#pragma unroll
      for (int k = 0; k < QPT; ++k) acc[k] += m[u][k] * w;
    }
  }
  for (; r < nc; ++r) {
    const double w = cf[r];
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int q = threadIdx.x + k * 256;
      if (q < n) acc[k] += ldg_stream(Pi + (size_t)r * maxG + q) * w;
    }
  }
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    const int q = threadIdx.x + k * 256;
    if (q < n) {
      const size_t s = (size_t)i * maxG + q;
      const double w = yb ? yb[s] + acc[k] : acc[k];
      outb[s] = wout ? wout[s] * w : w;
    }
  }
}

// y[d] = y_b[lo slot] + y_b[hi slot]
__global__ void scatter_kernel(int n_gamma, const int* __restrict__ gown, const double* __restrict__ yb,
                               double* __restrict__ y) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_gamma) return;
  y[d] = yb[gown[2 * d]] + yb[gown[2 * d + 1]];
}

// phi[i] = sum_q sign_q y[gpos[i][q]], sign = +1 on the high side of the box
// phi_i = sum over the interface slots of i of sign * y; gown != NULL: y is not
// assembled yet and is read from the per-slot values yb (y[g] = yb[own0] + yb[own1],
// the scatter fused away).
// (Vectors written by the stream predecessor carry no __restrict__ in the kernels that
// wait on it inside their own lifetime: their loads must not take the non-coherent path.)
__global__ void phi_kernel(int maxG, const int* __restrict__ nG, const int* __restrict__ gpos,
                           const int* __restrict__ gcode, const double* y, double* __restrict__ phi,
                           const int* __restrict__ gown, const double* yb) {
  __shared__ double red[32];
  pdl_trigger();   // PCG chain: the next small kernel may become resident now
  pdl_wait();      // predecessor complete, its writes visible
  const int i = blockIdx.x;
  double acc = 0.0;
  for (int q = threadIdx.x; q < nG[i]; q += blockDim.x) {
    size_t s = (size_t)i * maxG + q;
    const int g = gpos[s];
    double v = gown ? yb[gown[2 * g]] + yb[gown[2 * g + 1]] : y[g];
    acc += ((gcode[s] >> 2) & 1) ? v : -v;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) phi[i] = acc;
}

// Separable Laplacian solve on the S[0] x S[1] x S[2] subdomain grid:
// z = Dm (Qx (x) Qy (x) Qz) Lambda^+ (..)^T Dm phi  (Dm = D^{-1/2} or NULL).
// eig layout: [Qx (Sx*Sx) | Qy | Qz | lx (Sx) | ly | lz], Q row-major Q[a][a'].
__global__ void lap_solve_kernel(int S0, int S1, int S2, const double* __restrict__ eig,
                                 const double* __restrict__ dm, const double* __restrict__ phi,
                                 double* __restrict__ z) {
  extern __shared__ double sm[];
  const int N = S0 * S1 * S2;
  double* u = sm;
  double* w = u + N;
  double* es = w + N;   // eigen data staged in shared memory
  const int ne = S0 * S0 + S1 * S1 + S2 * S2 + S0 + S1 + S2;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) es[e] = eig[e];
  const double* Q[3] = {es, es + S0 * S0, es + S0 * S0 + S1 * S1};
  const double* lam = es + S0 * S0 + S1 * S1 + S2 * S2;
  const double* lx = lam;
  const double* ly = lam + S0;
  const double* lz = lam + S0 + S1;
  const int Sd[3] = {S0, S1, S2};
  const int st[3] = {1, S0, S0 * S1};
  for (int e = threadIdx.x; e < N; e += blockDim.x) u[e] = dm ? dm[e] * phi[e] : phi[e];
  __syncthreads();
  // forward: apply Q_a^T along every axis
  for (int a = 0; a < 3; ++a) {
    double* src = (a & 1) ? w : u;
    double* dst = (a & 1) ? u : w;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
      int ca = (e / st[a]) % Sd[a];
      int base = e - ca * st[a];
      double acc = 0.0;
      for (int k = 0; k < Sd[a]; ++k) acc += Q[a][k * Sd[a] + ca] * src[base + k * st[a]];
      dst[e] = acc;
    }
    __syncthreads();
  }
  // after 3 passes the data is in w
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    int a0 = e % S0, a1 = (e / S0) % S1, a2 = e / (S0 * S1);
    double l = lx[a0] + ly[a1] + lz[a2];
    w[e] = (l == 0.0) ? 0.0 : w[e] / l;   // Neumann null mode (exact 0); none with a Dirichlet axis
  }
  __syncthreads();
  for (int a = 0; a < 3; ++a) {
    double* src = (a & 1) ? u : w;
    double* dst = (a & 1) ? w : u;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
      int ca = (e / st[a]) % Sd[a];
      int base = e - ca * st[a];
      double acc = 0.0;
      for (int k = 0; k < Sd[a]; ++k) acc += Q[a][ca * Sd[a] + k] * src[base + k * st[a]];
      dst[e] = acc;
    }
    __syncthreads();
  }
  // result in u
  for (int e = threadIdx.x; e < N; e += blockDim.x) z[e] = dm ? dm[e] * u[e] : u[e];
}

// y[d] -= z[lo(d)] - z[hi(d)]   (Phi^T z with sign_lo = +1, sign_hi = -1)
__global__ void proj_apply_kernel(int n_gamma, int maxG, const int* __restrict__ gown, const double* __restrict__ z,
                                  double* __restrict__ y) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_gamma) return;
  int lo = gown[2 * d] / maxG, hi = gown[2 * d + 1] / maxG;
  y[d] -= z[lo] - z[hi];
}

// ------------------------------------------------------------- dot products

// Fused deterministic dot: per-block partials, the last block to finish sums
// them in index order and applies `op` (see bddc_dot).  MODE selects the
// elementwise pass that produces the reduced terms:
//   0  x . y  (op 200-299: sum |x|, op 300-399: max |x|, into slot op - 200 / - 300)
//   1  balanced projection then dot: y[d] -= z[lo(d)] - z[hi(d)] (solver.py:166-179),
//      acc += x[d] * y[d]  (the projected S p or M r and its dot with p or r)
//   2  CG update then residual norm: xv += alpha p, r -= alpha Ap (alpha = scal[2]),
//      acc += r . r   (solver.py:207-213)
struct DotArgs {
  const int* gown;
  int maxG;
  const double* z;     // MODE 1, 3: the subdomain Laplacian solve
  double* xv;          // MODE 2: iterate
  const double* p;     // MODE 2
  const double* Ap;    // MODE 2
  const double* yb;    // MODE 3: per-slot values, assembled on the fly
  // op 2 with cond != 0: the PCG WHILE node's condition is set by the reducing
  // block (relres > tol, no breakdown, it < maxit), no separate condition kernel
  unsigned long long cond;
  double tol;
  int maxit;
};

template <int MODE>
__global__ void dot_kernel(const double* x, double* y, long long n,
                           double* __restrict__ partial, unsigned* __restrict__ counter,
                           double* __restrict__ scal, int op, double* __restrict__ hist, DotArgs A) {
  __shared__ double red[32];
  __shared__ bool last;
  pdl_trigger();   // PCG chain: the next small kernel may become resident now
  pdl_wait();      // predecessor complete, its writes visible
  const bool amax = MODE == 0 && op >= 300 && op < 400, asum = MODE == 0 && op >= 200 && op < 300;
  double acc = 0.0;
  const double alpha = MODE == 2 ? scal[2] : 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    if (MODE == 1 || MODE == 3) {
      const int s0 = A.gown[2 * e], s1 = A.gown[2 * e + 1];
      const int lo = s0 / A.maxG, hi = s1 / A.maxG;
      const double v = (MODE == 3 ? A.yb[s0] + A.yb[s1] : y[e]) - (A.z[lo] - A.z[hi]);
      y[e] = v;
      acc += x[e] * v;
    } else if (MODE == 2) {
      A.xv[e] += alpha * A.p[e];
      const double v = y[e] - alpha * A.Ap[e];
      y[e] = v;
      acc += v * v;
    } else if (amax) {
      acc = fmax(acc, fabs(x[e]));
    } else if (asum) {
      acc += fabs(x[e]);
    } else {
      acc += x[e] * y[e];
    }
  }
  acc = amax ? block_max(acc, red) : block_sum(acc, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = acc;
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
    s = amax ? fmax(s, ((volatile double*)partial)[b]) : s + ((volatile double*)partial)[b];
  s = amax ? block_max(s, red) : block_sum(s, red);
  if (threadIdx.x == 0) {
    *counter = 0u;
    if (amax || asum) {
      scal[op - (amax ? 300 : 200)] = s;
      return;
    }
    // scal slots: 0 rz, 1 pAp, 2 alpha, 3 rr, 4 res0, 5 relres, 6 rz_new, 7 beta,
    // 8 bad (non-positive curvature), 9 iterations completed (device counter)
    const int itc = (int)scal[9];
    switch (op) {
      case 0:  // rz (initial)
        scal[0] = s;
        break;
      case 1: {  // pAp -> alpha, alphas[it]
        scal[1] = s;
        double a = scal[0] / s;
        if (!(s > 0.0)) scal[8] = 1.0;
        scal[2] = a;
        if (hist) hist[itc] = a;
        break;
      }
      case 2: {  // rr -> relres, it += 1, relres history[it]
        scal[3] = s;
        double rel = sqrt(s) / scal[4];
        scal[5] = rel;
        scal[9] = (double)(itc + 1);
        if (hist) hist[itc + 1] = rel;
        if (A.cond) {
          const bool go = !(rel <= A.tol) && scal[8] == 0.0 && itc + 1 < A.maxit;
          cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond, go ? 1u : 0u);
        }
        break;
      }
      case 3: {  // rz_new -> beta, betas[it-1]
        double b = s / scal[0];
        scal[6] = s;
        scal[7] = b;
        scal[0] = s;
        if (hist && itc >= 1) hist[itc - 1] = b;
        break;
      }
      case 4:  // res0 = ||r||, reset the counter, history[0] = 1
        scal[3] = s;
        scal[4] = sqrt(s);
        scal[5] = 1.0;
        scal[8] = 0.0;
        scal[9] = 0.0;
        if (hist) hist[0] = 1.0;
        break;
      default:  // plain store into slot (op - 100)
        scal[op - 100] = s;
    }
  }
}

// x += alpha p ; r -= alpha Ap
__global__ void cg_update_kernel(long long n, const double* __restrict__ scal, double* __restrict__ x,
                                 const double* __restrict__ p, double* __restrict__ r, const double* __restrict__ Ap) {
  const double a = scal[2];
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    x[e] += a * p[e];
    r[e] -= a * Ap[e];
  }
}

// p = z + beta p
__global__ void p_update_kernel(long long n, const double* scal, const double* z, double* p) {
  pdl_trigger();   // PCG chain: the next small kernel may become resident now
  pdl_wait();      // predecessor complete, its writes visible
  const double b = scal[7];
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    p[e] = z[e] + b * p[e];
}

// Dense (row-major, symmetric) GEMV y = M x over n rows, warp per row.
// y = M x, warp per row, 8 loads per lane in flight (fixed order: deterministic).
__global__ void gemv_kernel(int n, int ld, int ncol, const double* __restrict__ M, const double* x,
                            double* __restrict__ y) {
  pdl_trigger();   // PCG chain: the next small kernel may become resident now
  pdl_wait();      // predecessor complete, its writes visible
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n) return;
  const double* mr = M + (size_t)row * ld;
  double a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = 0.0;
  int c = lane;
  for (; c + 224 < ncol; c += 256) {
    double m[8], v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      m[u] = __ldg(mr + c + 32 * u);
      v[u] = x[c + 32 * u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] += m[u] * v[u];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (c + 32 * u < ncol) a[u] += __ldg(mr + c + 32 * u) * x[c + 32 * u];
  double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[row] = acc;
}

// y = M x with WPR warps per row (each a contiguous column chunk, partials summed
// in fixed order through shared memory: deterministic).  More warps per row keep
// more loads in flight when there are few rows (N x N projection operator).
template <int WPR>
__global__ void __launch_bounds__(256) gemv_split_kernel(int n, int ld, int ncol, const double* __restrict__ M,
                                                         const double* x, double* __restrict__ y) {
  __shared__ double part[8];
  pdl_trigger();   // PCG chain: the next small kernel may become resident now
  pdl_wait();      // predecessor complete, its writes visible
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * (8 / WPR) + w / WPR, pi = w % WPR;
  const int chunk = ((ncol + WPR * 32 - 1) / (WPR * 32)) * 32;
  const int c0 = pi * chunk, c1 = min(ncol, c0 + chunk);
  double acc = 0.0;
  if (row < n) {
    const double* mr = M + (size_t)row * ld;
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = 0.0;
    int c = c0 + lane;
    for (; c + 224 < c1; c += 256) {
      double m[8], v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        m[u] = __ldg(mr + c + 32 * u);
        v[u] = x[c + 32 * u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += m[u] * v[u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c + 32 * u < c1) a[u] += __ldg(mr + c + 32 * u) * x[c + 32 * u];
    acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  }
  if (lane == 0) part[w] = acc;
  __syncthreads();
  if (pi == 0 && lane == 0 && row < n) {
    double t = part[w];
    for (int q = 1; q < WPR; ++q) t += part[w + q];
    y[row] = t;
  }
}

// Dense pseudo-inverse of the separable subdomain-grid Laplacian (setup):
// W[e][f] = Qx[ex][fx] Qy[ey][fy] Qz[ez][fz] (spatial e, mode f), Ws = W Lambda^+.
__global__ void lap_kron_kernel(int S0, int S1, int S2, const double* __restrict__ eig, double* __restrict__ W,
                                double* __restrict__ Ws) {
  const int N = S0 * S1 * S2;
  const double* Qx = eig;
  const double* Qy = Qx + S0 * S0;
  const double* Qz = Qy + S1 * S1;
  const double* lx = Qz + S2 * S2;
  const double* ly = lx + S0;
  const double* lz = ly + S1;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)N * N;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t / N), f = (int)(t % N);
    const int ex = e % S0, ey = (e / S0) % S1, ez = e / (S0 * S1);
    const int fx = f % S0, fy = (f / S0) % S1, fz = f / (S0 * S1);
    const double w = Qx[ex * S0 + fx] * Qy[ey * S1 + fy] * Qz[ez * S2 + fz];
    const double lam = lx[fx] + ly[fy] + lz[fz];
    W[t] = w;
    Ws[t] = (lam == 0.0) ? 0.0 : w / lam;
  }
}

__global__ void scale_sym_kernel(int N, const double* __restrict__ dm, double* __restrict__ M) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)N * N;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t / N), f = (int)(t % N);
    M[t] *= dm[e] * dm[f];
  }
}

// Lanczos tridiagonal from CG coefficients (solver.py:236-251); kappa by
// Sturm bisection for the extreme eigenvalues.
__device__ int sturm_count(const double* d, const double* e2, int m, double x) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0) ++cnt;
  for (int k = 1; k < m; ++k) {
    if (q == 0.0) q = 1e-300;
    q = d[k] - x - e2[k - 1] / q;
    if (q < 0) ++cnt;
  }
  return cnt;
}

__global__ void lanczos_kernel(int m, const double* __restrict__ al, const double* __restrict__ be,
                               double* __restrict__ work, double* __restrict__ out) {
  double* d = work;
  double* e2 = work + m;
  if (threadIdx.x == 0) {
    d[0] = 1.0 / al[0];
    for (int k = 1; k < m; ++k) {
      d[k] = 1.0 / al[k] + be[k - 1] / al[k - 1];
      double o = sqrt(fmax(be[k - 1], 0.0)) / al[k - 1];
      e2[k - 1] = o * o;
    }
  }
  __syncthreads();
  {
    // warp 0: smallest eigenvalue (Sturm count >= 1), warp 1: largest (count >= m).
    // Multisection: the 32 lanes count at 32 interior points of the bracket at once,
    // so every pass shrinks it 33-fold (12 passes instead of ~60 dependent bisections).
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double lo = 1e308, hi = -1e308;
    for (int k = 0; k < m; ++k) {
      double r = 0.0;
      if (k > 0) r += sqrt(e2[k - 1]);
      if (k < m - 1) r += sqrt(e2[k]);
      lo = fmin(lo, d[k] - r);
      hi = fmax(hi, d[k] + r);
    }
    const int target = warp == 0 ? 1 : m;
    double a = lo, b = hi;
    for (int pass = 0; pass < 40; ++pass) {
      const double h = (b - a) / 33.0;
      if (!(h > 0.0) || a + h == a || b - h == b) break;
      const double x = a + (lane + 1) * h;
      const bool ge = sturm_count(d, e2, m, x) >= target;
      const unsigned mask = __ballot_sync(0xffffffffu, ge);
      const int first = mask ? __ffs(mask) - 1 : 32;   // counts are monotone in x
      const double nb = first < 32 ? a + (first + 1) * h : b;
      const double na = first > 0 ? a + first * h : a;
      a = na;
      b = nb;
    }
    if (lane == 0) out[warp] = 0.5 * (a + b);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double lmin = fmax(out[0], 2.2250738585072014e-308);
    out[2] = out[1] / lmin;
  }
}

// All eigenvalues of the symmetric tridiagonal (d, e) by bisection on Sturm
// counts: thread k brackets the (k+1)-th smallest one inside the Gershgorin
// interval (ascending output).
__global__ void tridiag_eigvals_kernel(int m, const double* __restrict__ d, const double* __restrict__ e,
                                       double* __restrict__ e2, double* __restrict__ out) {
  __shared__ double lohi[2];
  for (int k = threadIdx.x; k < m - 1; k += blockDim.x) e2[k] = e[k] * e[k];
  if (threadIdx.x == 0) {
    double lo = 1e308, hi = -1e308;
    for (int k = 0; k < m; ++k) {
      double r = 0.0;
      if (k > 0) r += fabs(e[k - 1]);
      if (k < m - 1) r += fabs(e[k]);
      lo = fmin(lo, d[k] - r);
      hi = fmax(hi, d[k] + r);
    }
    const double pad = 1e-14 * fmax(fabs(lo), fabs(hi)) + 1e-300;
    lohi[0] = lo - pad;
    lohi[1] = hi + pad;
  }
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double a = lohi[0], b = lohi[1];
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (a + b);
    if (mid == a || mid == b) break;
    if (sturm_count(d, e2, m, mid) >= k + 1) b = mid;
    else a = mid;
  }
  out[k] = 0.5 * (a + b);
}

// w[i] -= sum_j Q[j][i] c[j]  (Q: k rows of length n; j in order: deterministic)
__global__ void gemv_t_sub_kernel(int k, int n, const double* __restrict__ Q, const double* __restrict__ c,
                                  double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int j = 0; j < k; ++j) acc += Q[(size_t)j * n + i] * c[j];
  w[i] -= acc;
}

__global__ void axpby_kernel(long long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    y[e] = a * x[e] + (b == 0.0 ? 0.0 : b * y[e]);
}

}  // namespace

extern "C" int bddc_gather_gemv(int N, int maxG, const int* nG, const int* gpos, const double* Mats, const double* x,
                                const double* win, double* yb, void* stream) {
  gather_gemv_kernel<<<N, 256, maxG * sizeof(double), (cudaStream_t)stream>>>(maxG, nG, gpos, Mats, x, win, yb);
  LAUNCH_OK();
  return 0;
}

extern "C" size_t bddc_sym_packed_elems(int maxG) {
  int nt = maxG / 32;
  return (size_t)nt * (nt + 1) / 2 * 1024;
}

extern "C" size_t bddc_sym_packed16_elems(int maxG) {
  int nt = maxG / 16;
  return (size_t)nt * (nt + 1) / 2 * 256;
}
extern "C" int bddc_pack_sym16(int N, int maxG, const double* full, double* packed, void* stream) {
  if (maxG % 16) return bddc_set_error(BDDC_ERR_ARG, "pack_sym16: maxG must be a multiple of 16");
  dim3 g(64, N);
  pack_sym16_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(maxG, full, packed);
  LAUNCH_OK();
  return 0;
}
extern "C" int bddc_gather_symv16(int N, int maxG, const int* nG, const int* gpos, const double* packed,
                                  const double* x, const double* win, double* yb, int grid, void* stream) {
  if (maxG % 16) return bddc_set_error(BDDC_ERR_ARG, "gather_symv16: maxG must be a multiple of 16");
  const int nt = maxG / 16;
  const size_t shm = ((size_t)maxG + (size_t)nt * (nt + 1) * 16) * sizeof(double);
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(gather_symv16_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  if (grid <= 0 || grid > N) grid = N;
  gather_symv16_kernel<256><<<grid, 256, shm, (cudaStream_t)stream>>>(N, maxG, nG, gpos, packed, x, win, yb);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_pack_sym(int N, int maxG, const double* full, double* packed, void* stream) {
  if (maxG % 32) return bddc_set_error(BDDC_ERR_ARG, "pack_sym: maxG must be a multiple of 32");
  dim3 g(64, N);
  pack_sym_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(maxG, full, packed);
  LAUNCH_OK();
  return 0;
}

static int g_symv_threads = 256;
extern "C" void bddc_set_symv_threads(int t) { g_symv_threads = (t == 512) ? 512 : 256; }

static int g_symv_groups = 4;   // C4 precond beside the chain: 462 us (1), 430 (2), 426 (4)
extern "C" void bddc_set_symv_groups(int g) { g_symv_groups = (g == 1 || g == 2) ? g : 4; }

extern "C" int bddc_gather_symv(int N, int maxG, const int* nG, const int* gpos, const double* packed,
                                const double* x, const double* win, double* yb, int grid, void* stream) {
  int nt = maxG / 32;
  const size_t per = ((size_t)maxG + (size_t)nt * (nt + 1) * 32) * sizeof(double);
  if (grid <= 0 || grid > N) grid = N;
  // the grid-stride launch (T_i beside the coarse chain: one CTA per SM) takes
  // g_symv_groups subdomains at a time per CTA (more loads in flight per CTA)
  const int G = (grid < N) ? g_symv_groups : 1;
  const size_t shm = per * G;
  cudaStream_t s = (cudaStream_t)stream;
#define SYMV_CASE(T, GG)                                                                              \
  do {                                                                                                \
    if (shm > 48 * 1024)                                                                              \
      CUDA_OK(cudaFuncSetAttribute(gather_symv_kernel<T, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm)); \
    gather_symv_kernel<T, GG><<<grid, T, shm, s>>>(N, maxG, nG, gpos, packed, x, win, yb);            \
  } while (0)
  if (grid < N && g_symv_threads == 512) {
    if (G == 4) SYMV_CASE(512, 4);
    else if (G == 2) SYMV_CASE(512, 2);
    else SYMV_CASE(512, 1);
  } else {
    if (G == 4) SYMV_CASE(256, 4);
    else if (G == 2) SYMV_CASE(256, 2);
    else SYMV_CASE(256, 1);
  }
#undef SYMV_CASE
  LAUNCH_OK();
  return 0;
}

static size_t symv_bulk_smem(int maxG) {
  return (size_t)SB_NST * 8192 + (size_t)(2 + 2 * SB_NCW) * maxG * sizeof(double) +
         (2 * SB_NST + 6) * sizeof(uint64_t) + (2 + 2 * SB_TMAX) * sizeof(int);
}

// Persistent bulk-streamed variant: `grid` CTAs (<= 0: one per SM), `sched` two
// zero-initialised ints owned by this call site (re-armed by the kernel).
extern "C" int bddc_gather_symv_bulk(int N, int maxG, const int* nG, const int* gpos, const double* packed,
                                     const double* x, const double* win, double* yb, int grid, int* sched,
                                     void* stream) {
  if (maxG % 32 || maxG > 512) return bddc_set_error(BDDC_ERR_ARG, "gather_symv_bulk: maxG (multiple of 32, <= 512)");
  const size_t shm = symv_bulk_smem(maxG);
  static size_t configured = 0;
  if (shm > configured) {
    CUDA_OK(cudaFuncSetAttribute(symv_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    configured = shm;
  }
  if (grid <= 0) {
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, dev));
  }
  if (grid > N) grid = N;
  if (N == 0) return 0;
  CUDA_OK(launch_prio(symv_bulk_kernel, dim3(grid), dim3(SB_THREADS), shm, (cudaStream_t)stream, N, maxG, nG,
                      gpos, packed, x, win, yb, sched));
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_gather_gemv_t(int N, int maxG, int maxC, const int* nG, const int* nC, const int* gpos,
                                  const double* PsiT, const double* x, const double* win, double* v, void* stream) {
  CUDA_OK(launch_prio(gather_gemv_t_kernel, dim3(N), dim3(256), maxG * sizeof(double), (cudaStream_t)stream, maxG,
                      maxC, nG, nC, gpos, PsiT, x, win, v));
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_coarse_restrict(int nfc, const int* cown, const double* v, double* rhs, void* stream) {
  if (nfc <= 0) return 0;
  CUDA_OK(launch_prio(coarse_restrict_kernel, dim3((nfc + 255) / 256), dim3(256), 0, (cudaStream_t)stream, nfc, cown,
                      v, rhs));
  LAUNCH_OK();
  return 0;
}

static int g_prolong_direct = 1;
extern "C" void bddc_set_prolong_direct(int on) { g_prolong_direct = on ? 1 : 0; }

extern "C" int bddc_prolong(int N, int maxG, int maxC, const int* nG, const int* nC, const int* sub_rows,
                            const double* PsiT, const double* xc, const double* yb, const double* wout, double* outb,
                            void* stream) {
  if (maxG > PRO_QPT * 256) return bddc_set_error(BDDC_ERR_ARG, "prolong: maxG too large");
  if (g_prolong_direct) {
    cudaStream_t st = (cudaStream_t)stream;
    const size_t cshm = (size_t)maxC * sizeof(double);
    if (maxG <= 256)
      prolong_direct_kernel<1><<<N, 256, cshm, st>>>(maxG, maxC, nG, nC, sub_rows, PsiT, xc, yb, wout, outb);
    else if (maxG <= 512)
      prolong_direct_kernel<2><<<N, 256, cshm, st>>>(maxG, maxC, nG, nC, sub_rows, PsiT, xc, yb, wout, outb);
    else
      prolong_direct_kernel<4><<<N, 256, cshm, st>>>(maxG, maxC, nG, nC, sub_rows, PsiT, xc, yb, wout, outb);
    LAUNCH_OK();
    return 0;
  }
  const bool al = !(maxG & 1) && !(((uintptr_t)PsiT) & 15);
  const int ldt = al ? ((maxG + 1) & ~1) : maxG;
  size_t shm = ((size_t)((maxC + 1) & ~1) + 2 * (size_t)PRO_RB * ldt) * sizeof(double);
  if (al) {
    if (shm > 48 * 1024)
      CUDA_OK(cudaFuncSetAttribute(prolong_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    prolong_kernel<true><<<N, 256, shm, (cudaStream_t)stream>>>(maxG, maxC, nG, nC, sub_rows, PsiT, xc, yb, wout,
                                                                outb);
  } else {
    if (shm > 48 * 1024)
      CUDA_OK(cudaFuncSetAttribute(prolong_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    prolong_kernel<false><<<N, 256, shm, (cudaStream_t)stream>>>(maxG, maxC, nG, nC, sub_rows, PsiT, xc, yb, wout,
                                                                 outb);
  }
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_scatter(int n_gamma, const int* gown, const double* yb, double* y, void* stream) {
  if (n_gamma <= 0) return 0;
  scatter_kernel<<<(n_gamma + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n_gamma, gown, yb, y);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_phi(int N, int maxG, const int* nG, const int* gpos, const int* gcode, const double* y, double* phi,
                        void* stream) {
  phi_kernel<<<N, 256, 0, (cudaStream_t)stream>>>(maxG, nG, gpos, gcode, y, phi, nullptr, nullptr);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_phi_broken(int N, int maxG, const int* nG, const int* gpos, const int* gcode, const int* gown,
                               const double* yb, double* phi, void* stream) {
  PCG_LAUNCH(0, phi_kernel, dim3(N), dim3(256), 0, (cudaStream_t)stream, maxG, nG, gpos, gcode, (const double*)nullptr,
             phi, gown, yb);
  return 0;
}

// One mode product of the separable solve, thread per grid node (multi-CTA):
// out[e] = dmo[e] * (sum_k Q_a[.] * dmi[g] * in[g]) (/ Lambda if lamdiv); forward
// uses Q_a^T (Q[k][c]), backward Q_a (Q[c][k]).
__global__ void lap_mode_kernel(int S0, int S1, int S2, int a, int backward, const double* __restrict__ eig,
                                const double* __restrict__ dmi, const double* __restrict__ dmo, int lamdiv,
                                const double* in, double* __restrict__ out) {   // in: predecessor-written
  pdl_trigger();
  const int N = S0 * S1 * S2;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int Sd[3] = {S0, S1, S2};
  const int st[3] = {1, S0, S0 * S1};
  const double* Q = eig + (a == 0 ? 0 : (a == 1 ? S0 * S0 : S0 * S0 + S1 * S1));
  const double* lam = eig + S0 * S0 + S1 * S1 + S2 * S2;
  pdl_wait();
  if (e >= N) return;
  const int S = Sd[a], ca = (e / st[a]) % S, base = e - ca * st[a];
  double acc = 0.0;
  for (int k = 0; k < S; ++k) {
    const int g = base + k * st[a];
    const double v = dmi ? dmi[g] * in[g] : in[g];
    acc += (backward ? Q[ca * S + k] : Q[k * S + ca]) * v;
  }
  if (lamdiv) {
    const int a0 = e % S0, a1 = (e / S0) % S1, a2 = e / (S0 * S1);
    const double l = lam[a0] + lam[S0 + a1] + lam[S0 + S1 + a2];
    acc = (l == 0.0) ? 0.0 : acc / l;   // Neumann null mode only (exact 0)
  }
  out[e] = dmo ? dmo[e] * acc : acc;
}

extern "C" int bddc_lap_solve_mc(int S0, int S1, int S2, const double* eig, const double* dm, const double* phi,
                                 double* z, double* ws, void* stream) {
  const int N = S0 * S1 * S2;
  if (N <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  double* u = ws;
  double* w = ws + N;
  const dim3 g((N + 127) / 128), b(128);
  // forward Q_x^T, Q_y^T, Q_z^T (D^-1/2 on the way in, Lambda^+ on the way out)
  PDL_LAUNCH(lap_mode_kernel, g, b, 0, s, S0, S1, S2, 0, 0, eig, dm, (const double*)nullptr, 0, phi, u);
  PDL_LAUNCH(lap_mode_kernel, g, b, 0, s, S0, S1, S2, 1, 0, eig, (const double*)nullptr, (const double*)nullptr, 0,
             (const double*)u, w);
  PDL_LAUNCH(lap_mode_kernel, g, b, 0, s, S0, S1, S2, 2, 0, eig, (const double*)nullptr, (const double*)nullptr, 1,
             (const double*)w, u);
  // backward Q_z, Q_y, Q_x (D^-1/2 on the way out)
  PDL_LAUNCH(lap_mode_kernel, g, b, 0, s, S0, S1, S2, 2, 1, eig, (const double*)nullptr, (const double*)nullptr, 0,
             (const double*)u, w);
  PDL_LAUNCH(lap_mode_kernel, g, b, 0, s, S0, S1, S2, 1, 1, eig, (const double*)nullptr, (const double*)nullptr, 0,
             (const double*)w, u);
  PDL_LAUNCH(lap_mode_kernel, g, b, 0, s, S0, S1, S2, 0, 1, eig, (const double*)nullptr, dm, 0, (const double*)u, z);
  return 0;
}

extern "C" int bddc_lap_solve(int S0, int S1, int S2, const double* eig, const double* dm, const double* phi, double* z,
                              void* stream) {
  int N = S0 * S1 * S2;
  size_t shm = (2 * (size_t)N + S0 * S0 + S1 * S1 + S2 * S2 + S0 + S1 + S2) * sizeof(double);
  if (shm > 227 * 1024) return bddc_set_error(BDDC_ERR_ARG, "lap_solve: too many subdomains for one CTA");
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(lap_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  lap_solve_kernel<<<1, 1024, shm, (cudaStream_t)stream>>>(S0, S1, S2, eig, dm, phi, z);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_proj_apply(int n_gamma, int maxG, const int* gown, const double* z, double* y, void* stream) {
  if (n_gamma <= 0) return 0;
  proj_apply_kernel<<<(n_gamma + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n_gamma, maxG, gown, z, y);
  LAUNCH_OK();
  return 0;
}

extern "C" size_t bddc_dot_workspace(void) { return DOT_BLOCKS * sizeof(double) + 64; }

// Mode-B balance operators (solver.py:146-179 restricted to the floating set F):
// two face-graph Laplacians over the N subdomains, padded to n x n -- batch 0
// weighted by face size (Phi_F Phi_F^T), batch 1 unit weights (balanced shift) --
// with the rows / columns of non-floating subdomains replaced by the identity so
// the batched SPD inverse applies.  Face weights are integers: the atomic sums are
// exact (deterministic).  `out` must be zero on entry.
__global__ void dirichlet_laplacian_kernel(int N, int n, int nfaces, const int* __restrict__ faces,
                                           const int* __restrict__ floating, double* __restrict__ out) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nfaces) {
    const int i = faces[4 * f], j = faces[4 * f + 1];
    const double wts[2] = {(double)faces[4 * f + 3], 1.0};
    const bool fi = floating[i], fj = floating[j];
    for (int b = 0; b < 2; ++b) {
      double* L = out + (size_t)b * n * n;
      if (fi && fj) {
        L[(size_t)i * n + j] -= wts[b];
        L[(size_t)j * n + i] -= wts[b];
      }
      if (fi) atomicAdd(&L[(size_t)i * n + i], wts[b]);
      if (fj) atomicAdd(&L[(size_t)j * n + j], wts[b]);
    }
  }
  // identity rows for the non-floating subdomains and the padding
  for (int r = f; r < n; r += gridDim.x * blockDim.x)
    if (r >= N || !floating[r])
      for (int b = 0; b < 2; ++b) out[(size_t)b * n * n + (size_t)r * n + r] = 1.0;
}

// out[b] (N x N) = inverse restricted to F x F, zero elsewhere
__global__ void dirichlet_finish_kernel(int N, int n, const int* __restrict__ floating,
                                        const double* __restrict__ inv, double* __restrict__ out0,
                                        double* __restrict__ out1) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)N * N) return;
  const int r = (int)(e / N), c = (int)(e % N);
  const bool keep = floating[r] && floating[c];
  out0[e] = keep ? inv[(size_t)r * n + c] : 0.0;
  out1[e] = keep ? inv[(size_t)n * n + (size_t)r * n + c] : 0.0;
}

extern "C" int bddc_dirichlet_laplacian(int N, int n, int nfaces, const int* faces, const int* floating,
                                        double* out, void* stream) {
  const int total = imax(nfaces, n);
  dirichlet_laplacian_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(N, n, nfaces, faces, floating,
                                                                                   out);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_dirichlet_finish(int N, int n, const int* floating, const double* inv, double* out0,
                                     double* out1, void* stream) {
  const long long tot = (long long)N * N;
  if (tot == 0) return 0;
  dirichlet_finish_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(N, n, floating, inv,
                                                                                          out0, out1);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_dot(const double* x, const double* y, long long n, void* ws, double* scal, int op, double* hist,
                        void* stream) {
  double* partial = (double*)ws;
  unsigned* counter = (unsigned*)(partial + DOT_BLOCKS);
  dot_kernel<0><<<DOT_BLOCKS, DOT_THREADS, 0, (cudaStream_t)stream>>>(x, const_cast<double*>(y), n, partial,
                                                                     counter, scal, op, hist, DotArgs{});
  LAUNCH_OK();
  return 0;
}

// y -= Phi^T z (projection apply) fused with the dot x . y and its `op`.
extern "C" int bddc_proj_dot(int n_gamma, int maxG, const int* gown, const double* z, double* y, const double* x,
                             void* ws, double* scal, int op, double* hist, void* stream) {
  double* partial = (double*)ws;
  unsigned* counter = (unsigned*)(partial + DOT_BLOCKS);
  DotArgs A{gown, maxG, z, nullptr, nullptr, nullptr, nullptr, 0ull, 0.0, 0};
  dot_kernel<1><<<DOT_BLOCKS, DOT_THREADS, 0, (cudaStream_t)stream>>>(x, y, n_gamma, partial, counter, scal, op,
                                                                     hist, A);
  LAUNCH_OK();
  return 0;
}

// y = (yb[own0] + yb[own1]) - Phi^T z: scatter, projection apply and the dot x . y in one pass.
extern "C" int bddc_proj_dot_broken(int n_gamma, int maxG, const int* gown, const double* yb, const double* z,
                                    double* y, const double* x, void* ws, double* scal, int op, double* hist,
                                    void* stream) {
  double* partial = (double*)ws;
  unsigned* counter = (unsigned*)(partial + DOT_BLOCKS);
  DotArgs A{gown, maxG, z, nullptr, nullptr, nullptr, yb, 0ull, 0.0, 0};
  PCG_LAUNCH(2, dot_kernel<3>, dim3(DOT_BLOCKS), dim3(DOT_THREADS), 0, (cudaStream_t)stream, x, y, (long long)n_gamma,
             partial, counter, scal, op, hist, A);
  return 0;
}

// xv += alpha p, r -= alpha Ap (alpha = scal[2]) fused with r . r and its `op`.
extern "C" int bddc_cg_update_dot(long long n, double* xv, const double* p, double* r, const double* Ap, void* ws,
                                  double* scal, int op, double* hist, void* stream) {
  double* partial = (double*)ws;
  unsigned* counter = (unsigned*)(partial + DOT_BLOCKS);
  DotArgs A{nullptr, 1, nullptr, xv, p, Ap, nullptr, 0ull, 0.0, 0};
  dot_kernel<2><<<DOT_BLOCKS, DOT_THREADS, 0, (cudaStream_t)stream>>>(r, r, n, partial, counter, scal, op, hist, A);
  LAUNCH_OK();
  return 0;
}

// Same, and (op 2) the reducing block sets the PCG WHILE node's condition `cond`
// (a cudaGraphConditionalHandle from bddc_graph_handle).
extern "C" int bddc_cg_update_dot_cond(long long n, double* xv, const double* p, double* r, const double* Ap,
                                       void* ws, double* scal, int op, double* hist, unsigned long long cond,
                                       double tol, int maxit, void* stream) {
  double* partial = (double*)ws;
  unsigned* counter = (unsigned*)(partial + DOT_BLOCKS);
  DotArgs A{nullptr, 1, nullptr, xv, p, Ap, nullptr, cond, tol, maxit};
  PCG_LAUNCH(3, dot_kernel<2>, dim3(DOT_BLOCKS), dim3(DOT_THREADS), 0, (cudaStream_t)stream, (const double*)r, r, n,
             partial, counter, scal, op, hist, A);
  return 0;
}

extern "C" int bddc_cg_update(long long n, const double* scal, double* x, const double* p, double* r, const double* Ap,
                              void* stream) {
  cg_update_kernel<<<DOT_BLOCKS, 256, 0, (cudaStream_t)stream>>>(n, scal, x, p, r, Ap);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_p_update(long long n, const double* scal, const double* z, double* p, void* stream) {
  PCG_LAUNCH(4, p_update_kernel, dim3(DOT_BLOCKS), dim3(256), 0, (cudaStream_t)stream, n, scal, z, p);
  return 0;
}

extern "C" int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha, const double* A,
                                  int lda, long long sA, const double* B, int ldb, long long sB, double beta,
                                  double* C, int ldc, long long sC, int batch, int upper, void* stream);

// Lp = Dm W Lambda^+ W^T Dm (N x N, N = S0 S1 S2); ws: 2 N^2 doubles.
extern "C" int bddc_lap_dense(int S0, int S1, int S2, const double* eig, const double* dm, double* ws, double* Lp,
                              void* stream) {
  const int N = S0 * S1 * S2;
  if (N <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  double* W = ws;
  double* Ws = ws + (size_t)N * N;
  lap_kron_kernel<<<1024, 256, 0, s>>>(S0, S1, S2, eig, W, Ws);
  LAUNCH_OK();
  int r = bddc_dgemm_batched(0, 1, N, N, N, 1.0, Ws, N, 0, W, N, 0, 0.0, Lp, N, 0, 1, 0, stream);
  if (r) return r;
  if (dm) {
    scale_sym_kernel<<<1024, 256, 0, s>>>(N, dm, Lp);
    LAUNCH_OK();
  }
  return 0;
}

static int g_gemv_wpr = 0;   // 0: automatic
extern "C" void bddc_set_gemv_wpr(int wpr) { g_gemv_wpr = wpr; }

// `pdl`: launch as a programmatic dependent launch (PCG mask bit 1).  Only for a matrix no
// kernel queued before the call writes: the rows go through the non-coherent path, which
// requires them read-only for the kernel's whole (early-started) lifetime.
static int gemv_launch(int n, int ld, int ncol, const double* M, const double* x, double* y, int pdl, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // enough warps for ~60 per SM on the row count (few long rows: split them)
  int wpr = g_gemv_wpr;
  if (wpr <= 0) wpr = (n >= 8192 || ncol < 1024) ? 1 : (n >= 4096 ? 2 : 4);
  const int bit = pdl ? 1 : 31;   // bit 31 of the mask is never set: plain launch
  switch (wpr) {
    case 1: PCG_LAUNCH(bit, gemv_kernel, dim3((n + 7) / 8), dim3(256), 0, s, n, ld, ncol, M, x, y); break;
    case 2: PCG_LAUNCH(bit, gemv_split_kernel<2>, dim3((n + 3) / 4), dim3(256), 0, s, n, ld, ncol, M, x, y); break;
    case 4: PCG_LAUNCH(bit, gemv_split_kernel<4>, dim3((n + 1) / 2), dim3(256), 0, s, n, ld, ncol, M, x, y); break;
    default: PCG_LAUNCH(bit, gemv_split_kernel<8>, dim3(n), dim3(256), 0, s, n, ld, ncol, M, x, y); break;
  }
  return 0;
}

extern "C" int bddc_gemv(int n, int ld, int ncol, const double* M, const double* x, double* y, void* stream) {
  return gemv_launch(n, ld, ncol, M, x, y, 0, stream);
}

extern "C" int bddc_gemv_static(int n, int ld, int ncol, const double* M, const double* x, double* y, void* stream) {
  return gemv_launch(n, ld, ncol, M, x, y, 1, stream);
}

// w -= Q^T c for Q with k rows of length n (row-major), c of length k.
extern "C" int bddc_gemv_t_sub(int k, int n, const double* Q, const double* c, double* w, void* stream) {
  if (n <= 0 || k <= 0) return 0;
  gemv_t_sub_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(k, n, Q, c, w);
  LAUNCH_OK();
  return 0;
}

// Every eigenvalue of the m x m symmetric tridiagonal (diagonal d, off-diagonal e),
// ascending; work: m doubles.
extern "C" int bddc_tridiag_eigvals(int m, const double* d, const double* e, double* work, double* out,
                                    void* stream) {
  if (m <= 0) return 0;
  // each block recomputes the (cheap) Gershgorin bounds and squares e into work
  // (identical values: benign)
  tridiag_eigvals_kernel<<<(m + 127) / 128, 128, 0, (cudaStream_t)stream>>>(m, d, e, work, out);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_lanczos(int m, const double* al, const double* be, double* work, double* out, void* stream) {
  if (m <= 0) return 0;
  lanczos_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(m, al, be, work, out);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_axpby(long long n, double a, const double* x, double b, double* y, void* stream) {
  if (n <= 0) return 0;
  axpby_kernel<<<DOT_BLOCKS, 256, 0, (cudaStream_t)stream>>>(n, a, x, b, y);
  LAUNCH_OK();
  return 0;
}
