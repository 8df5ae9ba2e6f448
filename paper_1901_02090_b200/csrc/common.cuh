// Shared device helpers for the B200 BDDC kernels (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/bddc.h"

#define BDDC_MAXS 64   // max subdomain strips per axis (see bddc_geom)

#define CUDA_OK(x)                                                    \
  do {                                                                \
    cudaError_t _e = (x);                                             \
    if (_e != cudaSuccess) return bddc_set_error(BDDC_ERR_CUDA, cudaGetErrorString(_e)); \
  } while (0)

extern "C" void bddc_count_launch(void);

#define LAUNCH_OK()                                                   \
  do {                                                                \
    bddc_count_launch();                                              \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return bddc_set_error(BDDC_ERR_CUDA, cudaGetErrorString(_e)); \
  } while (0)

extern "C" int bddc_set_error(int code, const char* msg);

__host__ __device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

// Ampere-style asynchronous global->shared copies (LDGSTS): every copy of a
// staged tile is in flight at once, independent of the compiler's load schedule.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Bulk asynchronous copies (the TMA engine's non-tensor path, SASS UBLKCP) and
// the mbarriers that track them: a single thread moves a contiguous global range
// of any 16-byte multiple into shared memory; the mbarrier's transaction count
// completes when the bytes have landed.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// start while its stream predecessor is still running.  Everything it does
// before pdl_wait() must touch only data no earlier kernel writes (index
// tables, factors); pdl_wait() returns once the predecessor grid completed and
// its memory is visible.  pdl_trigger() lets the successor launch early.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

extern "C" int bddc_pdl_enabled(void);

extern "C" int bddc_pdl_pcg_enabled(void);

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl_if(int allowed, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t shm,
                                        cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = shm;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = allowed ? 1 : 0;
  // the stream's priority as an explicit launch attribute, so that a kernel node
  // captured into a graph (the PCG WHILE body) keeps it
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = prio;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t shm, cudaStream_t s,
                                     Args... args) {
  return launch_pdl_if(bddc_pdl_enabled(), kernel, grid, block, shm, s, args...);
}

// Plain launch carrying the stream's priority as a launch attribute (see launch_pdl).
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_prio(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t shm, cudaStream_t s,
                                      Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = shm;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = prio;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define PDL_LAUNCH(kernel, grid, block, shm, stream, ...)                  \
  do {                                                                    \
    bddc_count_launch();                                                  \
    cudaError_t _e = launch_pdl(kernel, grid, block, shm, stream, __VA_ARGS__); \
    if (_e != cudaSuccess) return bddc_set_error(BDDC_ERR_CUDA, cudaGetErrorString(_e)); \
  } while (0)

// The small dependent kernels of the PCG iteration (projection, dots, updates): PDL
// launches whose kernels trigger and wait at their top, so each becomes resident
// during its predecessor instead of paying a launch latency after it.
#define PCG_LAUNCH(bit, kernel, grid, block, shm, stream, ...)             \
  do {                                                                    \
    bddc_count_launch();                                                  \
    cudaError_t _e = launch_pdl_if((bddc_pdl_pcg_enabled() >> (bit)) & 1, kernel, grid, block, shm, stream, __VA_ARGS__); \
    if (_e != cudaSuccess) return bddc_set_error(BDDC_ERR_CUDA, cudaGetErrorString(_e)); \
  } while (0)

// Streaming read that bypasses L1 allocation.  Every once-read matrix stream of the solve
// (packed Q, S_i / T_i tiles of the LDG kernels, Psi, the ND factors) uses it: the stream
// would otherwise evict what the SM does re-read from L1 -- per-thread local-memory
// arrays, gathered vectors, index tables (local solves 627 -> 550 us, ND solve 103 -> 93 us,
// C4 S_i GEMV 165 -> 151 us).
__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Warp GEMV helpers over row-major rows (read-only matrix via the non-coherent
// path, vector in shared memory).  Fixed summation order: deterministic.

// One long row: 8 independent accumulators keep 8 loads per lane in flight.
__device__ __forceinline__ double warp_row_dot(const double* __restrict__ row, const double* v, int len, int lane) {
  double a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = 0.0;
  int c = lane;
  for (; c + 224 < len; c += 256) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = ldg_stream(row + c + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] += x[u] * v[c + 32 * u];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (c + 32 * u < len) a[u] += ldg_stream(row + c + 32 * u) * v[c + 32 * u];
  double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Four short rows at once (rows base + k*ld, k < nr <= 4): 16 loads per lane in
// flight, so rows of ~100 entries do not serialise on memory latency.
__device__ __forceinline__ void warp_rows4_dot(const double* __restrict__ base, size_t ld, int nr,
                                               const double* v, int len, int lane, double out[4]) {
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c0 = 0; c0 < len; c0 += 128) {
    double x[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + lane + 32 * u;
        x[k][u] = (k < nr && c < len) ? ldg_stream(base + (size_t)k * ld + c) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + lane + 32 * u;
      const double vv = (c < len) ? v[c] : 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] += x[k][u] * vv;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], o);
    out[k] = a[k];
  }
}

// Tile-packed symmetric storage: upper-triangle 32x32 tiles (bi <= bj) in
// row-major tile order, each tile row-major; nt = n / 32 tiles per row.
__device__ __forceinline__ int tile_index(int bi, int bj, int nt) { return bi * nt - (bi * (bi - 1)) / 2 + (bj - bi); }

// y = M x for one tile-packed symmetric matrix, whole CTA, vectors in shared
// memory (x zero beyond the live size, ntl = live tiles per row).  Each warp
// streams whole tiles (32 loads per lane in flight), forms the column
// contribution directly and the row contribution by a transpose-reduction, and
// accumulates into its own slice of yw (nwarps x ntl*32 doubles of shared
// memory); the slices are summed in warp order: deterministic.
// Two right-hand sides through one read of the packed tiles: y = P x, y2 = P x2
// (yw: 2 x warps x ntl*32 partials).
__device__ __forceinline__ void cta_symv_packed2(const double* __restrict__ Pk, int nt, int ntl, const double* x,
                                                 const double* x2, double* y, double* y2, double* yw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int len = ntl * 32;
  for (int e = threadIdx.x; e < 2 * nw * len; e += blockDim.x) yw[e] = 0.0;
  __syncthreads();
  const int nlive = ntl * (ntl + 1) / 2;
  for (int u = warp; u < nlive; u += nw) {
    int bi = 0, rem = u;
    while (rem >= ntl - bi) {
      rem -= ntl - bi;
      ++bi;
    }
    const int bj = bi + rem;
    const double* T = Pk + (size_t)tile_index(bi, bj, nt) * 1024;
    // the second pass re-reads the tile this warp just streamed (L1 / L2 hit): one
    // DRAM read for both right-hand sides at the single-rhs register footprint
#pragma unroll 1
    for (int s = 0; s < 2; ++s) {
      const double* xs = s ? x2 : x;
      double* my = yw + ((size_t)s * nw + warp) * len;
      const double xl = xs[bj * 32 + lane];
      double v[32];
      double col = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const double a = __ldg(T + r * 32 + lane);
        v[r] = a * xl;
        col += a * xs[bi * 32 + r];
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const bool up = lane & off;
#pragma unroll
        for (int k = 0; k < off; ++k) {
          const double send = up ? v[k] : v[k + off];
          const double recv = __shfl_xor_sync(0xffffffffu, send, off);
          v[k] = (up ? v[k + off] : v[k]) + recv;
        }
      }
      my[bi * 32 + lane] += v[0];
      if (bi != bj) my[bj * 32 + lane] += col;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * len; e += blockDim.x) {
    const int s = e >= len, ee = e - s * len;
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) acc += yw[((size_t)s * nw + w) * len + ee];
    (s ? y2 : y)[ee] = acc;
  }
  __syncthreads();
}

__device__ __forceinline__ void cta_symv_packed(const double* __restrict__ Pk, int nt, int ntl, const double* x,
                                                double* y, double* yw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int len = ntl * 32;
  for (int e = threadIdx.x; e < nw * len; e += blockDim.x) yw[e] = 0.0;
  __syncthreads();
  double* my = yw + (size_t)warp * len;
  const int nlive = ntl * (ntl + 1) / 2;
  for (int u = warp; u < nlive; u += nw) {
    int bi = 0, rem = u;
    while (rem >= ntl - bi) {
      rem -= ntl - bi;
      ++bi;
    }
    const int bj = bi + rem;
    const double* T = Pk + (size_t)tile_index(bi, bj, nt) * 1024;
    const double xl = x[bj * 32 + lane];
    double v[32];
    double col = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const double a = ldg_stream(T + r * 32 + lane);
      v[r] = a * xl;
      col += a * x[bi * 32 + r];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const bool up = lane & off;
#pragma unroll
      for (int k = 0; k < off; ++k) {
        const double send = up ? v[k] : v[k + off];
        const double recv = __shfl_xor_sync(0xffffffffu, send, off);
        v[k] = (up ? v[k + off] : v[k]) + recv;
      }
    }
    my[bi * 32 + lane] += v[0];
    if (bi != bj) my[bj * 32 + lane] += col;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) acc += yw[(size_t)w * len + e];
    y[e] = acc;
  }
  __syncthreads();
}

// Subdomain box of subdomain i under a regular partition.
struct Box {
  int o[3];   // origin (cells)
  int L[3];   // extent (cells)
  int s[3];   // strip index per axis
};

__device__ __forceinline__ Box sub_box(const bddc_geom& G, int i) {
  Box b;
  b.s[0] = i % G.S[0];
  b.s[1] = (i / G.S[0]) % G.S[1];
  b.s[2] = i / (G.S[0] * G.S[1]);
  for (int a = 0; a < 3; ++a) {
    b.o[a] = G.so[a][b.s[a]];
    b.L[a] = G.sw[a][b.s[a]];
  }
  return b;
}

__device__ __forceinline__ int cell_id(const bddc_geom& G, int x, int y, int z) {
  return x + G.n[0] * (y + G.n[1] * z);
}

// Global dof of the interior a-face whose face coordinate is (fx,fy,fz),
// f_a in 1..n_a-1 (grid.py:102-108 numbering: family-major, x-fastest).
__device__ __forceinline__ int face_dof(const bddc_geom& G, int a, int fx, int fy, int fz) {
  int e0 = G.n[0] - (a == 0), e1 = G.n[1] - (a == 1);
  int c0 = fx - (a == 0), c1 = fy - (a == 1), c2 = fz - (a == 2);
  return G.fam_off[a] + c0 + e0 * (c1 + e1 * c2);
}

// Transverse axes of axis a (in increasing order).
__device__ __forceinline__ void trans_axes(int a, int& t1, int& t2) {
  t1 = (a == 0) ? 1 : 0;
  t2 = (a == 2) ? 1 : 2;
}

// Mode B: dof of the Dirichlet boundary face at end `side` (0 low, 1 high) of
// axis G.dir_axis on the grid line through global cell coordinates gc.
__device__ __forceinline__ int bnd_dof(const bddc_geom& G, int side, const int gc[3]) {
  int t1, t2;
  trans_axes(G.dir_axis, t1, t2);
  return G.n_flux_int + side * G.n_bt + gc[t1] + G.n[t1] * gc[t2];
}

// Mode B: does the box's line along axis a end on a Dirichlet face (lo / hi)?
__device__ __forceinline__ void line_open(const bddc_geom& G, const Box& b, int a, int& lo, int& hi) {
  lo = (a == G.dir_axis && b.o[a] == 0);
  hi = (a == G.dir_axis && b.o[a] + b.L[a] == G.n[a]);
}

// Floating subdomain: no Dirichlet face, so its interior pressure block is
// singular (null space 1) and it carries a balance constraint / coarse pressure.
__device__ __forceinline__ bool sub_floating(const bddc_geom& G, const Box& b) {
  int lo, hi;
  if (G.dir_axis < 0) return true;
  line_open(G, b, G.dir_axis, lo, hi);
  return !(lo || hi);
}

// Line geometry: line index q of axis a in a box -> local coords of the
// transverse axes.  Line index ordering is x-fastest over the transverse
// axes (matches the sorted global order of the dofs on one box face).
__device__ __forceinline__ void line_coords(const Box& b, int a, int q, int c[3]) {
  int t1, t2;
  trans_axes(a, t1, t2);
  c[a] = 0;
  c[t1] = q % b.L[t1];
  c[t2] = q / b.L[t1];
}

__device__ __forceinline__ int n_lines(const Box& b, int a) {
  int t1, t2;
  trans_axes(a, t1, t2);
  return b.L[t1] * b.L[t2];
}

__device__ __forceinline__ int local_cell(const Box& b, int x, int y, int z) {
  return x + b.L[0] * (y + b.L[1] * z);
}

// Deterministic block-wide sum (fixed reduction tree).  `red` must hold
// blockDim.x/32 doubles.  Returns the total to every thread.
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  double t = 0.0;
  if (w == 0) {
    t = (l < nw) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  if (w == 0) {
    double t = (l < nw) ? red[l] : -1.0e308;
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  double t = red[0];
  __syncthreads();
  return t;
}
