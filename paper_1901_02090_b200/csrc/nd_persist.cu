// Whole nested-dissection coarse solve (forward, root pressure block, backward)
// as ONE persistent kernel with dataflow dependencies instead of one launch per
// tree level (see coarse_nd.py for the factorisation and the compact layout).
//
// Work items are claimed from a global queue in topological order (deepest
// level first for the forward sweep, root first for the backward sweep); a CTA
// that claims an item spins until the items it depends on have published their
// completion counters.  A CTA only waits on items claimed before its own, and
// those are held by CTAs that are already running, so the schedule cannot
// deadlock whatever the grid size or co-residency.  Everything produced inside
// the kernel (separator right-hand sides, update vectors, y, x) is read through
// L2 (ld.global.cg) because L1 is not coherent between SMs.
//
// Items (int4 {type | wpr << 8, node, r0, r1}):
//   GATHER  rs[sp+t] = r[g_t] - sum of descendant updates, t in [r0, r1)
//   FWD     rows [r0, r1) of [F11inv; X] r_sep  (rows < s -> y, rows >= s -> cbuf)
//   FWDF    GATHER + FWD of a whole node in one item (nodes with one row block)
//   PGATHER pressure right-hand sides [r0, r1) (pressures 1..N-1)
//   PGEMV   x_p = -Pc^-1 rp, rows [r0, r1)
//   BWD     x_sep = y - X^T x_bnd, separator rows [r0, r1), wpr warps per row
#include "common.cuh"

namespace {

enum { T_GATHER = 0, T_FWD = 1, T_FWDF = 2, T_PGATHER = 3, T_PGEMV = 4, T_BWD = 5 };

// node table columns (int): s, b, sp, bp, cbo, parent, child0, child1, nfwd, ngat, nbwd
enum { N_S = 0, N_B, N_SP, N_BP, N_CBO, N_PAR, N_CH0, N_CH1, N_NFWD, N_NGAT, N_NBWD, N_COLS };

struct NdArgs {
  const int4* items;
  int nitems;
  const int* node;            // nnodes x N_COLS
  const long long* off;       // compact data offset per node
  const int* sep_flat;        // global separator dof ids (sp-indexed)
  const int* bnd_flat;        // global boundary dof ids (bp-indexed)
  const int* lptr;            // gather lists over sp-indexed entries
  const int* lsrc;
  const int* pptr;            // pressure gather lists
  const int* psrc;
  const double* Fc;
  const double* Pcinv;
  const double* r;
  double* rs;
  double* ybuf;
  double* cbuf;
  double* prhs;
  double* x;
  int* cnt;                   // [queue head, pg_done, pv_done, fwd_done[n], gat_done[n], bwd_done[n]]
  int nnodes, root, N, nfc, npc, npg, npv;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 spins until *p >= want; then the whole CTA proceeds
__device__ __forceinline__ void wait_ge(const int* p, int want) {
  if (threadIdx.x == 0) {
    while (ld_acquire(p) < want) __nanosleep(20);
  }
  __syncthreads();
}

// all threads' writes done -> publish one completion (release-ordered add)
__device__ __forceinline__ void publish(int* p) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p) : "memory");
}

// 8 lanes per entry: rhs[t] = base[t] - sum_p cbuf[src[p]], t in [t0, t1)
__device__ void gather_block(int t0, int t1, const int* __restrict__ ptr, const int* __restrict__ src,
                             const double* cbuf, const double* __restrict__ base_vals, const int* __restrict__ gidx,
                             int gofs, double* out, bool out_shared, int out0) {
  const int sub = threadIdx.x & 7;
  for (int tb = t0; tb < t1; tb += (blockDim.x >> 3)) {
    const int t = tb + (threadIdx.x >> 3);
    double acc = 0.0;
    if (t < t1) {
      const int p1 = ptr[t + 1];
      for (int p = ptr[t] + sub; p < p1; p += 8) acc += __ldcg(cbuf + src[p]);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (t < t1 && sub == 0) {
      const double v = __ldg(base_vals + (gidx ? gidx[t] : gofs + t)) - acc;
      if (out_shared) out[t - out0] = v;
      else out[t] = v;
    }
  }
}

__global__ void __launch_bounds__(256) nd_persist_kernel(NdArgs a) {
  extern __shared__ double sm[];
  __shared__ int item_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int* head = a.cnt;
  int* pg_done = a.cnt + 1;
  int* pv_done = a.cnt + 2;
  int* fwd_done = a.cnt + 3;
  int* gat_done = fwd_done + a.nnodes;
  int* bwd_done = gat_done + a.nnodes;
  while (true) {
    if (threadIdx.x == 0) item_s = atomicAdd(head, 1);
    __syncthreads();
    const int it = item_s;
    __syncthreads();
    if (it >= a.nitems) break;
    const int4 w = a.items[it];
    const int type = w.x & 255, wpr = w.x >> 8, n = w.y, r0 = w.z, r1 = w.w;
    const int* nd = a.node + (size_t)(n >= 0 ? n : 0) * N_COLS;
    if (type == T_GATHER || type == T_FWD || type == T_FWDF) {
      const int s = nd[N_S], sp = nd[N_SP], cbo = nd[N_CBO];
      if (type != T_FWD) {
        for (int c = 0; c < 2; ++c) {
          const int ch = nd[N_CH0 + c];
          if (ch >= 0) wait_ge(fwd_done + ch, a.node[(size_t)ch * N_COLS + N_NFWD]);
        }
      }
      if (type == T_GATHER) {
        gather_block(sp + r0, sp + r1, a.lptr, a.lsrc, a.cbuf, a.r, a.sep_flat, 0, a.rs, false, 0);
        publish(gat_done + n);
        continue;
      }
      if (type == T_FWDF) {
        // every row block of the node gathers r_sep itself (L2 reads) instead of
        // waiting on a separate gather item: one dependency hop per level
        gather_block(sp, sp + s, a.lptr, a.lsrc, a.cbuf, a.r, a.sep_flat, 0, sm, true, sp);
      } else {
        wait_ge(gat_done + n, nd[N_NGAT]);
        for (int k = threadIdx.x; k < s; k += blockDim.x) sm[k] = __ldcg(a.rs + sp + k);
      }
      __syncthreads();
      const double* base = a.Fc + a.off[n];
      for (int row = r0 + 4 * warp; row < r1; row += 4 * nw) {
        const int nr = imin(4, r1 - row);
        double acc[4];
        warp_rows4_dot(base + (size_t)row * s, s, nr, sm, s, lane, acc);
        if (lane < nr) {
          const double v = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
          const int rr = row + lane;
          if (rr < s) a.ybuf[sp + rr] = v;
          else a.cbuf[cbo + rr - s] = v;
        }
      }
      publish(fwd_done + n);
      continue;
    }
    if (type == T_PGATHER) {
      wait_ge(fwd_done + a.root, a.node[(size_t)a.root * N_COLS + N_NFWD]);
      gather_block(r0, r1, a.pptr, a.psrc, a.cbuf, a.r, nullptr, a.nfc + 1, a.prhs, false, 0);
      publish(pg_done);
      continue;
    }
    if (type == T_PGEMV) {
      wait_ge(pg_done, a.npg);
      const int np = a.N - 1;
      for (int k = threadIdx.x; k < np; k += blockDim.x) sm[k] = __ldcg(a.prhs + k);
      __syncthreads();
      if (r0 == 0 && threadIdx.x == 0) a.x[a.nfc] = 0.0;
      for (int row = r0 + warp; row < r1; row += nw) {
        const double acc = warp_row_dot(a.Pcinv + (size_t)row * a.npc, sm, np, lane);
        if (lane == 0) a.x[a.nfc + 1 + row] = -acc;
      }
      publish(pv_done);
      continue;
    }
    // T_BWD
    {
      const int s = nd[N_S], b = nd[N_B], sp = nd[N_SP], bp = nd[N_BP];
      const int par = nd[N_PAR];
      if (par >= 0) wait_ge(bwd_done + par, a.node[(size_t)par * N_COLS + N_NBWD]);
      else wait_ge(pv_done, a.npv);
      for (int m = threadIdx.x; m < b; m += blockDim.x) sm[m] = __ldcg(a.x + a.bnd_flat[bp + m]);
      __syncthreads();
      const double* XT = a.Fc + a.off[n] + (size_t)s * s + (size_t)b * s;
      if (wpr <= 1) {
        for (int k = r0 + 4 * warp; k < r1; k += 4 * nw) {
          const int nr = imin(4, r1 - k);
          double acc[4];
          warp_rows4_dot(XT + (size_t)k * b, b, nr, sm, b, lane, acc);
          if (lane < nr) {
            const double v = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
            a.x[a.sep_flat[sp + k + lane]] = __ldcg(a.ybuf + sp + k + lane) - v;
          }
        }
      } else {
        double* part = sm + b;   // nw partial sums
        const int rpc = nw / wpr;
        const int rl = warp / wpr, pc = warp % wpr;
        const int chunk = ((b + wpr - 1) / wpr + 31) & ~31;
        const int c0 = imin(pc * chunk, b), c1 = imin(c0 + chunk, b);
        for (int kb = r0; kb < r1; kb += rpc) {
          const int k = kb + rl;
          double acc = 0.0;
          if (k < r1) acc = warp_row_dot(XT + (size_t)k * b + c0, sm + c0, c1 - c0, lane);
          if (lane == 0) part[warp] = acc;
          __syncthreads();
          if (threadIdx.x < rpc && kb + (int)threadIdx.x < r1) {
            double t = 0.0;
            for (int u = 0; u < wpr; ++u) t += part[threadIdx.x * wpr + u];
            const int kk = kb + threadIdx.x;
            a.x[a.sep_flat[sp + kk]] = __ldcg(a.ybuf + sp + kk) - t;
          }
          __syncthreads();
        }
      }
      publish(bwd_done + n);
    }
  }
}

}  // namespace

extern "C" int bddc_nd_persist_counters(int nnodes) { return 3 + 3 * nnodes; }

// One coarse solve: zero the counters, launch the persistent kernel.
extern "C" int bddc_nd_solve_persist(int nitems, const int* items, int nnodes, const int* node, const long long* off,
                                     const int* sep_flat, const int* bnd_flat, const int* lptr, const int* lsrc,
                                     const int* pptr, const int* psrc, const double* Fc, const double* Pcinv,
                                     const double* r, double* rs, double* ybuf, double* cbuf, double* prhs, double* x,
                                     int* cnt, int root, int N, int nfc, int npc, int npg, int npv, int smem_doubles,
                                     int grid, void* stream) {
  if (nitems <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_OK(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)(3 + 3 * nnodes), s));
  NdArgs a;
  a.items = (const int4*)items;
  a.nitems = nitems;
  a.node = node;
  a.off = off;
  a.sep_flat = sep_flat;
  a.bnd_flat = bnd_flat;
  a.lptr = lptr;
  a.lsrc = lsrc;
  a.pptr = pptr;
  a.psrc = psrc;
  a.Fc = Fc;
  a.Pcinv = Pcinv;
  a.r = r;
  a.rs = rs;
  a.ybuf = ybuf;
  a.cbuf = cbuf;
  a.prhs = prhs;
  a.x = x;
  a.cnt = cnt;
  a.nnodes = nnodes;
  a.root = root;
  a.N = N;
  a.nfc = nfc;
  a.npc = npc;
  a.npg = npg;
  a.npv = npv;
  size_t shm = (size_t)(smem_doubles + 8) * sizeof(double);
  if (shm > 48 * 1024)
    CUDA_OK(cudaFuncSetAttribute(nd_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  static int cached_grid = 0;
  static size_t cached_shm = 0;
  if (grid <= 0 && cached_grid > 0 && cached_shm == shm) grid = cached_grid;
  if (grid <= 0) {
    int per_sm = 0, dev = 0, sms = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nd_persist_kernel, 256, shm));
    grid = sms * (per_sm > 0 ? per_sm : 1);
    cached_grid = grid;
    cached_shm = shm;
  }
  nd_persist_kernel<<<grid, 256, shm, s>>>(a);
  LAUNCH_OK();
  return 0;
}
