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
