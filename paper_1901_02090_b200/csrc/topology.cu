// Interface topology of a box partition, built on the device in closed form
// (the tables decomposition.py:32-125 derives with per-subdomain Python loops;
// for tensor-product partitions every entry is an index formula).
//
// Slots of subdomain i are its interface dofs in increasing global dof id
// (decomposition.py:72-75): family x, then y, then z.  With l1/l2 the box-local
// transverse coordinates (line = l1 + L_t1 l2) and np = number of interface planes
// of the box on that axis (low plane first), the sorted position inside a family is
//   x: (l2 L_y + l1) np + plane        (dof ids run plane-fastest)
//   y: (l2 np + plane) L_x + l1        (a y-plane row is contiguous in x)
//   z: (plane L_y + l2) L_x + l1       (a z-plane is contiguous)
// and the rank of a dof among all interface dofs (gpos) follows the same pattern
// with the global extents and the S_a - 1 interface planes of axis a.
#include "common.cuh"

namespace {

__global__ void topo_slots_kernel(bddc_geom G, const int* __restrict__ face_base, int* __restrict__ nG,
                                  int* __restrict__ gpos, int* __restrict__ gcode, int* __restrict__ fslot,
                                  int* __restrict__ gown, int* __restrict__ gamma, int* __restrict__ gface) {
  const int i = blockIdx.x;
  const Box b = sub_box(G, i);
  int lo[3], hi[3], base[3], cnt[3];
  int tot = 0;
  for (int a = 0; a < 3; ++a) {
    lo[a] = (a < G.dim) && b.s[a] > 0;
    hi[a] = (a < G.dim) && b.s[a] < G.S[a] - 1;
    cnt[a] = (lo[a] + hi[a]) * n_lines(b, a);
    base[a] = tot;
    tot += cnt[a];
  }
  if (threadIdx.x == 0) nG[i] = tot;
  const int nx = G.n[0], ny = G.n[1], nz = G.n[2];
  const int off_y = (G.S[0] - 1) * ny * nz;
  const int off_z = off_y + nx * (G.S[1] - 1) * nz;
  const int fb = face_base[i];
  for (int q = threadIdx.x; q < G.maxG; q += blockDim.x) {
    const size_t at = (size_t)i * G.maxG + q;
    if (q >= tot) {
      gpos[at] = -1;
      gcode[at] = -1;
      continue;
    }
    const int a = q >= base[2] ? 2 : (q >= base[1] ? 1 : 0);
    const int r = q - base[a];
    const int np = lo[a] + hi[a];
    int l1, l2, plane;
    if (a == 0) {
      plane = r % np;
      const int line = r / np;
      l1 = line % b.L[1];
      l2 = line / b.L[1];
    } else if (a == 1) {
      l1 = r % b.L[0];
      const int t = r / b.L[0];
      plane = t % np;
      l2 = t / np;
    } else {
      l1 = r % b.L[0];
      const int t = r / b.L[0];
      l2 = t % b.L[1];
      plane = t / b.L[1];
    }
    int t1, t2;
    trans_axes(a, t1, t2);
    const int side = (plane == 0 && lo[a]) ? 0 : 1;  // 1: the box's high face (+axis points out)
    const int s = b.s[a] + side;                     // interface plane 1 .. S_a-1
    int c[3];
    c[t1] = b.o[t1] + l1;
    c[t2] = b.o[t2] + l2;
    c[a] = G.so[a][s];
    const int line = l1 + b.L[t1] * l2;
    int rank;
    if (a == 0)
      rank = (G.S[0] - 1) * (c[1] + ny * c[2]) + (s - 1);
    else if (a == 1)
      rank = off_y + c[0] + nx * ((s - 1) + (G.S[1] - 1) * c[2]);
    else
      rank = off_z + c[0] + nx * (c[1] + ny * (s - 1));
    gpos[at] = rank;
    gcode[at] = a | (side << 2) | (line << 3);
    fslot[((size_t)i * 6 + 2 * a + side) * G.maxF + line] = q;
    gown[2 * (size_t)rank + (side ? 0 : 1)] = i * G.maxG + q;
    if (side) {  // the low-side copy names the dof and its face (i, i + stride_a)
      gamma[rank] = face_dof(G, a, c[0], c[1], c[2]);
      gface[rank] = fb + (a >= 1 ? hi[0] : 0) + (a >= 2 ? hi[1] : 0);
    }
  }
}

__global__ void topo_cells_kernel(bddc_geom G, int* __restrict__ cell_sub) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= G.n_cells) return;
  int x[3] = {c % G.n[0], (c / G.n[0]) % G.n[1], c / (G.n[0] * G.n[1])};
  int s[3];
  for (int a = 0; a < 3; ++a) {
    int k = 0;
    while (k + 1 < G.S[a] && G.so[a][k + 1] <= x[a]) ++k;
    s[a] = k;
  }
  cell_sub[c] = s[0] + G.S[0] * (s[1] + G.S[1] * s[2]);
}

// solver.py:286-298: per face, max k over the low-side cells against min k over the
// high-side cells; flag set when some face has a ratio outside [1e-3, 1e3].
__global__ void face_jump_kernel(bddc_geom G, const int* __restrict__ faces, const double* __restrict__ k,
                                 int* __restrict__ flag) {
  __shared__ double smax[32], smin[32];
  const int f = blockIdx.x;
  const int i = faces[4 * f], a = faces[4 * f + 2], m = faces[4 * f + 3];
  const Box b = sub_box(G, i);
  const int stride_g = a == 0 ? 1 : (a == 1 ? G.n[0] : G.n[0] * G.n[1]);
  double kmax = 0.0, kmin = 1e300;
  for (int line = threadIdx.x; line < m; line += blockDim.x) {
    int c[3];
    line_coords(b, a, line, c);
    c[a] = b.L[a] - 1;
    const int own = cell_id(G, b.o[0] + c[0], b.o[1] + c[1], b.o[2] + c[2]);
    const int oth = own + stride_g;
    for (int d = 0; d < G.dim; ++d) {
      kmax = fmax(kmax, k[(size_t)own * G.dim + d]);
      kmin = fmin(kmin, k[(size_t)oth * G.dim + d]);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    kmax = fmax(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    kmin = fmin(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smax[threadIdx.x >> 5] = kmax;
    smin[threadIdx.x >> 5] = kmin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      kmax = fmax(kmax, smax[w]);
      kmin = fmin(kmin, smin[w]);
    }
    const double ratio = kmax / fmax(kmin, 1e-300);
    if (ratio > 1e3 || ratio < 1e-3) atomicOr(flag, 1);
  }
}

}  // namespace

extern "C" int bddc_topology_box(const bddc_geom* g, const int* face_base, int* nG, int* gpos, int* gcode,
                                 int* fslot, int* gown, int* gamma, int* gface, int* cell_sub, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_OK(cudaMemsetAsync(fslot, 0xff, (size_t)g->N * 6 * g->maxF * sizeof(int), s));
  topo_slots_kernel<<<g->N, 128, 0, s>>>(*g, face_base, nG, gpos, gcode, fslot, gown, gamma, gface);
  LAUNCH_OK();
  topo_cells_kernel<<<(g->n_cells + 255) / 256, 256, 0, s>>>(*g, cell_sub);
  LAUNCH_OK();
  return 0;
}

extern "C" int bddc_face_jumps(const bddc_geom* g, const int* faces, const double* k, int* flag, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_OK(cudaMemsetAsync(flag, 0, sizeof(int), s));
  if (g->n_faces == 0) return 0;
  face_jump_kernel<<<g->n_faces, 64, 0, s>>>(*g, faces, k, flag);
  LAUNCH_OK();
  return 0;
}
