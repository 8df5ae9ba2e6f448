/* libbddc — B200-native (sm_100a) adaptive-BDDC PCG for RT0/P0 Darcy flow.
 *
 * C ABI: plain device pointers (FP64 / int32) and sizes, a caller-owned
 * cudaStream_t passed as void*.  No torch types cross this boundary; the
 * Python host layer (paper_1901_02090_b200) passes tensor.data_ptr() values.
 * Every function returns 0 on success or a BDDC_ERR_* code; the message is
 * available from bddc_last_error().  Error codes map 1:1 onto the reference
 * exception classes (/root/reference/pkg/src/bddcflow/errors.py:4-48).
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/pkg/src/bddcflow/).
 */
#ifndef BDDC_H
#define BDDC_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.py:4-48 */
enum {
  BDDC_OK = 0,
  BDDC_ERR_ARG = 1,          /* InvalidArgumentError */
  BDDC_ERR_NUMERICAL = 2,    /* NumericalFailureError(where) */
  BDDC_ERR_RANK = 3,         /* ConstraintRankError */
  BDDC_ERR_CONFIG = 4,       /* ConfigurationError */
  BDDC_ERR_INTERNAL = 5,     /* InternalConsistencyError */
  BDDC_ERR_CUDA = 6          /* CUDA runtime failure (no reference analogue) */
};

#define BDDC_MAX_STRIPS 64

/* Grid + regular partition (grid.py:21-175, decomposition.py:128-151).
 * 2D problems are represented with n[2] = 1, h[2] = 1, S[2] = 1. */
typedef struct bddc_geom {
  int dim;
  int n[3];                        /* cells per axis */
  double h[3];                     /* cell sizes */
  double vol;                      /* cell volume (product of h over dim axes) */
  int S[3];                        /* splits per axis */
  int so[3][BDDC_MAX_STRIPS];      /* strip origins */
  int sw[3][BDDC_MAX_STRIPS];      /* strip widths (near-equal, decomposition.py:128-130) */
  int fam_off[4];                  /* flux dof offsets per face family */
  int n_cells, n_flux, N, n_gamma, n_faces;
  int maxG;                        /* padded interface slots per subdomain (multiple of 64) */
  int maxP;                        /* padded cells per subdomain (multiple of 64) */
  int maxL;                        /* max strip width */
  int maxF;                        /* max dofs on one box face */
  /* mode B (Dirichlet pressure on both ends of one axis; not in the reference):
   * dir_axis = that axis or -1 (mode A).  The boundary faces of dir_axis are
   * flux dofs numbered after the n_flux_int interior ones: low end, then high
   * end, n_bt faces each, x-fastest over the transverse axes; n_flux counts
   * them (n_flux = n_flux_int + 2 n_bt). */
  int dir_axis;
  int n_flux_int;
  int n_bt;
  /* RT0 element block per axis: c [[a_diag, a_off], [a_off, a_diag]],
   * c = h_a^2 / (6 V k_a): (2, 1) consistent, (3, 0) lumped (grid.py:204-227) */
  double a_diag;
  double a_off;
} bddc_geom;

const char* bddc_last_error(void);
int bddc_version(void);

/* ---------------------------------------------------------------- dense */

/* C[b] = alpha op(A[b]) op(B[b]) + beta C[b], row-major FP64 on DMMA
 * (mma.sync m8n8k4 f64).  upper != 0 computes only tiles on/above the
 * diagonal.  Replaces the dense BLAS products of coarse.py:179-185 and
 * adaptive.py:123-137. */
/* Same with per-batch live sizes: dims[b*dstride + 0..2] = (M_b, N_b, K_b) <= (M, N, K);
 * operands beyond them read as zero, output tiles entirely outside are
 * zero-filled when beta == 0 and left untouched otherwise. */
int bddc_dgemm_batched_dims(int transA, int transB, int M, int N, int K, double alpha,
                            const double* A, int lda, long long sA, const double* B, int ldb,
                            long long sB, double beta, double* C, int ldc, long long sC,
                            int batch, int upper, const int* dims, int dstride, void* stream);
int bddc_dgemm_batched(int transA, int transB, int M, int N, int K, double alpha,
                       const double* A, int lda, long long sA, const double* B, int ldb,
                       long long sB, double beta, double* C, int ldc, long long sC, int batch,
                       int upper, void* stream);

/* In-place inverse of a batch of SPD matrices (Cholesky, triangular inverse,
 * V V^T; recursive DMMA GEMMs above leaves of order <= b, b <= 64); replaces
 * SuperLU splu (substructure.py:66, coarse.py:159) and the dense coarse
 * lu_factor (coarse.py:196).  info (zero on entry) receives 1 + the batch index
 * of a matrix that met a non-positive pivot (0: all SPD). */
size_t bddc_spd_inverse_workspace(int n, int batch, int b);
/* Tuning knob: bit 0 = register leaves (32 / 64, default on; off = shared-memory
 * leaf), bit 1 = 64-leaf Cholesky and triangular inverse as two kernels (default on). */
void bddc_set_leaf_regs(int on);
int bddc_spd_inverse_batched(double* M, int n, int ld, long long sM, int batch, int b, void* ws,
                             int* info, void* stream);
/* In-situ timing log of the batched SPD inverses (bench's factorisation roofline
 * from the setup's own calls, i.e. the factorisations replacing substructure.py:66
 * and coarse.py:159, 196): enable (clears the log), then read entries
 * {n, batch, flags, ms} (events recorded on each call's stream). */
void bddc_spd_log_enable(int on);
int bddc_spd_log_read(double* out, int max_entries);
/* flags & 1: the caller reads the upper triangle only (no lower mirror pass). */
int bddc_spd_inverse_batched_ex(double* M, int n, int ld, long long sM, int batch, int b, void* ws,
                                int* info, int flags, void* stream);

/* ------------------------------------------------------- local operators */

/* Interface topology of a box partition built on the device in closed form
 * (decomposition.py:32-125: gamma_dofs, faces, signs; solver.py:92-93 _local_pos).
 * face_base[i] = number of faces (i', j') with i' < i (host prefix sum over N).
 * Out: nG (N), gpos / gcode (N x maxG, -1 padded; code = axis | side << 2 |
 * line << 3, side 1 = the +axis normal points out), fslot (N x 6 x maxF), gown
 * (n_gamma x 2 broken slots: [side-1 copy, side-0 copy]), gamma (global dof ids,
 * increasing), gface (face index per interface dof), cell_sub (n_cells). */
int bddc_topology_box(const bddc_geom* g, const int* face_base, int* nG, int* gpos, int* gcode,
                      int* fslot, int* gown, int* gamma, int* gface, int* cell_sub, void* stream);
/* solver.py:286-298: *flag = 1 when some face has max k (low-side cells) / min k
 * (high-side cells) outside [1e-3, 1e3].  faces: n_faces x 4 (i, j, axis, m). */
int bddc_face_jumps(const bddc_geom* g, const int* faces, const double* k, int* flag, void* stream);

/* c_a = h_a^2 / (6 V k_a) per cell (grid.py:204-227, 270-291). coef: 3 x n_cells
 * (one contiguous array per axis: coalesced rows in the stencil and line solves). */
int bddc_cell_coeffs(const bddc_geom* g, const double* k, double* coef, void* stream);
/* delta per interface slot (decomposition.py:212-239), N x maxG. */
int bddc_weights(const bddc_geom* g, int stiffness, const double* coef, const int* gcode,
                 double* delta, void* stream);
/* D_i = mean diag(A) over dofs touching subdomain i (grid.py:344-357). */
int bddc_rescale(const bddc_geom* g, const double* coef, double* Dsub, void* stream);

/* Interior KKT elimination (substructure.py:25-70) for all subdomains: the
 * Jacobi-scaled pressure Schur Ps = D^-1/2 (B_I A_II^-1 B_I^T) D^-1/2 + v v^T
 * (maxP^2 each, identity padded; scl = N x (maxP+1) scaling), the line-compact
 * G = B_G - B_I A_II^-1 A_IG (maxG x maxL) and S_A. */
int bddc_local_build(const bddc_geom* g, const double* coef, const int* fslot, double* P, double* Gc,
                     double* SAd, int* SApart, double* SAoff, double* scl, void* stream);
/* Q = P^+ from the inverse of Ps (in place). */
int bddc_local_pinv_fix(const bddc_geom* g, double* P, const double* scl, void* stream);
/* Dense S_i = sym(S_A + G^T Q G), identity padded (substructure.py:90-99). */
int bddc_local_schur(const bddc_geom* g, const int* gcode, const double* Q, const double* Gc,
                     const double* SAd, const int* SApart, const double* SAoff, double* Wt,
                     double* S, void* stream);

/* Batched interior KKT solves (substructure.py:72-116): harmonic_extend,
 * trace_solve, condense and the interior recovery (solver.py:375-382).
 * Q is tile-packed symmetric (bddc_pack_sym with n = maxP). */
typedef struct bddc_local_solve_args {
  const double* f_flux;   /* global flux vector read at interior dofs (or NULL) */
  double f_scale;
  const double* g_cell;   /* global cell vector in D-scaled units (or NULL) */
  double g_scale;
  const double* x_gamma;  /* continuous interface vector (indexed like gamma) or NULL */
  double x_scale;
  double* u_out;          /* global flux vector: interior dofs written */
  int u_mode;             /* 0: set, 1: add */
  double* rg_broken;      /* if non-NULL: A_IG^T u_I + B_G^T p per slot (N x maxG) */
  double* p_out;          /* if non-NULL: local pressures per cell */
  /* optional second right-hand side sharing f_flux and x_gamma but with the cell
   * load g_cell2 (Step 2's harmonic extension and trace solve, solver.py:326-335):
   * both solves read the packed pressure Schur inverse once; its interior fluxes
   * go to u_out2 (set) */
  const double* g_cell2;
  double g_scale2;
  double* u_out2;
} bddc_local_solve_args;
int bddc_local_solve(const bddc_geom* g, const double* coef, const int* gcode, const int* gpos,
                     const int* fslot, const double* Q, const double* Dsub,
                     const bddc_local_solve_args* a, void* stream);

/* -------------------------------------------------------------- adaptive */

/* Reduced pair eigenproblems on every face (adaptive.py:63-138), selection
 * of eigenvalues > tau, harvested rows and the reference's dependence
 * filter (adaptive.py:141-173, coarse.py:61-100); omega per face
 * (adaptive.py:56-60).  lam_out holds, per face, the eigenvalues in descending
 * order as far as the selection needs them (all above tau and the next one);
 * the remaining entries are NaN.  flist (nlist face ids, each with at most mmax
 * shared dofs) restricts the launch to a size class; NULL = every face.
 * full != 0 resolves the whole reduced spectrum (eigs-report). */
size_t bddc_pair_scratch_bytes(int n_faces);
/* MsMFEM baseline rows (adaptive.py:207-262) in Schur form, one per face:
 * rg = interface residuals (N x maxG) of the interior solutions for each
 * subdomain's unit source distribution; writes rows/qbasis like
 * bddc_pair_eigs (maxsel >= 1) and nadd (0/1) per face. */
int bddc_multiscale_rows(const bddc_geom* g, const int* faces, const int* fslot, const double* S,
                         const double* rg, int maxsel, double* rows, double* qbasis, int* nadd, int* err,
                         void* stream);
int bddc_pair_eigs(const bddc_geom* g, const int* faces, const int* fslot, const double* S,
                   const double* Sinv, const double* delta, double tau, int maxsel, double* lam_out,
                   int lam_ld, int* nsel, int* nadd, double* rows, double* omega, double* scratch,
                   double* qbasis, int* err, const int* flist, int nlist, int mmax, int full,
                   void* stream);

/* ---------------------------------------------------------------- coarse */

/* Per-subdomain coarse pieces (coarse.py:130-185, 237-245): Kc, Psi_Gamma^T, the
 * Delta-solve operator T (cancellation-free projected form) and the B0 row. */
int bddc_coarse_local(const bddc_geom* g, const int* sub_rows, const int* faces, const int* fslot,
                      const int* gcode, const int* nG, const double* rows, const double* qbasis,
                      int maxsel, const double* S, const double* Sinv, const double* Dsub, int maxC,
                      double* Ct, double* Y, double* E, double* gamma, double* Kc, double* Psi,
                      double* T, double* b0, void* inv_ws, int* dims, int* info, int part,
                      void* stream);
int bddc_pad_identity(double* M, int n, int npad, void* stream);

/* Nested-dissection multifrontal coarse solver (replaces the dense coarse
 * lu_factor / lu_solve of coarse.py:186-215; see coarse_nd.py). */
int bddc_nd_assemble(int m, int S, int Sf, int B, int nf, int slot, int K, const int* cmap,
                     const int* ckind, const int* sep_idx, double* F, const double* Fc, int Sc,
                     int nfc, const double* Kc, const int* sub_rows, const double* b0, int maxC,
                     void* stream);
/* Solves on the compact per-node layout (info = {s, bf, sep_ptr, bnd_ptr, cb_off}). */
/* tasks are triplets {node, row0, row1}; fwd gathers the level's separator
 * right-hand sides into rsbuf (ysize entries) first.  xdirect != NULL (a level
 * whose nodes have no boundary, i.e. the root): the separator solution is final
 * after the forward sweep and is written to x directly (no bwd for that level). */
/* cown != NULL: the right-hand side is not read from r but formed on the fly from
 * the per-subdomain restriction rows v (r[g] = v[cown[2g]] - v[cown[2g+1]] for the
 * nfc flux dofs, 0 for the pressures: the preconditioner's coarse load,
 * coarse.py:225-235), so no assembled rhs is written first. */
int bddc_nd_fwd(int ysize, int ntasks, int smax, const int* tasks, const int* info,
                const long long* data_off, const int* sep_flat, const int* lptr, const int* lsrc,
                const double* Fc, const double* r, const double* v, const int* cown, int nfc,
                double* rsbuf, double* ybuf, double* cbuf, double* xdirect, void* stream);
/* bwd: wpr (1, 2, 4, 8) warps share one separator row (tasks then hold 8/wpr rows per pass). */
int bddc_nd_bwd(int ntasks, int bfmax, int wpr, const int* tasks, const int* info,
                const long long* data_off, const int* sep_flat, const int* bnd_flat, const double* Fc,
                const double* ybuf, double* x, void* stream);
int bddc_nd_compact(int m, int S, int Sf, int nf, int B, const double* F, const double* X,
                    const int* info, const long long* data_off, double* Fc, void* stream);
/* Quasi-definite pivot blocks [flux (Sf) | eliminated pressures (Sp)]: mode 0 negates
 * the pressure block, mode 1 mirrors the off-diagonal block into the upper right. */
int bddc_nd_qd(int mode, int m, int Sf, int Sp, int nf, double* F, void* stream);
int bddc_fill(long long n, double v, double* a, void* stream);

/* ------------------------------------------------------------------- PCG */

/* y_b = M_i (win .* gather(x)) per subdomain (solver.py:103-107 schur_matvec,
 * solver.py:114-124 Delta part of precondition). */
int bddc_gather_gemv(int N, int maxG, const int* nG, const int* gpos, const double* Mats,
                     const double* x, const double* win, double* yb, void* stream);
/* Tile-packed symmetric storage (32x32 upper tiles; only the upper triangle of
 * `full` is read) and the gathered symmetric GEMV used for S_i and T_i in the
 * PCG loop (same contract as bddc_gather_gemv). */
size_t bddc_sym_packed_elems(int maxG);
int bddc_pack_sym(int N, int maxG, const double* full, double* packed, void* stream);
int bddc_gather_symv(int N, int maxG, const int* nG, const int* gpos, const double* packed,
                     const double* x, const double* win, double* yb, int grid, void* stream);
/* Tuning knob: subdomains taken at a time per CTA by the grid-stride launch (1, 2, 4). */
void bddc_set_symv_groups(int g);
/* 16 x 16-tile variant for small subdomains (maxG <= 256, a multiple of 16): the
 * packed bytes follow the live triangle more closely than 32-tiles. */
size_t bddc_sym_packed16_elems(int maxG);
int bddc_pack_sym16(int N, int maxG, const double* full, double* packed, void* stream);
int bddc_gather_symv16(int N, int maxG, const int* nG, const int* gpos, const double* packed,
                       const double* x, const double* win, double* yb, int grid, void* stream);
/* v_i = Psi_i^T (win .* gather(x)) (coarse.py:225-235 weighted_restriction); PsiT is
 * stored maxC x maxG per subdomain. */
int bddc_gather_gemv_t(int N, int maxG, int maxC, const int* nG, const int* nC, const int* gpos,
                       const double* PsiT, const double* x, const double* win, double* v,
                       void* stream);
int bddc_coarse_restrict(int nfc, const int* cown, const double* v, double* rhs, void* stream);
/* out_b = wout .* (y_b + Psi_i sigma x_c) (coarse.py:217-223 local_combination). */
int bddc_prolong(int N, int maxG, int maxC, const int* nG, const int* nC, const int* sub_rows,
                 const double* PsiT, const double* xc, const double* yb, const double* wout,
                 double* outb, void* stream);
/* y = sum over both copies (solver.py:100-101 scatter_add). */
int bddc_scatter(int n_gamma, const int* gown, const double* yb, double* y, void* stream);
/* Balanced projection (solver.py:166-179) as I - Phi^T (Phi Phi^T)^+ Phi. */
int bddc_phi(int N, int maxG, const int* nG, const int* gpos, const int* gcode, const double* y,
             double* phi, void* stream);
/* Same on the unassembled per-slot values yb (the scatter_add of solver.py:100-101
 * fused into the reads; net_flux_matrix solver.py:132-144). */
int bddc_phi_broken(int N, int maxG, const int* nG, const int* gpos, const int* gcode, const int* gown,
                    const double* yb, double* phi, void* stream);
int bddc_lap_solve(int S0, int S1, int S2, const double* eig, const double* dm, const double* phi,
                   double* z, void* stream);
/* Same, multi-CTA: six mode-product launches (PDL), ws = 2 N doubles. */
int bddc_lap_solve_mc(int S0, int S1, int S2, const double* eig, const double* dm, const double* phi,
                      double* z, double* ws, void* stream);
int bddc_proj_apply(int n_gamma, int maxG, const int* gown, const double* z, double* y,
                    void* stream);
/* PCG pieces (solver.py:186-233): fused deterministic dots with scalar ops,
 * vector updates, dense GEMV, Lanczos kappa (solver.py:236-251). */
size_t bddc_dot_workspace(void);
int bddc_dot(const double* x, const double* y, long long n, void* ws, double* scal, int op,
             double* hist, void* stream);
int bddc_cg_update(long long n, const double* scal, double* x, const double* p, double* r,
                   const double* Ap, void* stream);
int bddc_p_update(long long n, const double* scal, const double* z, double* p, void* stream);
/* Dense (Phi Phi^T)^+ of the separable subdomain-grid Laplacian (setup; ws holds
 * 2 N^2 doubles, N = S0 S1 S2): Lp = Dm W Lambda^+ W^T Dm, W = Qx (x) Qy (x) Qz. */
int bddc_lap_dense(int S0, int S1, int S2, const double* eig, const double* dm, double* ws, double* Lp,
                   void* stream);
int bddc_gemv(int n, int ld, int ncol, const double* M, const double* x, double* y, void* stream);
/* The same product for a static M (written by no kernel queued before the call, e.g. the
 * balance operator of solver.py:166-179 built at setup), launched as a programmatic
 * dependent launch inside the PCG chain. */
int bddc_gemv_static(int n, int ld, int ncol, const double* M, const double* x, double* y, void* stream);
/* Tuning knob for bddc_gemv: warps per row (1, 2, 4, 8; 0 = automatic by shape). */
void bddc_set_gemv_wpr(int wpr);
/* Tuning knob: threads per CTA (256 or 512) of grid-stride bddc_gather_symv launches. */
void bddc_set_symv_threads(int t);
/* Tuning knob: threads per CTA (256 or 512) of bddc_pair_eigs launches whose
 * faces need more than half an SM's shared memory (default 512). */
void bddc_set_pair_threads(int t);
/* Tuning knob: bddc_prolong streams PsiT straight from HBM (1, default) or
 * through cp.async-staged shared-memory chunks (0). */
void bddc_set_prolong_direct(int on);
int bddc_lanczos(int m, const double* al, const double* be, double* work, double* out,
                 void* stream);
int bddc_axpby(long long n, double a, const double* x, double b, double* y, void* stream);

/* Device-resident PCG loop (solver.py:204-227): a CUDA graph with a
 * conditional WHILE node whose body is one captured PCG iteration. */
int bddc_graph_begin(void** state_out, void* stream);
int bddc_graph_while(void* state, void* stream);
int bddc_graph_end(void* state, void* stream);
int bddc_graph_launch(void* state, void* stream);
int bddc_graph_destroy(void* state);
unsigned long long bddc_graph_handle(void* state);
int bddc_pcg_cond(void* state, const double* scal, double tol, int maxit, void* stream);

/* --------------------------------------------------------------- stencil */

/* Matrix-free RT0 flux mass apply (grid.py:294-307): y = alpha A u + beta y. */
int bddc_flux_A(const bddc_geom* g, const double* coef, const double* u, double alpha, double beta,
                double* y, void* stream);
/* out = s_f f + s_b D (B u) (grid.py:310-324, solver.py:337). */
int bddc_cell_div(const bddc_geom* g, const double* u, const double* fvec, double s_f, double s_b,
                  const int* cell_sub, const double* Dsub, double* out, void* stream);
/* y = alpha B^T p + beta y. */
int bddc_grad(const bddc_geom* g, const double* p, double alpha, double beta, double* y,
              void* stream);
/* Pressure recovery (solver.py:254-274) via DCT Neumann solve. */
int bddc_dct_init(const bddc_geom* g, double* dct, void* stream);
int bddc_neumann_solve(const bddc_geom* g, const double* dct, double* rhs, double* tmp,
                       void* stream);
int bddc_sub_mean(long long n, const double* sum, double* v, void* stream);

/* Per-subdomain sums of a cell vector (solver.py:318 rq, 351-352 targets). */
int bddc_sub_sum(const bddc_geom* g, const double* v, double* out, double scale, const double* Dsub,
                 void* stream);
/* Interface <-> flux vector moves: mode 0 set, 1 add, 2 gather into gv. */
int bddc_gamma_flux(int n, const int* gamma, double* gv, double* flux, int mode, void* stream);
/* balanced_shift (solver.py:146-164) from the unit-Laplacian solve z. */
int bddc_face_shift(int n, int n_faces, const int* gface, const int* faces, const double* z,
                    double* w, void* stream);

/* fs = D f (grid.py:250-251). */
int bddc_scale_cells(const bddc_geom* g, const double* f, const int* cell_sub, const double* Dsub,
                     double* out, void* stream);

/* Same product, persistent and bulk-streamed: `grid` CTAs (<= 0: one per SM)
 * take subdomains from a ticket counter; each streams its live packed tiles
 * with cp.async.bulk into an mbarrier-tracked shared-memory ring.  `sched`:
 * two ints, zero before the first call, owned by one call site (the kernel
 * re-arms them).  Replaces schur_apply / delta_solve loops (solver.py:103-128). */
int bddc_gather_symv_bulk(int N, int maxG, const int* nG, const int* gpos, const double* packed,
                          const double* x, const double* win, double* yb, int grid, int* sched,
                          void* stream);

/* Mode B balance operators (solver.py:146-179 on the floating set): the two
 * padded face-graph Laplacians (face-size and unit weights; identity rows for
 * non-floating subdomains) into `out` (2 n^2, zero on entry), and after their
 * batched SPD inverse the N x N operators with zero rows/columns off F. */
int bddc_dirichlet_laplacian(int N, int n, int nfaces, const int* faces, const int* floating,
                             double* out, void* stream);
int bddc_dirichlet_finish(int N, int n, const int* floating, const double* inv, double* out0,
                          double* out1, void* stream);

/* PCG fusions (solver.py:186-233): the balanced projection's apply step
 * y -= Phi^T z fused with the dot x . y, and the CG update x += alpha p,
 * r -= alpha Ap fused with r . r; `op` as for bddc_dot. */
int bddc_proj_dot(int n_gamma, int maxG, const int* gown, const double* z, double* y, const double* x,
                  void* ws, double* scal, int op, double* hist, void* stream);
int bddc_cg_update_dot(long long n, double* x, const double* p, double* r, const double* Ap, void* ws,
                       double* scal, int op, double* hist, void* stream);
/* The same inside the captured PCG loop: the reducing block also sets the WHILE
 * node's condition `cond` (bddc_graph_handle) from relres, breakdown and maxit
 * (solver.py:204-227's loop test), replacing the separate bddc_pcg_cond kernel. */
int bddc_cg_update_dot_cond(long long n, double* x, const double* p, double* r, const double* Ap,
                            void* ws, double* scal, int op, double* hist, unsigned long long cond,
                            double tol, int maxit, void* stream);
/* Scatter fused into the projection (solver.py:100-101 + 166-179):
 * y = (yb[own0] + yb[own1]) - Phi^T z and the PCG dot x . y (solver.py:205-222)
 * (yb: per-slot values, N x maxG, as written by the GEMV / prolongation). */
int bddc_proj_dot_broken(int n_gamma, int maxG, const int* gown, const double* yb, const double* z,
                         double* y, const double* x, void* ws, double* scal, int op, double* hist,
                         void* stream);

/* preconditioned_spectrum (oracle.py:114-141) pieces: w -= Q^T c (Q: k rows of
 * length n), and every eigenvalue of a symmetric tridiagonal (bisection on
 * Sturm counts, ascending; work: m doubles). */
int bddc_gemv_t_sub(int k, int n, const double* Q, const double* c, double* w, void* stream);
int bddc_tridiag_eigvals(int m, const double* d, const double* e, double* work, double* out, void* stream);

size_t bddc_geom_size(void);
/* Kernel launches issued so far (bench.py's gpu_launches). */
unsigned long long bddc_launch_count(void);

/* Page-lock a caller-owned host array in place / release it (solve()'s source
 * upload, solver.py:301 f argument).  A failed registration is cleared from
 * the runtime's error state before returning BDDC_ERR_CUDA. */
int bddc_host_register(void* p, size_t bytes);
int bddc_host_unregister(void* p);

#ifdef __cplusplus
}
#endif
#endif /* BDDC_H */
