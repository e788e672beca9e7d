/*
 * sumfact_b200 — C ABI of the B200-native SIPG sum-factorisation hot path.
 *
 * One shared library (paper_2407_09621_b200/libsumfact_b200.so, sm_100a).  Every
 * entry point takes DEVICE pointers owned by the caller (torch allocates them),
 * plain sizes and a cudaStream_t passed as void*; it only enqueues work and
 * returns 0 or a negative SF_E* code (text in sf_last_error()).  No global
 * mutable state; host-thread-safe across streams.
 *
 * Reference mapping (paths relative to /root/reference/pkg/src/sumfact):
 *   The reference's native plugin point is _core/__init__.py:12-24, which binds
 *   contract_f8/contract_f4 (_core/_contract.pyx:14-45): one batched 1-D
 *   contraction per call on host arrays.  That boundary is μs-grained and
 *   host-resident, so the drop-in sits one level up, at the operator calls the
 *   reference's Python API makes.  Each entry below names the
 *   reference function it replaces.
 *
 * Vectors: flat lexicographic (z, y, x) arrays, x fastest, exactly the
 * reference layout (discretization.py:93-100, 135-145).  Storage dtype is
 * double for mode 0 (fp64) and float for modes 1..3 (precision.py:36-39).
 * Vector pointers and ghost planes must be 16-byte aligned (vector loads and
 * cp.async chunks; cudaMalloc / torch give 256); SF_EINVAL otherwise.
 * Modes: 0 fp64, 1 fp32, 2 fp16, 3 fp16_ec (precision.py:29-33, 206-230).
 * Degrees: k = 1..SF_MAX_DEGREE (K = k+1 nodes per cell and axis).
 */
#ifndef SUMFACT_B200_H
#define SUMFACT_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define SF_ABI_VERSION 5  /* 2: sf_div, SF_LINCOMB_MAX_TERMS; 3: sf_quad_*; 4: sf_smooth_colour_zrange,
                            sf_copy_uncovered; 5: sf_dense_apply */
#define SF_MAX_DEGREE 7

#define SF_OK 0
#define SF_EINVAL (-1)        /* bad argument (reference: ValueError/TypeError/IndexError) */
#define SF_EUNSUPPORTED (-2)  /* degree/mode outside the compiled set */
#define SF_ECUDA (-3)         /* CUDA launch/runtime error */

/* The local cell grid of one level.  nx, ny, nz: cells per axis (even, >= 2).
 * ghost_lo / ghost_hi: optional device arrays holding the K dof planes just
 * below z = 0 / above the top z plane (z-slab decomposition, NCCL halo); NULL
 * means that side is the domain boundary (Nitsche terms). */
typedef struct sf_grid {
  int nx, ny, nz;
  const void* ghost_lo;
  const void* ghost_hi;
} sf_grid;

/* Host-side matrix blocks (double, row-major), built once per level by the
 * Python host from the reference's 1-D matrices (basis.py, discretization.py:108-131):
 *   level_op : M_cell[K*K] | D[K*K] | ucol[K] | urow[K] | bl[K] | br[K]
 *              D = L_smooth[(F,F)][:K,:K], U = F_cross[:K,K:], ucol = U[:,0], urow = U[K-1,:],
 *              bl = (B_left-H_left)[:,0], br = (B_right-H_right)[:,K-1]   (cell-wise form)
 *   patch_eig: V[4][2K][2K] | lam[4][2K]   kind = 2*left_bnd + right_bnd, eigh(L_smooth[kind], M_patch)
 *   embedding: P[2K][K]                     basis.py:243-252
 */

int sf_abi_version(void);
const char* sf_last_error(void);

/* v = A u on the grid (batch vectors at stride nx*ny*nz*K^3).
 * Replaces apply_operator(hier, level, u, mode)            discretization.py:216-266
 * (and, batched over unit vectors, materialize_operator   discretization.py:269-279). */
int sf_vmult(int mode, int k, const sf_grid* grid, const double* level_op, const void* u, void* v, int batch,
             void* stream);

/* v = A u restricted to the cells [z0, z1) along z (even bounds; batch 1): the interior / boundary
 * split of a z-slab vmult, so the interior overlaps the ghost-plane exchange (slab.py). */
int sf_vmult_zrange(int mode, int k, const sf_grid* grid, int z0, int z1, const double* level_op, const void* u,
                    void* v, void* stream);

/* One colour of the multiplicative vertex-patch smoother: x_new = x_old + sum over
 * the colour's patches of P^-1 (b - A x_old)|patch; uncovered cells copied.
 * shift[i] in {0,1} along tensor axis i (x = 0).  x_old != x_new.  x_old = NULL: the current iterate is zero
 * (a V-cycle's first, unshifted colour): r = b, no operator application, bitwise the pass on a zero vector;
 * SF_EINVAL for a shifted colour, SF_EUNSUPPORTED where only the generic kernel applies (degrees other than
 * 7 / 3 / 1, grids the tensor-core tiles do not cover) -- the caller then passes the zero vector.
 * Replaces one iteration of the colour loop of MultigridPreconditioner.smooth
 *                                                          multigrid.py:186-203 (PatchSolver.apply_batch :71-83). */
int sf_smooth_colour(int mode, int k, const sf_grid* grid, const int* shift, const double* level_op,
                     const double* patch_eig, const void* x_old, const void* b, void* x_new, void* stream);

/* One colour restricted to the tiles whose first z cell lies in [z0, z1) (z0 = shift[2] + 2 t, whole 2-cell tiles),
 * WITHOUT the copy of the cells the shifted colour leaves uncovered (sf_copy_uncovered does that once): a z-slab
 * rank runs its interior tiles while the ghost cells are in flight and the boundary tiles after.  Q7 (k = 7) only;
 * SF_EUNSUPPORTED otherwise.  Same operator as sf_smooth_colour                 multigrid.py:186-203. */
int sf_smooth_colour_zrange(int mode, int k, const sf_grid* grid, const int* shift, int z0, int z1,
                            const double* level_op, const double* patch_eig, const void* x_old, const void* b,
                            void* x_new, void* stream);
/* x_new = x_old on the cells a shifted colour does not cover (the last step of sf_smooth_colour). */
int sf_copy_uncovered(int mode, int k, const sf_grid* grid, const int* shift, const void* x_old, void* x_new,
                      void* stream);

/* coarse = R (b - A x) (x != NULL) or R b (x == NULL), R = P^T on each axis.
 * Replaces `r = b - apply_operator(x); restrict(r)`        multigrid.py:249-250, 112-125. */
int sf_residual_restrict(int mode, int k, const sf_grid* fine_grid, const double* level_op,
                         const double* embedding, const void* x, const void* b, void* coarse, void* stream);

/* fine += P e (P on each axis).
 * Replaces `x + prolongate(hier, level-1, e, mode)`        multigrid.py:252, 128-143. */
int sf_prolongate_add(int mode, int k, const sf_grid* coarse_grid, const double* embedding, const void* e,
                      void* fine, void* stream);

/* out = P^-1 in on `count` contiguous (2K)^3 patches (numpy order z,y,x) sharing one boundary
 * kind per axis; kinds[i] for tensor axis i (x = 0), kind = 2*left_bnd + right_bnd.
 * Replaces PatchSolver.apply_batch(w, kinds, mode)          multigrid.py:71-83. */
int sf_patch_apply(int mode, int k, long long count, const int* kinds, const double* patch_eig, const void* in,
                   void* out, void* stream);

/* out[o, i, r] = sum_k m[i, k] u[o, k, r] on device arrays u (outer, n, inner), m (rows, n),
 * out (outer, rows, inner): double for mode 0, float otherwise; ascending k with one rounded
 * multiply and add per term (bitwise contract_f8 / contract_f4), modes applied per operand as
 * contract_mode does.
 * Replaces contract_batch -> _impl.contract_f8 / contract_f4   _core/__init__.py:27-59,
 *          contract_mode                                      precision.py:206-230. */
int sf_contract(int mode, long long outer, int n, long long inner, int rows, const void* m, const void* u, void* out,
                void* stream);

/* ---- vector kernels for FGMRES and the V-cycle boundary (krylov.py:49-137, multigrid.py:262-266) ---- */

/* out = (dtype_out) in, dtype 0 = double, 1 = float.  Replaces np.asarray(x, dtype=...). */
int sf_convert(long long n, const void* in, int in_dtype, void* out, int out_dtype, void* stream);

/* Deterministic (fixed-order, atomic-free) double dot product x.y written to *out_dev.
 * scratch_dev: SF_DOT_SCRATCH doubles of device memory owned by the caller.
 * Replaces `V[i] @ w` and np.linalg.norm's sum of squares   krylov.py:54,73-84. */
#define SF_DOT_SCRATCH 1024
int sf_dot(long long n, const double* x, const double* y, double* out_dev, double* scratch_dev, void* stream);

/* y += coef * x with coef = sign * (*coef_dev) (device scalar, so MGS never syncs the host).
 * Replaces `w = w - H[i, j] * V[i]`                          krylov.py:76,83. */
int sf_axpy_dev(long long n, double sign, const double* coef_dev, const double* x, double* y, void* stream);

/* Fused modified-Gram-Schmidt step: w += sign * (*coef_dev) * x (as sf_axpy_dev), then *out_dev = y . w_new
 * (y == NULL: w_new . w_new), bitwise equal to the separate sf_axpy_dev + sf_dot; one pass over w.
 * Replaces `w = w - H[i, j] * V[i]; H[i + 1, j] = V[i + 1] @ w`     krylov.py:73-84. */
int sf_axpy_dot(long long n, double sign, const double* coef_dev, const double* x, double* w, const double* y,
                double* out_dev, double* scratch_dev, void* stream);
/* *out1_dev = x1 . y and *out2_dev = x2 . y in one pass over y, each bitwise equal to sf_dot;
 * scratch_dev: 2 * SF_DOT_SCRATCH doubles. */
int sf_dot2(long long n, const double* x1, const double* x2, const double* y, double* out1_dev, double* out2_dev,
            double* scratch_dev, void* stream);

/* Largest term count sf_lincomb accepts (larger FGMRES bases fall back to the sf_axpby chain). */
#define SF_LINCOMB_MAX_TERMS 128
/* out = sum_{t < m} coefs[t] * vecs[t] (m <= SF_LINCOMB_MAX_TERMS device vectors, host pointer/coefficient arrays), accumulated in
 * term order as m successive sf_axpby(coefs[t], vecs[t], 1.0, out) from out = 0 -- bitwise -- in one pass.
 * Replaces the FGMRES solution update x = sum_i y_i Z_i        krylov.py:120-124. */
int sf_lincomb(long long n, int m, const double* const* vecs, const double* coefs, double* out, void* stream);

/* y = x / d elementwise (IEEE division, the reference's rounding).  Replaces V = [b / beta] and
 * V.append(w / h_next)                                        krylov.py:57,106. */
int sf_div(long long n, const double* x, double d, double* y, void* stream);

/* y = alpha * x + beta * y (host scalars; y may alias nothing).  Replaces x += y_i Z_i (chain form). */
int sf_axpby(long long n, double alpha, const double* x, double beta, double* y, void* stream);

/* float variant used inside low-precision V-cycles: y = alpha * x + beta * y (fp32). */
int sf_axpby_f32(long long n, float alpha, const float* x, float beta, float* y, void* stream);

/* y = A x, A dense n x n fp64 row-major on the device (n <= 2^20): the coarse-level solve as a product with the
 * explicit inverse of the mode's demoted coarse matrix, one launch per V-cycle.  x_dtype / y_dtype: 0 f64,
 * 1 f32; demote16 != 0 rounds x to binary16 first (the fp16 mode's bs = demote16(bs)).  Deterministic.
 * Replaces scipy.linalg.lu_solve(factor, bs)                     multigrid.py:230-239. */
int sf_dense_apply(long long n, const double* A, const void* x, int x_dtype, int demote16, void* y, int y_dtype,
                   void* stream);

/* ---- device pre/post-processing with general data (discretization.py:317-459) ----
 * Level with n cells per axis, degree k (K = k + 1 nodes), q Gauss points per cell axis (k + 2 or k + 3);
 * a z-chunk of nzc cells starting at global cell z0.  Gauss-point data are tabulated by the caller on the
 * chunk's (nzc q) x (n q) x (n q) point grid (z, y, x); w = the n q per-axis weights (times h).
 *
 * sf_quad_error: *out_dev = sum over the chunk of w_z w_y w_x (I u - fq)^2, I = Sz (x) Sy (x) Sx applied to
 * u (the chunk's cells, flat (z, y, x)); mats = [Sx | Sy | Sz], each q x K (values, or one derivative axis).
 * part_dev: n * n * nzc doubles of scratch (fixed-order two-level reduction).
 * Replaces l2_error / h1_seminorm_error's _quadrature_values + weighted sum   discretization.py:405-459. */
int sf_quad_error(int k, int q, int n, int z0, int nzc, const double* u, const double* mats, const double* fq,
                  const double* w, double* part_dev, double* out_dev, void* stream);
/* sf_quad_load: b (the chunk's cells) = (S^T (x) S^T (x) S^T)(w f) cell by cell; st = S^T (K x q).
 * Replaces assemble_rhs's cell integrals                                        discretization.py:317-348. */
int sf_quad_load(int k, int q, int n, int z0, int nzc, const double* fq, const double* st, const double* w,
                 double* b, void* stream);
/* sf_face_load: b (local slab [z0, z0 + nzc) cells) += Nitsche data term of one domain face: normal tensor
 * axis 0..2, side 0 / 1; g = the face's (n q)^2 point grid (slow, fast tangential axis, global); coef = the
 * K normal coefficients (gamma e0 + d0, or gamma e1 - d1).  Replaces _rhs_boundary   discretization.py:351-394. */
int sf_face_load(int k, int q, int n, int z0, int nzc, int axis, int side, const double* g, const double* st,
                 const double* w, const double* coef, double* b, void* stream);
const char* sf_quad_last_error(void);

/* ---- binary16 primitives of the precision semantics (precision.py:60-197), same cvt as the FP16 kernels ---- */

/* fp32 -> binary16 bit patterns, round to nearest even, subnormals exact, overflow to inf, NaN -> 0x7E00|sign.
 * Replaces precision.to_half                                    precision.py:60-113. */
int sf_to_half(long long n, const float* x, unsigned short* bits, void* stream);
/* binary16 bit patterns -> exact fp32 (NaN -> 0x7FC00000 whatever its sign, as the reference's sign * nan).
 * Replaces precision.from_half                                  precision.py:116-127. */
int sf_from_half(long long n, const unsigned short* bits, float* x, void* stream);
/* fp32 -> binary16 -> fp32 (numpy's float16 cast, NaN payload top bits kept).
 * Replaces precision.demote16                                   precision.py:130-137. */
int sf_demote16(long long n, const float* x, float* out, void* stream);
/* main = to_half(x), residual = to_half((x - from_half(main)) * 2^11); *range_flag_dev |= 1 when some |x| > 65504
 * or x is not finite (the caller raises HalfRangeError).  Replaces precision.ec_split   precision.py:160-167. */
int sf_ec_split(long long n, const float* x, unsigned short* main_bits, unsigned short* resid_bits, int* range_flag_dev,
                void* stream);
/* out (m x n, row-major f32) = A_h B_h + corr / 2^11, corr = A_d B_h (refine 0 both / 1 left) + A_h B_d (0 both /
 * 2 right); A (m x k), B (k x n) given as row-major main / residual half bit patterns, fp32 accumulation.
 * Replaces precision.ec_matmul                                  precision.py:178-197. */
int sf_ec_matmul(int m, int k, int n, const unsigned short* a_main, const unsigned short* a_resid,
                 const unsigned short* b_main, const unsigned short* b_resid, int refine, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SUMFACT_B200_H */
