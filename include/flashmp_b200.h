/*
 * flashmp_b200.h -- C ABI of the B200-native FlashMP hot path (libflashmp_b200.so).
 *
 * The reference (arXiv 2508.07193 "FlashMP", pure Python package `flashmp`) has no
 * native boundary: its hot path is the duck-typed Python interface
 *     op.apply(list) -> list            ref: pkg/src/flashmp/schwarz.py:377-388
 *     prec.apply(list) -> list          ref: pkg/src/flashmp/schwarz.py:320-339
 *     bicgstab/gmres(op, prec, b, cfg)  ref: pkg/src/flashmp/krylov.py:146, 242
 * backed by numpy/scipy calls.  Each entry point below replaces one of those calls;
 * the Python package `paper_2508_07193_b200` binds them with ctypes and keeps the
 * reference class names and signatures on top.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; all arithmetic is FP64.
 *  - A field is component-major (3, bz, by, bx), x fastest: the reference layout
 *    (ref: pkg/src/flashmp/grid.py:1-14) restricted to one GPU's block.
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous on it.
 *  - Return value: 0 on success, negative on error; fmp_last_error() gives the text.
 *    Nothing on an apply path allocates device memory; callers own every buffer.
 *  - Reductions are deterministic: fixed-order two-level trees, no atomics.
 */
#ifndef FLASHMP_B200_H
#define FLASHMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMP_ABI_VERSION 1

/* ---------------------------------------------------------------- geometry */

/* One GPU's block of the global grid plus its ghost shell.
 * A point (c,k,j,i) in block-local coordinates outside [0,b*) reads
 *   0                       when it lies outside the global box (zero-ghost Dirichlet,
 *                           ref: pkg/src/flashmp/operators.py:1-21), otherwise
 *   ghost[0|1] (x-lo|hi)    shape (3, bz+2P, by+2P, P)   when i is outside,
 *   ghost[2|3] (y-lo|hi)    shape (3, bz+2P, P, bx)      when only j/k are outside and j is,
 *   ghost[4|5] (z-lo|hi)    shape (3, P, by, bx)         when only k is outside.
 * Single-GPU blocks cover the global box and pass NULL ghosts. */
typedef struct fmp_block {
  int64_t bx, by, bz;          /* block extents */
  int64_t gx0, gy0, gz0;       /* global coordinates of the block origin */
  int64_t nx, ny, nz;          /* global extents */
  int64_t halo;                /* ghost width P (>= 1 when any ghost is set) */
  const double* ghost[6];
} fmp_block;

int fmp_abi_version(void);
int fmp_last_error(char* buf, size_t len);
/* Scratch (in doubles) every reduction entry point below needs. */
int64_t fmp_reduce_scratch_doubles(void);
/* Number of kernels this library has launched in the process (cuBLAS calls excluded). */
int64_t fmp_launch_count(void);

/* ---------------------------------------------------------------- stencils (K7/K13)
 * y = x + alpha*(C_b C_f x + Lambda x) with boundary=1, the corrected operator
 *   ref: pkg/src/flashmp/operators.py:167-175 (apply_operator) and the CSR blocks of
 *   DistributedOperator.apply, ref: pkg/src/flashmp/schwarz.py:377-388;
 * boundary is a bit set: FMP_STENCIL_LAMBDA (1) includes Lambda; without it Lambda is dropped
 *   (ref: operators.py:172-173, with_boundary=False); FMP_STENCIL_NO_IDENTITY (2) drops the
 *   identity, y = alpha*(C_b C_f [+ Lambda]) x, so boundary=2 with alpha=1 is the double curl
 *   M x itself (ref: operators.py:128-131, apply_double_curl).
 * mode: 0 = y only; 1 = y and dots[0] = (y, w); 2 = y, dots[0] = (y, w), dots[1] = (y, y);
 *       3 = no y: dots[0] = ||w - A x||^2   (the true-residual check, ref: krylov.py:139-143).
 * dots is a device pointer to >= 2 doubles; scratch has fmp_reduce_scratch_doubles(). */
#define FMP_STENCIL_LAMBDA 1
#define FMP_STENCIL_NO_IDENTITY 2
int fmp_stencil_apply(const fmp_block* blk, double alpha, int boundary, int mode,
                      const double* x, double* y, const double* w,
                      double* dots, double* scratch, void* stream);

/* Split form for overlapping a ghost exchange (multi-GPU): FMP_PART_INTERIOR computes
 * every point whose stencil reads no neighbour ghost cell (call it while the ghosts are in flight),
 * FMP_PART_BOUNDARY the rest plus the fused reductions (call it after they landed).  Both parts
 * together write exactly what fmp_stencil_apply (FMP_PART_ALL) writes, with the same dots. */
#define FMP_PART_ALL 0
#define FMP_PART_INTERIOR 1
#define FMP_PART_BOUNDARY 2
int fmp_stencil_apply_part(const fmp_block* blk, double alpha, int boundary, int mode, int part,
                           const double* x, double* y, const double* w,
                           double* dots, double* scratch, void* stream);

/* out = curl_f(x) (kind 0) or curl_b(x) (kind 1)      ref: operators.py:119-125 */
int fmp_curl(const fmp_block* blk, int kind, const double* x, double* out, void* stream);

/* CN right-hand side R = E + dt*curl_b(H) - (dt^2/4)*C_b C_f E    ref: cn_driver.py:54-59.
 * blkE / blkH carry the ghosts of E and H respectively.  Runs on the SpMV's TMA z-march (E
 * through the plane ring, H read per point); FMP_CN_RHS_POINT=1: thread-per-point kernel. */
int fmp_cn_rhs(const fmp_block* blkE, const fmp_block* blkH, double dt,
               const double* E, const double* H, double* R, void* stream);

/* H_new = H - dt/2 (curl_f(E_new) + curl_f(E_old))               ref: cn_driver.py:90-91 */
int fmp_cn_h_update(const fmp_block* blkNew, const fmp_block* blkOld, double dt,
                    const double* H, const double* E_new, const double* E_old,
                    double* H_new, void* stream);

/* ---------------------------------------------------------------- Krylov vectors (K8)
 * n = number of doubles.  Elementwise results are rounded exactly as numpy evaluates
 * the reference expressions (products and sums rounded separately, no FMA
 * contraction), so they match the reference bit for bit on equal inputs.      */
/* out = a*x + b*y                     ref: krylov.py:120-123 (_Dist.lincomb) */
int fmp_vec_lincomb(int64_t n, double a, const double* x, double b, const double* y,
                    double* out, void* stream);
/* y += a*x                            ref: krylov.py:125-129 (_Dist.axpy_into) */
int fmp_vec_axpy(int64_t n, double a, const double* x, double* y, void* stream);
/* out = a*x                           ref: krylov.py:131-133 (_Dist.scale) */
int fmp_vec_scale(int64_t n, double a, const double* x, double* out, void* stream);
/* out[0] = (x, y)                     ref: krylov.py:108-112 (_Dist.dot) */
int fmp_vec_dot(int64_t n, const double* x, const double* y, double* out,
                double* scratch, void* stream);
/* y += a*x, then dots[0] = (z, y_new); z may equal y (the norm)   ref: krylov.py:301-309
 * (one modified Gram-Schmidt step fused with the next step's inner product) */
int fmp_vec_axpy_dot(int64_t n, double a, const double* x, double* y, const double* z,
                     double* dots, double* scratch, void* stream);
/* out = x + c_0 v_0 + c_1 v_1 + ... evaluated left to right with every product and sum rounded,
 * i.e. the reference's copy + axpy_into loop (ref: krylov.py:348-350) in one pass.
 * v and coef are HOST arrays of k device pointers / coefficients. */
int fmp_vec_combine(int64_t n, const double* x, int k, const double* const* v, const double* coef,
                    double* out, void* stream);
/* BiCGSTAB p-update, in place: p = r + beta*(p + (-omega)*v)   ref: krylov.py:181-182 */
int fmp_bicg_p(int64_t n, const double* r, double* p, const double* v,
               double beta, double omega, void* stream);
/* BiCGSTAB tail: x += alpha*p_hat; x += omega*s_hat; r = s + (-omega)*t;
 * then dots[0] = (r_shadow, r_new) -- the next iteration's rho. ref: krylov.py:213-216, 171 */
int fmp_bicg_xr(int64_t n, double* x, const double* p_hat, const double* s_hat,
                const double* s, const double* t, double* r, const double* r_shadow,
                double alpha, double omega, double* dots, double* scratch, void* stream);
/* The same for x = 0 on entry (BiCGSTAB's first iteration, ref: krylov.py:154 x = zeros_like(b)): x is
 * written without being read, so it needs no zero fill; bit-identical to fmp_bicg_xr on a zeroed x. */
int fmp_bicg_xr0(int64_t n, double* x, const double* p_hat, const double* s_hat,
                 const double* s, const double* t, double* r, const double* r_shadow,
                 double alpha, double omega, double* dots, double* scratch, void* stream);

/* ---------------------------------------------------------------- subdomain solves (K1-K5)
 * A preconditioner plan batches every subdomain of one GPU block.  Subdomains are
 * grouped by extended shape; each shape shares its SVD factors and its dense C^-1.
 * Descriptors are plain int64 records in device memory (layout below). */

typedef struct fmp_subdomain {   /* 16 x int64 */
  int64_t ext[3];        /* extended box extents (ex, ey, ez) */
  int64_t ext_lo[3];     /* extended box origin in block-local coordinates (may be < 0) */
  int64_t own_off[3];    /* owned tile offset inside the extended box */
  int64_t own[3];        /* owned tile extents */
  int64_t shape;         /* index into the shape table */
  int64_t column;        /* column of this subdomain in its shape's Y/Z matrices */
  int64_t ws_off;        /* element offset of this subdomain's 3*V_ext workspace slot */
  int64_t in_off;        /* element offset of this subdomain's input for compact inputs (mode FACES) */
} fmp_subdomain;

typedef struct fmp_shape {       /* 20 x int64 */
  int64_t ext[3];
  int64_t m;             /* boundary-correction size (ref: subdomain.py:235-238) */
  int64_t m_comp[3];     /* rows per component */
  int64_t ut_off[3];     /* offset (doubles) of U^T per axis in the factor buffer */
  int64_t vt_off[3];     /* offset of V^T per axis */
  int64_t s_off[3];      /* offset of the singular values per axis */
  int64_t qw_off;        /* offset of the per-point block-inverse table: (q, w) pairs, point-major,
                            q = 1/(1+alpha|s|^2), w = (1-q)/|s|^2  so  B^-1 y = q y + w s (s.y) */
  int64_t ld;            /* row stride of C^-1 [m][ld], Y and Z [n_s][ld]: m rounded up to 4,
                            padding zero-filled */
  int64_t group;         /* shape whose C^-1, Y and Z this shape shares (itself if canonical).
                            Shapes that are cyclic axis rotations of each other have C matrices
                            equal up to a row/column permutation, so one C^-1 and one GEMM serve
                            the whole group; members use disjoint Y/Z columns (fmp_subdomain.column) */
  int64_t rowmap_off;    /* offset into desc->rowmap of this shape's map from its own correction
                            rows to the group's rows (m int32 entries), or -1 for the identity */
} fmp_shape;
#define FMP_SUBDOMAIN_WORDS 16
#define FMP_SHAPE_WORDS 20

typedef struct fmp_precond_desc {
  double alpha;
  int64_t n_sub, n_shape;
  const fmp_subdomain* subs;     /* device, n_sub records, grouped by shape */
  const fmp_shape* shapes;       /* device, n_shape records */
  const fmp_subdomain* subs_host;/* host copy (launch geometry) */
  const fmp_shape* shapes_host;  /* host copy */
  const int64_t* shape_first;    /* host: first subdomain of each shape (n_shape+1 entries) */
  const double* factors;         /* device: concatenated U^T, V^T, S blocks */
  const double* const* cinv;     /* host array of n_shape device pointers to C^-1, [m][ld]
                                    (members of a group pass the group's pointer) */
  double* work_a;                /* device workspace, >= sum 3*V_ext (+ padding) doubles */
  double* work_b;                /* device workspace, same size */
  double* corr;                  /* device: n_sub * 6 * pmax^2 doubles (correction planes) */
  double* const* ymat;           /* host array of n_shape device pointers, [n_group_cols][ld] each */
  double* const* zmat;           /* host array of n_shape device pointers, [n_group_cols][ld] each */
  int64_t pmax;                  /* max extent over all shapes */
  const int32_t* rowmap;         /* device: concatenated row maps of non-canonical shapes (may be NULL) */
} fmp_precond_desc;

typedef struct fmp_precond fmp_precond;

int fmp_precond_create(const fmp_precond_desc* desc, fmp_precond** out);
int fmp_precond_destroy(fmp_precond* p);

/* Solve modes */
#define FMP_SOLVE_WOODBURY 0  /* full RAS apply: z(owned) = A_i^-1 S_i r   (schwarz.py:320-339) */
#define FMP_SOLVE_EXACT    1  /* (I + alpha M)^-1 only, no boundary correction (subdomain.py:255-262) */
#define FMP_SOLVE_FACES    2  /* Y[:, col] = ((I + alpha M)^-1 r_i)[rows]: C assembly (subdomain.py:196-204) */

/* RAS apply over every subdomain of the block.
 * mode WOODBURY/EXACT: input r is a block field (ghosts in blk), output z is a block
 *   field; each subdomain writes its owned tile (disjoint, so z is fully written when
 *   the owned tiles cover the block).
 * mode FACES: input r holds compact per-subdomain fields at in_off; output goes to
 *   the shape's Y matrices (z unused). */
int fmp_precond_apply(fmp_precond* p, const fmp_block* blk, int mode,
                      const double* r, double* z, void* stream);

/* Split form for overlapping a ghost exchange: FMP_PART_INTERIOR runs the work that reads no
 * neighbour ghost (the forward restriction + x/y transform of the subdomains whose extended boxes
 * stay inside the block), FMP_PART_BOUNDARY everything else.  Call INTERIOR while the ghosts are
 * in flight and BOUNDARY after they landed (same stream); together they equal fmp_precond_apply. */
int fmp_precond_apply_part(fmp_precond* p, const fmp_block* blk, int mode, int part,
                           const double* r, double* z, void* stream);

/* BiCGSTAB's s = r + beta v followed by z = M s (ref: krylov.py:199-201, vec.lincomb(1.0, r,
 * -alpha, v) then precond.apply(s)), as one apply: the forward plane pass forms s per point as
 * each plane of r lands, applies the preconditioner to it and writes s (every owned point, so
 * the whole block).  s and z are bit-identical to fmp_vec_lincomb(n, 1, r, beta, v, s) +
 * fmp_precond_apply(p, blk, mode, s, z).  Blocks with ghosts, FACES mode and plans on the
 * general / large kernels run exactly that two-pass form. */
int fmp_precond_apply_lincomb(fmp_precond* p, const fmp_block* blk, int mode, const double* r,
                              const double* v, double beta, double* s, double* z, void* stream);

/* BiCGSTAB's direction update p_new = r + beta (p_old - omega v) followed by z = M p_new
 * (ref: krylov.py:179-187, two vec.lincomb calls then precond.apply(p)) as one apply, the same
 * way: the forward plane pass forms p_new per point from the landed plane of p_old and writes
 * it.  p_new must be a separate buffer (other subdomains read p_old around the owned tiles while
 * p_new is written).  Bit-identical to copying p_old to p_new, fmp_bicg_p on p_new, then
 * fmp_precond_apply(p_new); blocks with ghosts etc. run exactly that. */
int fmp_precond_apply_bicg_p(fmp_precond* p, const fmp_block* blk, int mode, const double* r,
                             const double* p_old, const double* v, double beta, double omega,
                             double* p_new, double* z, void* stream);

/* ---------------------------------------------------------------- halo exchange (K10)
 * The ghost shell of fmp_block is filled in three phases -- 0: z faces, 1: y faces extended over
 * the z ghosts, 2: x faces extended over both (edges and corners without diagonal messages);
 * side 0 = the low face, 1 = the high face.  ref: the Exchanger messages of schwarz.py:217-257.
 * fmp_halo_slab_doubles: doubles in one slab of the phase (a message is that + 1 tag double).
 * fmp_halo_pack: out[0..n) = the slab this block sends to its neighbour on `side` (read through
 *   the ghosts of the earlier phases already set in blk), out[n] = tag.
 * fmp_halo_unpack: copy a received message (n + 1 doubles) into blk->ghost[slot of phase, side]
 *   unless `in` already IS that slot, and compare its tag with `tag`: a mismatch (lost or stale
 *   message) ORs bit (1 << slot) into *status (device-visible, e.g. pinned host memory; may be
 *   NULL).  Ghost slots must hold n + 1 doubles. */
#define FMP_HALO_Z 0
#define FMP_HALO_Y 1
#define FMP_HALO_X 2
int64_t fmp_halo_slab_doubles(const fmp_block* blk, int phase);
int fmp_halo_pack(const fmp_block* blk, int phase, int side, const double* x, double* out,
                  double tag, void* stream);
int fmp_halo_unpack(const fmp_block* blk, int phase, int side, const double* in, double tag,
                    int* status, void* stream);

/* Stage timing (for benchmarks): enable=1 records CUDA events between the kernels of every
 * later fmp_precond_apply on its stream; fmp_precond_stage_ms synchronises on the last apply's
 * final event and writes up to n per-stage times in ms, in this order:
 *   0 forward plane pass, 1 forward column pass + B^-1, 2 face projections (Y),
 *   3 Y slicing (Ozaki; 0 otherwise), 4 Woodbury GEMM Z = C^-1 Y, 5 correction planes,
 *   6 correction + inverse column pass, 7 inverse plane pass + prolongation.
 * Returns the number of stages written. */
#define FMP_PRECOND_STAGES 8
int fmp_precond_profile(fmp_precond* p, int enable);
int fmp_precond_stage_ms(fmp_precond* p, float* ms, int n);

/* Kernel family the plan runs its transform passes with (diagnostics and tests; no reference
 * counterpart): FMP_PATH_GENERAL (CTA-synchronous kernels, any extent <= 72), FMP_PATH_FAST
 * (warp-independent, <= 2 distinct extents <= 36), FMP_PATH_LARGE (warp-independent, extents
 * 41..72).  FMP_FORCE_GENERAL=1 in the environment at plan creation selects the general path. */
#define FMP_PATH_GENERAL 0
#define FMP_PATH_FAST 1
#define FMP_PATH_LARGE 2
int fmp_precond_path(const fmp_precond* p);

/* Zero-slice skipping of the plan's Ozaki GEMM: out[0] = fraction of the C^-1 INT8 slice blocks
 * streamed, out[1] = fraction of the dense MMA work (28 slice products per chunk) issued.  The
 * all-zero slice blocks (leading digits of entries far from the diagonal, whole zero K chunks)
 * are skipped, which changes no bit of the result (diagnostics and tests; no reference
 * counterpart).  1.0 for the cuBLAS / own GEMMs or with FMP_OZ_DENSE=1.  Returns the number of
 * values written (<= n). */
int fmp_precond_ozaki_stats(const fmp_precond* p, double* out, int n);

/* Diagnostics: with FMP_OZ_PROF=1 in the environment, the last Ozaki GEMM launch's per-CTA
 * MMA-issuer cycles {total, waiting for operand stages, waiting for the epilogue, tiles} for the
 * first n CTAs (tools/oz_prof.py).  Returns -1 when profiling is off. */
int fmp_debug_ozaki_prof(long long* out, int n);

/* Restriction only: out[ws_off(i) ...] = S_i^gamma r for every subdomain i, in the
 * reference's extended-vector order (ref:schwarz.py:217-257).  out has the plan's
 * workspace size.  Exposes the index maps of the fused solve for bit-exact tests. */
int fmp_precond_restrict(fmp_precond* p, const fmp_block* blk, const double* r, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FLASHMP_B200_H */
