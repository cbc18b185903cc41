/*
 * helmdef_b200.h -- C-ABI drop-in for the reference's hot path
 *
 *   SolverSetup compose(const DiscreteSystem&, const PrecondSpec&)   inc/precond.hpp:149
 *   GmresResult gmres(op, rhs, start, monitor, const GmresOptions&)   inc/linalg.hpp:41-42
 *
 * called as a pair from run_cell (src/harness.cpp:222-224).  The pair is
 * replaced as one unit: the reference's LinearOp/ResidualFn closures map host
 * Eigen vectors to host Eigen vectors (inc/linalg.hpp:17, 22), so replacing
 * only the closure would force two host<->device copies per operator call.
 * hd_create() does what compose() does at setup (Galerkin multigrid
 * hierarchy, deflation matrix E = Z^T A Z and its exact solver, device
 * buffers); hd_solve() runs the transformed right-hand side, start vector,
 * unrestarted left-preconditioned GMRES with the true-residual monitor and
 * returns the reference's GmresResult fields plus OperationCounts.
 *
 * Plain C: pointers and sizes only, no CUDA or torch types.  Complex vectors
 * are interleaved (re, im) doubles, the layout of Eigen::VectorXcd; 2D index
 * iy*per_dim + ix (x fastest), the reference's kron(outer=y, inner=x) layout
 * (inc/assembly.hpp:37, src/assembly.cpp:255).
 *
 * Errors: a non-zero hd_status; hd_last_error() returns the thread-local
 * message.  This replaces the reference's std::runtime_error on LU failure or
 * zero smoother diagonal (src/linalg.cpp:98-99, src/precond.cpp:98-99, 128);
 * non-convergence is not an error (converged = 0), as in the reference.
 *
 * Threading: one hd_ctx is used by one host thread at a time; distinct
 * contexts may run concurrently (each owns its stream), mirroring the
 * reference's per-cell ownership in the sweep pool (src/harness.cpp:281-307).
 */
#ifndef HELMDEF_B200_H
#define HELMDEF_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HD_OK = 0,
  HD_ERR_INVALID = 1,     /* bad argument / unsupported combination        */
  HD_ERR_CUDA = 2,        /* CUDA runtime / cuBLAS / cuSOLVER failure       */
  HD_ERR_FACTOR = 3,      /* singular coarse operator or zero diagonal      */
  HD_ERR_NO_DEVICE = 4,   /* no CUDA device: there is no CPU fallback       */
  HD_ERR_NONFINITE = 5    /* NaN/Inf residual or Arnoldi norm: the solve
                             stopped (the reference would run on to maxit) */
} hd_status;

/* Wave-number field kinds (WaveField, inc/problems.hpp:18-29), plus the
 * BASELINE config-4 wedge, which the reference's WaveField cannot express
 * (SURVEY.md §0 C8): three layers split by two lines, K2 integrated with the
 * reference's (p+1)-point Gauss rule per direction and k(x,y)^2 sampled at the
 * Gauss points (oracle/helmdef_oracle.py wedge_2d freezes the same rule). */
enum { HD_FIELD_CONSTANT = 0, HD_FIELD_LAYERED = 1, HD_FIELD_WEDGE = 2 };

/* Model problem (helmdef::Problem, inc/problems.hpp:50-60) restricted to the
 * iteration-study problems: point_source_1d / point_source_2d /
 * layered_medium_2d (src/problems.cpp:45-74). */
typedef struct {
  int dim;              /* 1 or 2                                             */
  int order;            /* B-spline degree p                                  */
  int elements;         /* elements per direction                            */
  double k;             /* base wave number                                  */
  int field_kind;       /* HD_FIELD_*                                         */
  double multipliers[16]; /* layered: block(bx,by) = multipliers[4*by+bx];
                             wedge: [0..2] = top, middle, bottom layer        */
  double lines[4];      /* wedge: top iff y > lines[0] + lines[1] x, else middle
                           iff y > lines[2] + lines[3] x, else bottom          */
  int point_source;     /* 0: load at (1/2, 1/2) as the reference
                           (src/assembly.cpp:251-256); 1: at source[]       */
  double source[2];     /* (x_s, y_s) when point_source = 1                   */
} hd_problem;

/* Discrete system as the device consumes it (DiscreteSystem,
 * inc/assembly.hpp:43-52, in factored form).  For dim = 2,
 *   A      = kron(M1, S1) + kron(S1, M1) - K2,
 *   K2     = k^2 kron(M1, M1)                          (constant field)
 *          = sum_{by,bx} (k m_{by,bx})^2 kron(B_by, B_bx) (layered field),
 *          = shift_mass_2d as a general 2D stencil           (wedge field),
 * for dim = 1, A = S1 - k^2 M1 (+ corner at (n-1, n-1)).  Bands are reduced
 * (Dirichlet rows dropped), per_dim x (2*order+1), row-major,
 * band[i*(2p+1) + (j-i+p)] = X(i, j). */
typedef struct {
  int dim;
  int order;
  int elements;
  int per_dim;
  int field_kind;
  double k;
  double multipliers[16];
  const double* stiffness_band;   /* S1                                    */
  const double* mass_band;        /* M1                                    */
  const double* interval_mass;    /* layered: 4 bands B_0..B_3 (else NULL)  */
  double corner_re, corner_im;    /* 1D only: added to A(n-1,n-1)          */
  /* wedge (any non-separable K2): K2 as a 2D stencil, N x (2p+1)^2 doubles,
   * shift_mass_2d[(iy*n+ix)*(2p+1)^2 + (dy+p)*(2p+1) + (dx+p)]
   *   = K2(iy*n+ix, (iy+dy)*n + ix+dx), zero where the neighbour is outside.  */
  const double* shift_mass_2d;
} hd_system;

/* PrecondSpec (inc/precond.hpp:122-130) plus MultigridOptions::coarsest
 * (inc/precond.hpp:57-61). */
typedef struct {
  int deflate;
  double drop;
  int shift;
  double beta2;
  int cycles;          /* >= 1: multigrid V-cycles; <= 0: exact shifted inverse
                          (C_ex, src/precond.cpp:203-211): fast diagonalisation
                          (2D constant k), banded LU (1D), dense or block
                          tridiagonal LU (layered / wedge fields)             */
  int smooth_steps;
  double omega;
  int coarsest;        /* per-dimension size solved directly (reference: 32) */
} hd_precond;

/* GmresOptions (inc/linalg.hpp:24-27). */
typedef struct {
  int max_iterations;
  double tolerance;
} hd_gmres;

/* GmresResult scalars (inc/linalg.hpp:29-34) + OperationCounts
 * (inc/precond.hpp:114-119) + timings. */
typedef struct {
  int iterations;
  int converged;
  long matvecs;
  long coarse_solves;
  long shift_solves;
  long vcycles;
  double t_setup_s;    /* hd_create: device hierarchy + factorisations        */
  double t_solve_s;    /* hd_solve: CUDA-event time of the whole solve          */
  int kernel_launches; /* own device kernels launched by the last hd_solve      */
  int library_calls;   /* cuBLAS calls (coarse fast-diagonalisation GEMMs)     */
} hd_report;

typedef struct hd_ctx hd_ctx;

/* ---- host assembly (mirrors src/assembly.cpp; not accelerated) ---------- */

/* Retained basis functions per direction (src/assembly.cpp:174-184). */
int hd_problem_per_dim(const hd_problem* pb);

/* Assemble the reduced 1D factors and the point-source load vector
 * (src/assembly.cpp:163-258).  stiffness_band / mass_band: per_dim*(2p+1);
 * interval_mass: 4*per_dim*(2p+1) for layered fields (may be NULL otherwise);
 * rhs: 2*per_dim^dim doubles (interleaved complex). */
hd_status hd_assemble(const hd_problem* pb, double* stiffness_band, double* mass_band,
                      double* interval_mass, double* rhs);

/* Non-separable K2 of a wedge problem as the 2D stencil hd_system.shift_mass_2d
 * expects (N x (2p+1)^2 doubles, N = per_dim^2). */
hd_status hd_assemble_field(const hd_problem* pb, double* shift_mass_2d);

/* ---- the drop-in solver ------------------------------------------------ */

/* compose() (inc/precond.hpp:149, src/precond.cpp:196-265): build the
 * preconditioner on one device.  devices/n_devices: the CUDA device to use
 * (NULL/0 = current device).  n_devices > 1 is rejected: the multi-GPU
 * program is one process per GPU, each calling hd_create_dist for its slab. */
hd_status hd_create(const hd_system* sys, const hd_precond* spec, const int* devices,
                    int n_devices, hd_ctx** out);

/* compose() on a row-slab decomposition of the 2D grid:
 * nslabs bands of iy rows with halo rows, halo exchange before every apply
 * and transfer, the gather level and the deflation coarse vector assembled
 * whole, reductions combined in slab order -- the multi-GPU program, run here
 * with all slabs on one device (copies for the exchanges).  hd_solve /
 * hd_solve_device / hd_apply then use the slabs.  Constant field, shift with
 * cycles >= 1 (the DC_MG family). */
hd_status hd_create_slabs(const hd_system* sys, const hd_precond* spec, int nslabs, hd_ctx** out);

/* The same slab program with one slab per process (one process per GPU,
 * SURVEY.md §8(e)): this process owns slab `rank` of `nranks` on CUDA device
 * `device`.  Halo rows travel by NCCL send/recv, the gather-level and
 * deflation coarse vectors by NCCL broadcasts from their row owners, the
 * reduction partials by NCCL allgathers combined in slab order (so every
 * process computes the same scalars and takes the same branches).
 * nccl_id: the 128-byte ncclUniqueId from hd_nccl_unique_id on rank 0, passed
 * to every rank by the caller (e.g. a torch.distributed broadcast).  hd_solve
 * takes the whole rhs on every rank and returns the whole x on every rank.
 * NCCL is loaded at run time (dlopen "libnccl.so.2"). */
hd_status hd_nccl_unique_id(unsigned char* nccl_id_out /* 128 bytes */);
hd_status hd_create_dist(const hd_system* sys, const hd_precond* spec, int rank, int nranks,
                         const unsigned char* nccl_id, int device, hd_ctx** out);

/* Slab count of a context (0: single domain); gather_level and the nslabs+1
 * fine row bounds are written when non-NULL. */
int hd_slab_info(const hd_ctx* ctx, int* gather_level, int* bounds);

/* gmres(compose(...)): host buffers.  rhs: 2N doubles; x_out: 2N doubles;
 * residuals_out: max_iterations (+1) doubles (may be NULL).  Includes the
 * host->device copy of rhs and the device->host copy of x. */
hd_status hd_solve(hd_ctx* ctx, const hd_gmres* opt, const double* rhs, double* x_out,
                   double* residuals_out, hd_report* report);

/* Same solve with rhs / x already resident in device memory (device
 * pointers of 2N doubles on the context's device). */
hd_status hd_solve_device(hd_ctx* ctx, const hd_gmres* opt, const double* d_rhs,
                          double* d_x, double* residuals_out, hd_report* report);

/* Exact direct solve x = A^-1 rhs of the unshifted operator on the current
 * device -- the reference's DirectSolver(sys.A).solve(sys.rhs) behind
 * RunRecord::direct_gap (src/harness.cpp:234-238, src/linalg.cpp:94-102):
 * fast diagonalisation (2D constant k), banded LU (1D), dense or block
 * tridiagonal LU (layered / wedge).  Host buffers of 2N doubles; builds and
 * frees a transient context. */
hd_status hd_direct_solve(const hd_system* sys, const double* rhs, double* x_out);

/* Vector length N (= per_dim^dim) and multigrid level count of a context. */
long hd_size(const hd_ctx* ctx);
int hd_levels(const hd_ctx* ctx);

/* Test hooks (device pointers): y = A x (the unshifted operator) and
 * y = MG^-1 x (c V-cycles of the shifted operator) and y = op(x) (the full
 * composed left-preconditioned operator, src/precond.cpp:236-245). */
hd_status hd_apply(hd_ctx* ctx, int which, const double* d_x, double* d_y);
enum { HD_APPLY_A = 0, HD_APPLY_SHIFTED = 1, HD_APPLY_MG = 2, HD_APPLY_PROJECT = 3, HD_APPLY_OP = 4,
       HD_APPLY_Q = 5 };

/* Test hook on multigrid level `level` (device pointers, level sizes):
 *   0: y = M_l x            1: y = omega D_l^-1 x       2: y = x + omega D_l^-1 (x - M_l x)
 *   3: y = x - M_l x        4: y = Z_l^T x (l -> l+1)   5: y += Z_l x (l+1 -> l)
 *   6: y = M_L^-1 x (coarsest level exact solve)                                      */
hd_status hd_debug_level(hd_ctx* ctx, int which, int level, const double* d_x, double* d_y);
int hd_level_size(const hd_ctx* ctx, int level);

/* Run subsequent work of this context on an external CUDA stream
 * (cudaStream_t passed as void*; NULL restores the context's own stream). */
hd_status hd_set_stream(hd_ctx* ctx, void* stream);

/* Per-launch profiling: when enabled, every device launch of the next solves
 * is bracketed by CUDA events on the launch stream and tagged with its kind
 * and algorithmic bytes (compulsory HBM traffic of that launch).  hd_profile
 * (enable) also clears previous records; hd_profile_read sums one kind. */
enum { HD_K_OP_FINE = 0, HD_K_OP_COARSE = 1, HD_K_JACOBI0 = 2, HD_K_TRANSFER = 3, HD_K_EXACT = 4,
       HD_K_MGS = 5, HD_K_ITERATE = 6, HD_K_VEC = 7, HD_K_GIVENS = 8, HD_K_LIBGEMM = 9, HD_K_DGEMM = 10,
       HD_K_COUNT = 11 };
/* (HD_K_DGEMM and HD_K_LIBGEMM record FLOPs, not bytes, in hd_profile_read's "bytes".) */
hd_status hd_profile(hd_ctx* ctx, int enable);
hd_status hd_profile_read(hd_ctx* ctx, int kind, long* launches, double* ms, double* bytes);

/* Memory checking without compute-sanitizer (not available on the GPU pool):
 * with HD_POISON=1 in the environment every device allocation of the library
 * is filled with 0xFF bytes (NaN in every double) and framed by poisoned guard
 * zones, so reads of never-written memory poison the result and out-of-bounds
 * stores change a guard.  Returns the number of changed guards over all live
 * allocations of the process (0 when HD_POISON is unset), -1 on a CUDA error. */
long hd_debug_check_guards(void);

void hd_destroy(hd_ctx* ctx);
const char* hd_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* HELMDEF_B200_H */
