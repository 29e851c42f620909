/* bpqn.h -- C ABI of libbpqn, the B200 (sm_100a) hot path of arXiv 2604.10089
 * ("A Bifidelity Proximal Quasi-Newton Method for Dense Rigid Body Suspension
 * Collision Resolution"): the LCP matrix-vector product w = D^T M D lambda with a
 * boundary-integral Stokes mobility solve inside, and the paper's Mono-PQN /
 * Bi-PQN LCP solvers on top of it.
 *
 * Citations: PAPER.md line numbers (P:n); the discretisation the paper leaves
 * open is fixed by the readings R1..R30 in DESIGN.md ("Readings").
 *
 * Conventions (all entry points):
 *  - Arrays are fp64 unless marked i32.  "_dev" = device pointer (e.g. a torch
 *    tensor's data_ptr()), "_host" = host pointer.  Vectors of rigid-body
 *    quantities are ordered (Fx,Fy,Fz,Tx,Ty,Tz) / (Ux,Uy,Uz,Ox,Oy,Oz) per sphere
 *    (P:71), row-major [Np][6].  Surface densities are [N][3] row-major with node
 *    index m*Nq + k*2p + l (sphere m, polar ring k from the north pole, azimuth l).
 *  - Ownership: the caller allocates and owns every I/O buffer.  The library owns
 *    its workspace (allocated in bpqn_geometry_init, grown in bpqn_contacts) and
 *    frees it in bpqn_geometry_destroy.  The hot calls allocate nothing.
 *  - Streams: all device work is enqueued on `stream` (a cudaStream_t passed as
 *    void*, NULL = legacy default stream).  Calls that return host scalars
 *    (stats, reports, counts) synchronise that stream before returning.
 *  - Threads: a handle is single-owner (not thread-safe); distinct handles may be
 *    used concurrently from different threads.
 *  - Errors: every call returns an int status (BPQN_OK = 0 on success) and sets
 *    a thread-local message readable with bpqn_last_error().  There is no CPU
 *    fallback: without a usable CUDA device every call returns BPQN_ERR_CUDA.
 */
#ifndef BPQN_H
#define BPQN_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BPQN_OK = 0,
  BPQN_ERR_INVALID = 1,   /* null pointer, bad size, p < 2 or p > BPQN_P_MAX, a <= 0, mu <= 0, overlap, lambda < 0 */
  BPQN_ERR_CUDA = 2,      /* CUDA runtime error (message has the CUDA string) */
  BPQN_ERR_OOM = 3,       /* device allocation failed */
  BPQN_ERR_NOCONV = 4,    /* GMRES or PQN reached max iterations; outputs hold the last iterate */
  BPQN_ERR_STALLED = 5,   /* PQN step length vanished twice (after one memory reset) */
  BPQN_ERR_NAN = 6,       /* NaN/Inf detected */
  BPQN_ERR_CAPACITY = 7   /* more contacts than max_contacts (count is still returned) */
};

typedef struct bpqn_geom* bpqn_geom_t;   /* one discretisation (fidelity) over one set of spheres */

/* Discretisation options; NULL -> defaults.  p_s: order of the rotated singular
 * self grid (default 2p, R6).  d_near: target-to-sphere distance below which the
 * refined near rule replaces the coarse rule (default 4 pi a / p, R8).
 * near_n1/near_n2/near_nphi: refined-rule node counts (defaults 2p+16, p+8, 4p). */
typedef struct {
  int p_s;
  double d_near;
  int near_n1, near_n2, near_nphi;
  int build_single_layer; /* 1 (default): also precompute S-kernel near/self data */
  int fmm_order;          /* 0 (default): K1 is the direct all-pairs sum.  3..12: the all-pairs coarse sum is
                             evaluated by a kernel-independent FMM (fmm_order points per edge of the
                             equivalent / check cube surfaces, uniform octree; SURVEY NEXT-4,
                             for N >> 3e5) -- an approximation whose relative error is set by the order
                             (measured: profiles/r02_fmm.md); not with sharding.  Orders 5..8 apply the
                             M2L translations through shared row / column skeletons (tolerance about the
                             order's own error: the compressed order 6 has 2.0e-4 instead of 1.4e-4 on
                             the D layer; environment BPQN_FMM_M2L_TOL=0 keeps them exact;
                             profiles/r02_fmm_m2l.md). */
} bpqn_disc_opts;

/* GMRES options (R9).  NULL -> tol 1e-12 (relative residual), restart 100 (<= 500),
 * max 1000, precond 1.  precond = 1: right block-Jacobi preconditioning by the exact
 * inverse of the same-sphere block (D_self - I/2 + Pi_R, identical for every sphere);
 * right preconditioning leaves the residual -- hence the stopping test -- that of
 * the unpreconditioned system.  0: plain GMRES. */
typedef struct {
  double tol;
  int restart;
  int max_iters;
  int precond;
  int recycle;        /* 1: start from the least-squares combination of this handle's earlier
                         solutions and keep this solve's (rhs, solution) pair (Krylov
                         recycling across the MVPs of one LCP solve).
                         The store holds up to 1024 orthonormalised pairs within min(4 GB, a
                         quarter of the free device memory) per handle; it is allocated (and
                         emptied) by bpqn_gmres_recycle_reset and at the start of bpqn_solve_lcp
                         -- never inside an MVP: without a reserved store recycle = 1 is a no-op.
                         A solve's pair is kept if its new direction has norm > 1e-8 |rhs|.
                         0: off.  BB-PGD takes its step length from differences of consecutive
                         MVPs and is sensitive to the tolerance-level error a recycled initial
                         guess carries: with tol equal to the KKT tolerance it needs more MVPs
                         (c4 DVI steps: 24 against 12) and, combined with relax_fmm, can stagnate
                         -- use recycle = 0 or tol <= 1e-2 eps_kkt for BB-PGD
                         (profiles/r02_dvi_c4_refine.md); Mono-/Bi-PQN are not affected. */
  int relax_fmm;      /* 1: FMM-accelerated refinement on a handle built with fmm_order > 0 (NEXT-4;
                         the paper's far field is an FMM): every Krylov step applies the
                         operator with the FMM far field, each restart cycle reduces its own residual
                         by relax_delta, and every cycle starts from -- and the solve stops only on --
                         the DIRECT residual b - A x (the all-pairs K1).  Defect correction with an
                         approximate inner operator: the returned x meets tol for the direct operator,
                         exactly like relax_fmm = 0 on a direct handle.  Everything outside the Krylov
                         steps (the mobility right-hand side S[f], the residuals) is direct.
                         BPQN_ERR_INVALID on a handle without an FMM.  0 (default): off -- an FMM
                         handle then uses the FMM for every application, a direct handle the direct
                         sum.  Measured: profiles/r02_fmm_refine.md. */
  double relax_delta; /* residual reduction per refinement cycle; <= 0 (default) -> 3e-3 */
} bpqn_gmres_opts;

typedef struct {
  int iters;          /* GMRES (Arnoldi) iterations */
  int restarts;
  double rel_resid;   /* final relative residual estimate ||b - A x|| / ||b|| */
  double ms;          /* device time of the whole call (CUDA events) */
  int applies;        /* operator applications (iterations + restart / initial-guess residuals) */
  int fmm_applies;    /* of which with the FMM far field (relax_fmm, or an FMM handle); with relax_fmm
                         restarts counts the refinement cycles after the first */
} bpqn_gmres_stats;

typedef struct {
  int method;                 /* 0 = Mono-PQN (Alg. 1), 1 = Bi-PQN (Alg. 3),
                                 2 = BB-PGD, the paper's baseline (eq. spectralStepSize) */
  int k_max;                  /* outer iteration cap (default 200) */
  double eps_kkt_abs;         /* ||min(x, Ax+b)||_2 stop, default 1e-10 */
  double eps_kkt_rel;         /* relative KKT stop; <= 0 disables (default 0) */
  double tau;                 /* forward step (R11, default 1) */
  int refresh_period;         /* gradient-cache refresh (R18, default 20) */
  double sub_eps_factor;      /* Bi-PQN subproblem tolerance factor (R22, default 1e-2) */
  int sub_k_max;              /* Bi-PQN subproblem iteration cap (default 50) */
  double prox_tol;            /* Alg. 4 tolerance; <= 0 -> 1e-12 max(1, |x~|_inf) */
  int prox_jmax;              /* Alg. 4 iteration cap (default 100) */
  double curv_skip;           /* BFGS curvature skip threshold (R16, default 1e-12) */
  bpqn_gmres_opts gm_hi, gm_lo;
  double cost_ratio;          /* t_lo/t_hi for E-MVPs; <= 0 -> measured */
  double sub_forcing;         /* Bi-PQN only, default 0 (off, R22): > 0 solves each subproblem to
                                 max(sub_eps_factor eps, sub_forcing * current hi KKT error)
                                 (inexact proximal Newton; not in the paper) */
  int verify_secants;         /* Bi-PQN, test-only (default 0): before every subproblem measure
                                 max_j |B^(k) s_j - y_j|_inf / max(1, |y_j|_inf) over the re-used
                                 secant pairs (reading R34) with extra, uncounted lo MVPs;
                                 reported in bpqn_report.secant_residual */
  int lo_dense;               /* Bi-PQN: 1 = form the low-fidelity LCP matrix A^ = D^T M_lo D once per solve
                                 (all Nc mobility solves as one block GMRES on the dense completed
                                 double-layer operator of `lo`, FP64 GEMMs on the tensor cores; gm_lo's
                                 tolerance per column; R38) and apply it as an Nc x Nc product for
                                 every low-fidelity MVP; falls back to matrix-free lo MVPs if the dense
                                 operator (8 (3 N_lo)^2 bytes) does not fit.  2: auto -- form A^ when at least
                                 a quarter of the b_l are negative (a hard LCP with hundreds of lo MVPs).
                                 0 (default): matrix-free */
  int warm_start;             /* bpqn_dvi_step only: 1 (default) starts each step's LCP from the previous step's
                                 lambda of the same sphere pairs (0 for new pairs) -- Alg. 1 / 3's x^(-1)
                                 (P:336); 0: from lambda = 0.  The solution is the same unique lambda*
                                 (P:190); only the iteration counts change. */
} bpqn_solve_opts;

typedef struct {
  int iterations, hi_mvps, lo_mvps, gmres_iters_hi, gmres_iters_lo;
  double e_mvps, cost_ratio, kkt_abs, kkt_rel, objective, ms_total, ms_hi, ms_lo;
  int termination;            /* 0 KKT_ABS, 1 KKT_REL, 2 MAX_ITER, 3 STALLED */
  double secant_residual;     /* see bpqn_solve_opts.verify_secants (0 otherwise) */
  int lo_mvps_init;           /* Bi-PQN: lo MVPs of the low-fidelity initialisation (Alg. 3 line 1) */
  int lo_dense_columns;       /* lo_dense: columns formed (= Nc; 0 when matrix-free) */
  int lo_dense_gmres_iters;   /* lo_dense: iterations of the batched GMRES */
  double ms_lo_dense;         /* lo_dense: wall time of forming A^ (included in ms_lo and ms_total) */
} bpqn_report;

/* Defaults for the option structs above. */
void bpqn_default_disc_opts(bpqn_disc_opts* o);
void bpqn_default_gmres_opts(bpqn_gmres_opts* o);
void bpqn_default_solve_opts(bpqn_solve_opts* o);

/* Build one discretisation of Np spheres of radius a in fluid of viscosity mu at
 * SH order p (grids R10, projection R7, self quadrature R5/R6, near rule R8):
 * grids, SH analysis, the per-sphere self operators E (FP64 tensor-core GEMM
 * operands) and the per-incidence refined near-rule tensors in SH-coefficient space
 * ([6][nb] per (target node, source sphere) incidence); workspace for GMRES.
 * centers_host [Np][3].  Fails with BPQN_ERR_INVALID if two spheres overlap. */
#define BPQN_P_MAX 25 /* largest SH order: the rule precompute holds 3 ceil(nb/2) <= 1024 tiles, nb = p^2 + 2p */
int bpqn_geometry_init(bpqn_geom_t* out, int n_spheres, const double* centers_host, double radius,
                       double mu, int p, const bpqn_disc_opts* opts, void* stream);
int bpqn_geometry_destroy(bpqn_geom_t g);

/* Sizes of a geometry: N surface nodes, Nq nodes per sphere, near incidences,
 * bytes of device memory held. */
int bpqn_geometry_info(bpqn_geom_t g, int* n_nodes, int* nq, long long* n_incidences,
                       long long* device_bytes);

/* Contact detection (R20): pairs i<j with gap |c_j-c_i| - 2a < gap_threshold,
 * lexicographic.  Writes up to max_contacts entries: pairs_dev [max][2] i32,
 * normals_dev [max][3] (n = (c_j-c_i)/|c_j-c_i|), gaps_dev [max]; *n_contacts_host
 * = total count (BPQN_ERR_CAPACITY if it exceeds max_contacts).  Stores the set in
 * the handle as the contact set of bpqn_lcp_mvp. */
int bpqn_contacts(bpqn_geom_t g, double gap_threshold, int max_contacts, int* n_contacts_host,
                  int* pairs_dev, double* normals_dev, double* gaps_dev, void* stream);

/* Install an explicit contact set (e.g. the hi-fidelity set into the lo-fidelity
 * handle, required by Bi-PQN).  Device arrays as in bpqn_contacts. */
int bpqn_set_contacts(bpqn_geom_t g, int n_contacts, const int* pairs_dev, const double* normals_dev,
                      const double* gaps_dev, void* stream);

/* u = S_full[f] + D_full[q] at all N nodes (the discrete layer operator, O6).
 * f_dev or q_dev may be NULL (treated as zero).  All [N][3]. */
int bpqn_layer_apply(bpqn_geom_t g, const double* f_dev, const double* q_dev, double* u_dev, void* stream);

/* Tangential Janus slip (R13): u_s = -B (a_m - (xi.a_m) xi) where xi.a_m > 0, else 0.
 * axes_host [Np][3] unit axes; slip_dev [N][3]. */
int bpqn_janus_slip(bpqn_geom_t g, const double* axes_host, double B, double* slip_dev, void* stream);

/* Mobility (Fig. 1): (U, Omega) = M_slip(F, T; u_s) by the
 * completed double-layer BIE (R1-R4) solved with device GMRES from q0 = 0.
 * ft_dev [Np][6], slip_dev [N][3] or NULL, uo_dev [Np][6].  st may be NULL. */
int bpqn_mobility_apply(bpqn_geom_t g, const double* ft_dev, const double* slip_dev, double* uo_dev,
                        const bpqn_gmres_opts* gm, bpqn_gmres_stats* st, void* stream);

/* LCP MVP: w = D^T M D lambda for the handle's contact set.
 * lambda_dev, w_dev [Nc]. */
int bpqn_lcp_mvp(bpqn_geom_t g, const double* lambda_dev, double* w_dev, const bpqn_gmres_opts* gm,
                 bpqn_gmres_stats* st, void* stream);

/* b = (Phi + dt D^T U_nc)/dt with U_nc = M_slip(F_nc, 0; u_s) (R14).
 * fnc_dev [Np][3], slip_dev [N][3] or NULL, b_dev [Nc]. */
int bpqn_lcp_b(bpqn_geom_t g, const double* fnc_dev, const double* slip_dev, double dt, double* b_dev,
               const bpqn_gmres_opts* gm, bpqn_gmres_stats* st, void* stream);

/* LCP solve 0 <= A x + b  _|_  x >= 0, A = D^T M D by BB-PGD (o->method == 2),
 * Mono-PQN (lo == NULL or o->method == 0) or Bi-PQN (lo = coarser-p handle over the same
 * spheres with the same contact set).  b_dev [Nc]; lambda_dev [Nc]: in = x_init
 * (>= 0), out = solution.  rep may be NULL. */
int bpqn_solve_lcp(bpqn_geom_t hi, bpqn_geom_t lo, const double* b_dev, double* lambda_dev,
                   const bpqn_solve_opts* o, bpqn_report* rep, void* stream);

/* The whole LCP matrix A = D^T M D of the handle's contact set, row-major [Nc][Nc] into A_host:
 * all Nc mobility solves by right-preconditioned (block) GMRES on the dense completed double-layer
 * operator (8 (3N)^2 bytes of device memory, FP64 GEMMs; gm's tolerance per column).  This is how
 * bpqn_solve_opts.lo_dense forms the low-fidelity A^ (R38); the paper analyses dense A / A^ offline
 * (Fig. 3).  BPQN_ERR_OOM if the dense operator does not fit; N <= 65535 nodes.  st: iters =
 * GMRES iterations (one block GMRES over all Nc columns when 3N >= 100 Nc, each iteration one operator
 * application to all columns; otherwise Nc per-column GMRES processes advancing together), ms = wall time.
 * Synchronises the stream. */
int bpqn_lcp_matrix_dense(bpqn_geom_t g, const bpqn_gmres_opts* gm, double* A_host, bpqn_gmres_stats* st,
                          void* stream);

/* The handle's completed double-layer GMRES operator A_op = -I/2 + D_full + Pi_R (O7) as a dense
 * row-major [3N][3N] matrix written to A_dev (caller-owned, 8 (3N)^2 bytes): A_dev q equals the matrix-free
 * operator applied to q (coarse pairs, refined near rows, self blocks).  Diagnostic / preconditioner
 * studies; N <= 65535, unsharded. */
int bpqn_operator_dense(bpqn_geom_t g, double* A_dev, void* stream);

/* Report of one DVI time step (bpqn_dvi_step). */
typedef struct {
  int n_contacts;           /* candidate contacts (gap < delta) at the start of the step */
  int active_contacts;      /* lambda_l > 0 */
  int solve_rc;             /* bpqn_solve_lcp return code (0 when there were no contacts) */
  double min_gap_before, min_gap_after;
  double ms_total;          /* host wall time of the step */
  bpqn_report lcp;          /* LCP solver report (zeros when there were no contacts) */
  bpqn_gmres_stats gm_nc, gm_c;   /* non-collisional and collisional mobility solves */
} bpqn_step_report;

/* One forward-Euler step of the collision-resolving DVI (eq. dvi; SURVEY
 * NEXT-2) on the spheres of `hi` (and its low-fidelity twin `lo`, or NULL):
 *   contacts (gap < delta) at the current centres;
 *   U_nc = M_slip(F_nc, 0; u_s) with the Janus slip of the current axes (R13, B = slip_B);
 *   b = Phi/dt + D^T U_nc;  lambda from bpqn_solve_lcp(hi, lo, b, x_init, o), x_init = the previous
 *   step's lambda of the same pairs (o->warm_start, default) or 0;
 *   U = U_nc + M D lambda;  c <- c + dt U,  a <- normalise(a + dt Omega x a)
 *   (orientation reading R32; quaternions are out of scope);
 * then both handles are moved to the new centres (bpqn_geometry_update).
 * centers_host, axes_host [Np][3] in/out; fnc_host [Np][3]; uo_host [Np][6] out (U, Omega) or
 * NULL.  Returns the solver's code; BPQN_ERR_INVALID if the step makes spheres overlap (the
 * handles then keep the old centres; reduce dt). */
int bpqn_dvi_step(bpqn_geom_t hi, bpqn_geom_t lo, double* centers_host, double* axes_host, const double* fnc_host,
                  double slip_B, double dt, double delta, const bpqn_solve_opts* o, double* uo_host,
                  bpqn_step_report* rep, void* stream);

/* Move a geometry handle to new centres (same Np, p, a, mu): nodes, near incidences and
 * correction rows are rebuilt; the grid, SH analysis, self operators and the block-Jacobi
 * inverse are kept.  The contact set and the GMRES recycling store are cleared.
 * BPQN_ERR_INVALID if two spheres overlap (the handle is then unusable until updated
 * with valid centres). */
int bpqn_geometry_update(bpqn_geom_t g, const double* centers_host, void* stream);

/* Same solvers on explicit dense operators (test-only; SPEC.md worked examples):
 * A_host, Ahat_host [n][n] row-major (Ahat NULL -> Mono-PQN), b_host, x_host [n]. */
int bpqn_solve_lcp_dense(const double* A_host, const double* Ahat_host, int n, const double* b_host,
                         double* x_host, const bpqn_solve_opts* o, bpqn_report* rep);
/* The same with device arrays (SURVEY 8(b) signature): A_dev, Ahat_dev [n][n] (Ahat NULL -> Mono-PQN),
 * b_dev, x_dev [n] (x: in = x_init, out = solution); all copies on `stream`, which is synchronised. */
int bpqn_solve_lcp_dense_dev(const double* A_dev, const double* Ahat_dev, int n, const double* b_dev, double* x_dev,
                             const bpqn_solve_opts* o, bpqn_report* rep, void* stream);

/* Multi-GPU (one process per GPU): shard the target side of the layer
 * operator.  Rank r of `world` owns spheres [Np r/world, Np (r+1)/world); every operator
 * application computes only the owned rows (K1 targets x all sources, K2 and K3 for the
 * owned spheres), copies them into send_dev (rows = ceil(Np/world) * Nq nodes, [rows][3],
 * zero-padded) and calls allgather(user) once the handle's stream has been synchronised;
 * the callback must fill recv_dev ([world][rows][3], rank-major -- e.g. NCCL
 * all_gather_into_tensor) and return 0.  Everything else (GMRES, contacts, D, PQN) runs
 * replicated on full vectors, deterministically, so all ranks take the same decisions.
 * send_dev / recv_dev / user stay owned by the caller and must outlive the sharding.
 * world = 1 restores the single-GPU operator (symmetric K1). */
int bpqn_geometry_shard(bpqn_geom_t g, int rank, int world, double* send_dev, double* recv_dev,
                        int (*allgather)(void* user), void* user);

/* Symmetric K1 on a sharded handle (after bpqn_geometry_shard with world > 1): instead of the
 * one-directional kernel over the owned target rows, every rank runs an equal share of the
 * symmetric kernel's unordered (target block, source tile) units -- half the pair work of the
 * one-directional split -- whose partial sums cover all rows.  Each operator application then
 * fills rs_send_dev ([world][rows][3], rank-major, rows as in bpqn_geometry_shard, zero-padded)
 * and, after synchronising the handle's stream, calls reduce_scatter(user), which must write
 * into rs_recv_dev ([rows][3]) the element-wise sum over ranks of their chunk for this rank
 * (e.g. NCCL reduce_scatter_tensor) and return 0; K2 / K3 and the all-gather follow as in
 * bpqn_geometry_shard.  Needs Nq >= 32 (p >= 4) and Np <= 4096 (else error 1).  A NULL callback
 * switches back to the one-directional kernel, and so does every later bpqn_geometry_shard
 * call (the buffers are sized for one world).  Buffers and user stay owned by the caller. */
int bpqn_geometry_shard_symmetric(bpqn_geom_t g, double* rs_send_dev, double* rs_recv_dev,
                                  int (*reduce_scatter)(void* user), void* user);

/* Multi-GPU with the library's own NCCL communicator: the same
 * target-side sharding as bpqn_geometry_shard (rank r of `world` owns spheres [Np r/world,
 * Np (r+1)/world)), but the collectives of every operator application -- the reduce-scatter of the
 * symmetric K1 partial sums (symmetric != 0; K1 then runs an equal share of the symmetric kernel's
 * units on every rank) and the all-gather of the owned rows -- are NCCL calls enqueued on the
 * handle's stream: no host synchronisation and no callback; the reduce-scatter overlaps K2.
 * bpqn_nccl_unique_id fills 128 bytes on one rank; the caller distributes them (e.g. a
 * torch.distributed broadcast) and every rank calls bpqn_geometry_shard_nccl with them (collective).
 * world = 1 is allowed (a one-rank communicator: the sharded code path on one GPU).  The library
 * owns the communicator and the exchange buffers (freed by bpqn_geometry_destroy or a later
 * bpqn_geometry_shard call).  NCCL is loaded at run time (libnccl.so.2; the copy the process already
 * has, e.g. torch's); BPQN_ERR_CUDA if it is missing. */
int bpqn_nccl_unique_id(void* uid128);
int bpqn_geometry_shard_nccl(bpqn_geom_t g, int rank, int world, const void* uid128, int symmetric);

/* Reserve (first call: allocate; BPQN_OK with recycling left off if the memory is not there)
 * and empty the GMRES recycling store of a handle (see bpqn_gmres_opts.recycle). */
int bpqn_gmres_recycle_reset(bpqn_geom_t g);

/* Diagnostic (tests; not on the hot path): exhaustive sweep of the MUFU.RSQ64H seed y of
 * rsqrt.approx.ftz.f64 that K1 / K2 refine with a truncated series: for every
 * input rr = 2^e (1 + m) with e in [exp_lo, exp_hi] and every 20-bit high mantissa pattern (the
 * seed reads the high word; the low word's extremes bound e = 1 - rr y^2 monotonically) writes
 * max |1 - rr y^2| to *max_abs_e (host).  Allocates and synchronises the default stream. */
int bpqn_diag_rsqrt_seed(int exp_lo, int exp_hi, double* max_abs_e);

/* Thread-local message for the last non-zero return. */
const char* bpqn_last_error(void);

/* Kernel-level profiling hooks (bench.py).  bpqn_profile_reset(g, 1) clears the
 * counters and makes every later operator application record CUDA events on its
 * stream around K1 (all-pairs), K2 (near) and K3 (self) -- no host sync is added.
 * bpqn_profile_get synchronises on the last event and returns the summed device
 * times (ms) since the reset, the algorithmic GFLOP of the timed K1 launches
 * (DESIGN.md "Roofline"), the number of K1 launches and of all libbpqn kernel
 * launches.  Any output pointer may be NULL. */
int bpqn_profile_get(bpqn_geom_t g, double* ms_allpairs, double* ms_near, double* ms_self,
                     double* allpairs_gflop, long long* allpairs_launches, long long* kernel_launches);
int bpqn_profile_reset(bpqn_geom_t g, int enable_events);

#ifdef __cplusplus
}
#endif
#endif /* BPQN_H */
