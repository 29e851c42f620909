// Internal declarations of libbpqn (B200 / sm_100a).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/bpqn.h"

namespace bpqn {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};
#define BPQN_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::bpqn::Error{e_ == cudaErrorMemoryAllocation ? BPQN_ERR_OOM : BPQN_ERR_CUDA,    \
                          std::string(#call) + ": " + cudaGetErrorString(e_)};               \
  } while (0)
#define BPQN_CHECK_LAUNCH() BPQN_CUDA(cudaGetLastError())
#define BPQN_REQUIRE(cond, msg)                                  \
  do {                                                           \
    if (!(cond)) throw ::bpqn::Error{BPQN_ERR_INVALID, (msg)};   \
  } while (0)

// ---------------------------------------------------------------- device buffer
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    BPQN_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  size_t bytes() const { return n * sizeof(T); }
};

// ---------------------------------------------------------------- geometry
// Host-side description of the order-p grid (reading R10): (p+1) Gauss-Legendre
// nodes in t = cos(theta) (descending), 2p equispaced phi.
struct Grid {
  int p = 0, nq = 0;
  std::vector<double> t, omega, theta, phi;  // [p+1], [p+1], [p+1], [2p]
  std::vector<double> xi;                    // [nq][3] unit normals
  std::vector<double> w;                     // [nq] area weights (a^2 omega pi/p)
};
void gauss_legendre_desc(int n, std::vector<double>& t, std::vector<double>& w);
void build_grid(int p, double a, Grid& g);
int sh_count(int p);  // dim V_p = p^2 + 2p

// Kernel timing for bench.py: when enabled, every operator application records
// 4 events (no host sync); bpqn_profile_get synchronises once and sums them.
struct Profile {
  bool events = false;
  std::vector<cudaEvent_t> pool;  // groups of 5 per operator application (layer.cu)
  size_t used = 0;
  double ms_allpairs = 0, ms_near = 0, ms_self = 0;
  double allpairs_flop = 0;       // algorithmic flops of the timed K1 launches
  long long allpairs_launches = 0, launches = 0;
};

// One GMRES restart cycle as a CUDA graph (gmres.cu): a conditional WHILE node whose body is
// one Arnoldi step; valid for one set of buffer addresses / restart length / preconditioner flag.
struct CycleGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle h = 0;
  cudaStream_t cap = nullptr;
  bool ok = true, warm = false, pre = false;
  int m = -1;
  const void *V = nullptr, *S = nullptr, *red = nullptr;
  long long launches = 0, k1 = 0;  // kernel launches / K1 launches per step
  void clear() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    m = -1;
    warm = false;  // the next cycle runs uncaptured first (attribute setup for new sizes)
  }
  ~CycleGraph() {
    clear();
    if (cap) cudaStreamDestroy(cap);
  }
};

// Launch layout of the last symmetric K1 launch: how k_row_reduce finds its partial sums.
struct K1Layout {
  bool sym = false;  // symmetric kernel (else the one-directional kernel over rows t0..)
  int ks_b = 0, tpb = 0, nt = 0, nb = 0, grid = 0, t0 = 0;
  long long ubeg = 0, units = 0;
  size_t psrc_ld = 0;
};

struct Geom {
  int np = 0, p = 0, nq = 0, n = 0, nb = 0;
  double a = 1, mu = 1, d_near = 0;
  int p_s = 0, n1 = 0, n2 = 0, nphi = 0;
  bool single_layer = true;
  int sms = 148;
  std::vector<double> centers;  // host [np][3]
  Grid grid;

  // static node data
  DBuf<double> X;        // [N][3] node positions
  DBuf<double> src;      // [N][8] {y0,y1,y2,w, n0,n1,n2,0}
  DBuf<double> centers_d;// [np][3]
  DBuf<double> xi_d;     // [nq][3]
  DBuf<double> w_d;      // [nq]
  DBuf<double> analysis; // [nb][nq] SH analysis (projection = Ynodes * analysis)

  // self operators, row-major [3nq][3nq]
  DBuf<double> E_S;   // S_self - naive same-sphere Stokeslet
  DBuf<double> E_L;   // D_self - naive same-sphere stresslet (layer operator)
  DBuf<double> E_A;   // E_L - I/2 + Pi_R (GMRES operator)
  DBuf<double> Minv;  // inverse of the same-sphere block D_self - I/2 + Pi_R (block-Jacobi, K4)

  // near incidences (target i, source sphere m), sorted by (i, m)
  long long n_inc = 0;
  DBuf<int> inc_t, inc_m;        // [n_inc]
  DBuf<int> nt_list, nt_ptr;     // near targets (unique) and CSR into incidences
  int n_near_targets = 0;
  // K2 order: the same incidences sorted by (m, i), cut into chunks of <= K2_CHUNK positions
  // of one source sphere; refined-rule tensors in SH-coefficient space, symmetric (a, c)
  // packed xx xy xz yy yz zz: u_i[a] += sum_c sum_b T[pos][sym(a,c)][b] coef_m[b][c]
  DBuf<int> cm_t, cm_m;          // [n_inc] target node / source sphere per position
  DBuf<int> chunks;              // [n_chunks][2] position ranges
  int n_chunks = 0;
  DBuf<double> T_S, T_D;         // [n_inc][6][nb'], nb' = nb rounded up to even (zero pad)
  DBuf<double> coef;             // [2][KC_Z][np][nb'][3] SH coefficients of the densities, per node slab (K2)

  // contacts
  int nc = 0, nc_cap = 0;
  DBuf<int> pairs;        // [cap][2]
  DBuf<double> normals;   // [cap][3]
  DBuf<double> gaps;      // [cap]

  // workspaces (all allocated at init / update: the hot calls allocate nothing)
  DBuf<double> packed;   // K1 packed source records [npad][<=14]
  DBuf<double> k1_pseg, k1_psrc;  // symmetric K1 partial sums (allpairs.cu, deterministic reduction)
  K1Layout k1lay;
  DBuf<double> k2_pinc;  // [n_inc][3] K2 per-incidence sums (K2 order)
  DBuf<int> row_ptr, row_pos;  // [N+1], [n_inc]: K2 positions of each target row, (target, sphere) order
  DBuf<double> k3_part;  // K3 split-K partial tiles
  DBuf<unsigned> k3_cnt; // K3 per-tile arrival counters (self-resetting)
  DBuf<double> far;      // [N][3] all-pairs accumulator
  DBuf<double> nearout;  // [N][3]
  DBuf<double> rhs, sol, tmp, tmp2, tmp3;  // [N][3]
  DBuf<double> V;        // GMRES basis [(m+1)][3N]
  DBuf<double> red;      // reduction scratch
  DBuf<double> scal;     // device scalars
  DBuf<double> ft, uo;   // [np][6]
  DBuf<int> gm_ctl;      // GMRES device control words (gmres.cu)
  bool gm_ctl_init = false;
  DBuf<double> gm_z, gm_vin;  // Arnoldi step operator output / input
  // GMRES recycling store (gmres.cu): W orthonormal past rhs, Z = A_op^-1 W
  DBuf<double> rec_W, rec_Z;
  int rec_k = 0, rec_cap = 0;
  double* host_scal = nullptr;  // pinned

  Profile prof;
  CycleGraph gm_cycle;
  cudaStream_t side = nullptr;            // K2 overlapped with K1 (layer.cu)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool overlap_k2 = false;
  // target-side sharding over ranks (bpqn_geometry_shard, NEXT-4): this rank owns spheres
  // [sh_s0, sh_s1) = nodes [sh_t0, sh_t1) and near-target list entries [sh_k0, sh_k1);
  // after each operator application the owned rows go through sh_fn (an all-gather of
  // sh_rows * 3 doubles per rank from sh_send into sh_recv, user-owned device buffers).
  int shard_rank = 0, shard_world = 1;
  int sh_s0 = 0, sh_s1 = 0, sh_t0 = 0, sh_t1 = 0, sh_k0 = 0, sh_k1 = 0, sh_rows = 0;
  double *sh_send = nullptr, *sh_recv = nullptr;
  int (*sh_fn)(void* user) = nullptr;
  void* sh_user = nullptr;
  // optional symmetric K1 when sharded (bpqn_geometry_shard_symmetric): every rank runs an equal
  // share of the symmetric kernel's units over all targets; the partial sums go through
  // sh_rs_fn (a reduce-scatter of [world][sh_rows][3] from sh_rs_send into sh_rs_recv)
  double *sh_rs_send = nullptr, *sh_rs_recv = nullptr;
  int (*sh_rs_fn)(void* user) = nullptr;
  void* sh_rs_user = nullptr;
  std::vector<int> nt_list_h;  // host copy of the near-target list (shard ranges)
  // NCCL sharding (bpqn_geometry_shard_nccl, comm.cu): the library's own communicator and exchange
  // buffers; collectives are enqueued on the handle's stream (no host sync, no callback)
  void* nccl_comm = nullptr;
  bool sh_sym_nccl = false;  // symmetric K1 split with the NCCL reduce-scatter
  DBuf<double> sh_own_send, sh_own_recv, sh_own_rs_send, sh_own_rs_recv;
  // far-field FMM replacing K1 (fmm.cu; bpqn_disc_opts.fmm_order > 0)
  int fmm_order = 0, fmm_max_leaf = 0;
  // false: apply_operator uses the direct K1 even though the handle has an FMM (relaxed GMRES,
  // bpqn_gmres_opts.relax_fmm: direct in the early steps, the FMM once the residual allows it)
  bool fmm_on = true;
  int last_lo_mvps = -1;
  std::vector<long long> dvi_keys;  // DVI warm start: the last step's contact pairs (i Np + j, sorted) and lambda
  std::vector<double> dvi_lam;  // lo handle: lo MVPs of the last Bi-PQN solve it served (the lo_dense auto rule)
  struct Fmm* fmm = nullptr;
  bool sharded() const { return shard_world > 1 || nccl_comm != nullptr; }
  ~Geom();
};

// scope in which an FMM handle's applications use the direct K1 (when `on`); restores the flag
struct FmmDirect {
  Geom& g;
  bool prev;
  FmmDirect(Geom& g_, bool on) : g(g_), prev(g_.fmm_on) {
    if (on) g.fmm_on = false;
  }
  ~FmmDirect() { g.fmm_on = prev; }
};

// ---------------------------------------------------------------- kernels / passes
enum Mode { MODE_S = 0, MODE_D = 1, MODE_SD = 2 };

constexpr int K2_CHUNK = 64;  // incidence positions per K2 block
void precompute(Geom& g, cudaStream_t st, bool with_self);
void invert_in_place(double* A, int n, cudaStream_t st);  // Gauss-Jordan, partial pivoting  // self E matrices + near matrices

// out = Layer(sigmaS, sigmaD) with the given self matrix (E), mode selects the kernels.
// Es used for sigS, Ed for sigD (either may be null when the density is null).
void apply_operator(Geom& g, const double* sigS, const double* sigD, const double* Es, const double* Ed,
                    double* out, cudaStream_t st);

double allpairs_flops_per_pair(int mode);
void profile_collect(Geom& g);
void launch_allpairs(Geom& g, int mode, const double* sigS, const double* sigD, double* out, cudaStream_t st);
void k1_reserve(Geom& g);
// out rows [r0, r1) = (K1 partials of the last symmetric launch, or far) + (K2 partials if with_k2)
void launch_row_reduce(Geom& g, bool k1_partials, const double* far, bool with_k2, double* out, int r0, int r1,
                       cudaStream_t st);
void layer_reserve(Geom& g);  // K2 / K3 workspace (layer.cu)
bool k1_sharded_symmetric(const Geom& g);
void launch_near(Geom& g, const double* sigS, const double* sigD, cudaStream_t st);  // -> g.k2_pinc
// out (+)= E X per sphere (columns [s0, s1)), deterministic split-K
void launch_self_gemm(Geom& g, const double* E, const double* X, double* out, int accumulate, cudaStream_t st,
                      int s0 = 0, int s1 = -1);

// GMRES on A_op q = rhs (A_op = E_A + coarse + near); returns stats.
int gmres_solve(Geom& g, const double* rhs, double* x, const bpqn_gmres_opts& o, bpqn_gmres_stats& st,
                cudaStream_t s);
void gmres_reserve(Geom& g, int restart);   // basis and scratch for a restart length (init: default 100)
void gmres_recycle_reserve(Geom& g);        // recycling store (outside the hot calls; may stay off)

// Low-fidelity LCP matrix densified in HBM (dense_lo.cu, reading R38)
constexpr int GM_BATCH_MAX_M = 128;
struct DenseLoStats {
  int columns = 0, iters = 0, restart = 0;
  long long col_iters = 0;  // sum over columns of their iterations (the GEMM work with compaction)
  double ms_rhs = 0, ms_total = 0;
  size_t bytes = 0;
};
size_t dense_lo_bytes(const Geom& g, int restart);
void assemble_dense_operator(Geom& g, double* A_dev, cudaStream_t s);  // [3N][3N] row-major
// A^ = D^T M D of the handle's contact set (row-major Nc x Nc, host) by one batched GMRES over all
// Nc unit vectors with a dense operator; throws BPQN_ERR_OOM if it does not fit
int densify_lcp(Geom& g, const bpqn_gmres_opts& o, std::vector<double>& Ahat, DenseLoStats& st, cudaStream_t s);

// dense linear algebra on the device (dense_lo.cu): column-major cuBLAS DGEMM / DTRSM (lower
// triangular, non-unit; side 0 = left, 1 = right; trans 0 = N, 1 = T), blocked Cholesky (lower,
// strict upper triangle zeroed)
void blas_dgemm(cudaStream_t st, int ta, int tb, int m, int n, int k, double alpha, const double* A, int lda,
                const double* B, int ldb, double beta, double* C, int ldc);
void blas_dtrsm(cudaStream_t st, int side, int trans, int m, int n, const double* L, int ldl, double* B, int ldb);
void dev_potrf(cudaStream_t st, double* A, int n, int lda);
bool blas_dgemm_grouped(cudaStream_t st, int G, const int* m, const int* n, const int* k, const double* alpha,
                        const double* const* A_dev, const int* lda, const double* const* B_dev, const int* ldb,
                        double* const* C_dev, const int* ldc);

// FMM (fmm.cu): tree and lists from the host node positions; the K1 coarse sum into out [N][3]
void fmm_build(Geom& g, const std::vector<double>& X_host, cudaStream_t st);
void fmm_apply(Geom& g, const double* sigS, const double* sigD, double* out, cudaStream_t st);
void fmm_free(struct Fmm* f);

// NCCL (comm.cu)
void comm_unique_id(void* out128);
void comm_init(Geom& g, int rank, int world, const void* uid128);
void comm_destroy(Geom& g);
void comm_allgather(Geom& g, const double* send, double* recv, size_t count, cudaStream_t st);
void comm_reduce_scatter(Geom& g, const double* send, double* recv, size_t count, cudaStream_t st);

// small kernels (contacts.cu)
void launch_pt(Geom& g, const double* ft, double* f, cudaStream_t st);
void launch_rigid_readout(Geom& g, const double* q, double* uo, cudaStream_t st);  // uo = -(Ubar, Obar)
void launch_d_scatter(Geom& g, const double* lam, double* ft, cudaStream_t st);
void launch_dt_gather(Geom& g, const double* uo, double* w, double dt_scale, const double* add,
                      cudaStream_t st);
void launch_axpby(double* y, double a, const double* x, double b, size_t n, cudaStream_t st);
void launch_slip(Geom& g, const double* axes_dev, double B, double* slip, cudaStream_t st);
int detect_contacts(Geom& g, double thr, int max_contacts, int* pairs, double* normals, double* gaps,
                    cudaStream_t st);

}  // namespace bpqn

// the opaque C handle is a Geom
struct bpqn_geom : public bpqn::Geom {};
