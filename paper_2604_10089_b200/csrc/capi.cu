// C ABI of libbpqn (declarations and contracts in include/bpqn.h).
#include <algorithm>
#include <chrono>
#include <limits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bpqn_internal.h"
#include "pqn.h"

namespace bpqn {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

Geom::~Geom() {
  try {
    comm_destroy(*this);
  } catch (...) {
  }
  fmm_free(fmm);
  if (host_scal) cudaFreeHost(host_scal);
  for (auto& e : prof.pool)
    if (e) cudaEventDestroy(e);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (side) cudaStreamDestroy(side);
}

template <class F>
static int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return BPQN_ERR_INVALID;
  }
}

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static void upload(DBuf<double>& d, const std::vector<double>& h, cudaStream_t st) {
  d.alloc(h.size());
  if (!h.empty()) BPQN_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
}
static void upload_i(DBuf<int>& d, const std::vector<int>& h, cudaStream_t st) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) BPQN_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
}

static bpqn_gmres_opts gm_or_default(const bpqn_gmres_opts* gm) {
  bpqn_gmres_opts o;
  bpqn_default_gmres_opts(&o);
  if (gm) o = *gm;
  if (o.restart <= 0) o.restart = 100;
  if (o.max_iters <= 0) o.max_iters = 1000;
  if (!(o.tol > 0)) o.tol = 1e-12;
  return o;
}

// Owned spheres / nodes / near-target entries of this rank (bpqn_geometry_shard).
static void shard_ranges(Geom& g) {
  if (!g.sharded()) return;
  g.sh_s0 = (int)((long long)g.np * g.shard_rank / g.shard_world);
  g.sh_s1 = (int)((long long)g.np * (g.shard_rank + 1) / g.shard_world);
  g.sh_t0 = g.sh_s0 * g.nq;
  g.sh_t1 = g.sh_s1 * g.nq;
  g.sh_rows = (int)((g.np + g.shard_world - 1) / g.shard_world) * g.nq;
  g.sh_k0 = (int)(std::lower_bound(g.nt_list_h.begin(), g.nt_list_h.end(), g.sh_t0) - g.nt_list_h.begin());
  g.sh_k1 = (int)(std::lower_bound(g.nt_list_h.begin(), g.nt_list_h.end(), g.sh_t1) - g.nt_list_h.begin());
}

// Nodes, source records and near incidences for a set of centres (init and update):
// validates that no two spheres overlap; incidences (target i, sphere m) with
// |x_i - c_m| - a < d_near (R8), sorted by (i, m).
static void set_centers(Geom& G, const double* centers_host, cudaStream_t st) {
  Geom* g = &G;
  g->gm_cycle.clear();  // the captured GMRES cycle holds the old near data and grid sizes
  const double radius = g->a;
  const int n_spheres = g->np;
  g->centers.assign(centers_host, centers_host + 3 * (size_t)n_spheres);
  for (int i = 0; i < n_spheres; ++i)
    for (int j = i + 1; j < n_spheres; ++j) {
      double dx = g->centers[3 * j] - g->centers[3 * i], dy = g->centers[3 * j + 1] - g->centers[3 * i + 1],
             dz = g->centers[3 * j + 2] - g->centers[3 * i + 2];
      double d = std::sqrt(dx * dx + dy * dy + dz * dz);
      BPQN_REQUIRE(d - 2 * radius > 0, "spheres " + std::to_string(i) + " and " + std::to_string(j) + " overlap");
    }
  const int nq = g->nq, N = g->n;
  std::vector<double> X(3 * (size_t)N), src(8 * (size_t)N);
  for (int m = 0; m < g->np; ++m)
    for (int k = 0; k < nq; ++k) {
      size_t i = (size_t)m * nq + k;
      for (int c = 0; c < 3; ++c) {
        X[3 * i + c] = g->centers[3 * m + c] + radius * g->grid.xi[3 * k + c];
        src[8 * i + c] = X[3 * i + c];
        src[8 * i + 4 + c] = g->grid.xi[3 * k + c];
      }
      src[8 * i + 3] = g->grid.w[k];
      src[8 * i + 7] = 0.0;
    }
  upload(g->X, X, st);
  upload(g->src, src, st);
  upload(g->centers_d, g->centers, st);
  fmm_build(*g, X, st);  // far-field FMM tree and lists (only when fmm_order > 0)
  std::vector<std::pair<int, int>> inc;
  for (int n = 0; n < g->np; ++n)
    for (int m = 0; m < g->np; ++m) {
      if (m == n) continue;
      double dx = g->centers[3 * m] - g->centers[3 * n], dy = g->centers[3 * m + 1] - g->centers[3 * n + 1],
             dz = g->centers[3 * m + 2] - g->centers[3 * n + 2];
      if (std::sqrt(dx * dx + dy * dy + dz * dz) - 2 * radius >= g->d_near) continue;
      for (int k = 0; k < nq; ++k) {
        size_t i = (size_t)n * nq + k;
        double rx = X[3 * i] - g->centers[3 * m], ry = X[3 * i + 1] - g->centers[3 * m + 1],
               rz = X[3 * i + 2] - g->centers[3 * m + 2];
        if (std::sqrt(rx * rx + ry * ry + rz * rz) - radius < g->d_near) inc.emplace_back((int)i, m);
      }
    }
  std::sort(inc.begin(), inc.end());
  g->n_inc = (long long)inc.size();
  std::vector<int> it(inc.size()), im(inc.size()), ntl, ntp;
  for (size_t k = 0; k < inc.size(); ++k) {
    it[k] = inc[k].first;
    im[k] = inc[k].second;
    if (k == 0 || inc[k].first != inc[k - 1].first) {
      ntl.push_back(inc[k].first);
      ntp.push_back((int)k);
    }
  }
  ntp.push_back((int)inc.size());
  g->n_near_targets = (int)ntl.size();
  g->nt_list_h = ntl;
  shard_ranges(*g);
  upload_i(g->inc_t, it, st);
  upload_i(g->inc_m, im, st);
  upload_i(g->nt_list, ntl, st);
  upload_i(g->nt_ptr, ntp, st);
  // K2 order: by (source sphere, target), chunks of one sphere
  std::vector<std::pair<int, int>> bym(inc.size());
  for (size_t k = 0; k < inc.size(); ++k) bym[k] = {inc[k].second, inc[k].first};
  std::sort(bym.begin(), bym.end());
  std::vector<int> ct(inc.size()), cm(inc.size()), ch;
  for (size_t k = 0; k < bym.size(); ++k) {
    cm[k] = bym[k].first;
    ct[k] = bym[k].second;
    if (k == 0 || bym[k].first != bym[k - 1].first || (int)k - ch.back() == K2_CHUNK) {
      if (k) ch.push_back((int)k);
      ch.push_back((int)k);
    }
  }
  if (!bym.empty()) ch.push_back((int)bym.size());
  g->n_chunks = (int)ch.size() / 2;
  upload_i(g->cm_t, ct, st);
  upload_i(g->cm_m, cm, st);
  upload_i(g->chunks, ch, st);
  // per target row: its K2 positions in source-sphere order (k_row_reduce's fixed summation order)
  std::vector<int> rp((size_t)N + 1, 0), rpos(ct.size());
  for (int t : ct) rp[t + 1]++;
  for (int i = 0; i < N; ++i) rp[i + 1] += rp[i];
  {
    std::vector<int> fill(rp.begin(), rp.end() - 1);
    for (size_t k = 0; k < ct.size(); ++k) rpos[fill[ct[k]]++] = (int)k;
  }
  upload_i(g->row_ptr, rp, st);
  upload_i(g->row_pos, rpos, st);
  k1_reserve(*g);
  layer_reserve(*g);
  BPQN_CUDA(cudaStreamSynchronize(st));  // host staging vectors go out of scope
}

// (U, Omega) = M_slip(ft; slip) -> uo (device); returns GMRES status
static int mobility(Geom& g, const double* ft, const double* slip, double* uo, const bpqn_gmres_opts& o,
                    bpqn_gmres_stats& st, cudaStream_t s) {
  BPQN_REQUIRE(g.E_S.p, "geometry built without single-layer data (build_single_layer = 0)");
  launch_pt(g, ft, g.tmp.p, s);
  {
    FmmDirect direct(g, o.relax_fmm != 0);  // relaxed GMRES: the right-hand side with the direct K1
    apply_operator(g, g.tmp.p, nullptr, g.E_S.p, nullptr, g.rhs.p, s);
  }
  const size_t n3 = 3 * (size_t)g.n;
  if (slip) launch_axpby(g.rhs.p, 1.0, slip, -1.0, n3, s);
  else launch_axpby(g.rhs.p, 0.0, g.rhs.p, -1.0, n3, s);
  int rc = gmres_solve(g, g.rhs.p, g.sol.p, o, st, s);
  launch_rigid_readout(g, g.sol.p, uo, s);
  return rc;
}

static int lcp_mvp(Geom& g, const double* lam, double* w, const bpqn_gmres_opts& o, bpqn_gmres_stats& st,
                   cudaStream_t s) {
  BPQN_REQUIRE(g.nc > 0, "no contacts installed (call bpqn_contacts or bpqn_set_contacts)");
  launch_d_scatter(g, lam, g.ft.p, s);
  int rc = mobility(g, g.ft.p, nullptr, g.uo.p, o, st, s);
  launch_dt_gather(g, g.uo.p, w, 1.0, nullptr, s);
  return rc;
}

}  // namespace bpqn

using namespace bpqn;

extern "C" {

const char* bpqn_last_error(void) { return g_err.c_str(); }

void bpqn_default_disc_opts(bpqn_disc_opts* o) {
  if (!o) return;
  o->p_s = 0;
  o->d_near = 0.0;
  o->near_n1 = 0;
  o->near_n2 = 0;
  o->near_nphi = 0;
  o->build_single_layer = 1;
  o->fmm_order = 0;
}

void bpqn_default_gmres_opts(bpqn_gmres_opts* o) {
  if (!o) return;
  o->tol = 1e-12;
  o->restart = 100;
  o->max_iters = 1000;
  o->precond = 1;
  o->recycle = 0;
  o->relax_fmm = 0;
  o->relax_delta = 0.0;
}

void bpqn_default_solve_opts(bpqn_solve_opts* o) {
  if (!o) return;
  o->method = 0;
  o->k_max = 200;
  o->eps_kkt_abs = 1e-10;
  o->eps_kkt_rel = 0.0;
  o->tau = 1.0;
  o->refresh_period = 20;
  o->sub_eps_factor = 1e-2;
  o->sub_k_max = 50;
  o->prox_tol = 0.0;
  o->prox_jmax = 100;
  o->curv_skip = 1e-12;
  bpqn_default_gmres_opts(&o->gm_hi);
  bpqn_default_gmres_opts(&o->gm_lo);
  o->gm_hi.recycle = o->gm_lo.recycle = 1;
  o->cost_ratio = 0.0;
  o->sub_forcing = 0.0;
  o->verify_secants = 0;
  o->lo_dense = 0;
  o->warm_start = 1;
}

int bpqn_geometry_init(bpqn_geom_t* out, int n_spheres, const double* centers_host, double radius, double mu,
                       int p, const bpqn_disc_opts* opts, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(out && centers_host, "null pointer");
    BPQN_REQUIRE(n_spheres >= 1, "n_spheres must be >= 1");
    BPQN_REQUIRE(p >= 2, "p must be >= 2");
    BPQN_REQUIRE(p <= BPQN_P_MAX, "p must be <= 25 (precompute tile capacity)");
    BPQN_REQUIRE(radius > 0 && mu > 0, "radius and mu must be > 0");
    *out = nullptr;
    int dev = 0;
    BPQN_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    BPQN_CUDA(cudaGetDeviceProperties(&prop, dev));
    cudaStream_t st = S(stream);
    auto g = new bpqn_geom();
    try {
      g->sms = prop.multiProcessorCount;
      g->np = n_spheres;
      g->p = p;
      g->a = radius;
      g->mu = mu;
      bpqn_disc_opts o;
      bpqn_default_disc_opts(&o);
      if (opts) o = *opts;
      g->p_s = o.p_s > 0 ? o.p_s : 2 * p;
      g->d_near = o.d_near > 0 ? o.d_near : 4.0 * M_PI * radius / p;
      g->n1 = o.near_n1 > 0 ? o.near_n1 : 2 * p + 16;
      g->n2 = o.near_n2 > 0 ? o.near_n2 : p + 8;
      g->nphi = o.near_nphi > 0 ? o.near_nphi : 4 * p;
      // shared-memory tables of the rule precompute (geometry.cu k_quad_rows)
      BPQN_REQUIRE(g->p_s + 1 <= 128 && 2 * g->p_s <= 256 && g->n1 + g->n2 <= 128 && g->nphi <= 256,
                   "discretisation options exceed the precompute tables (p_s <= 63, n1 + n2 <= 128, nphi <= 256)");
      g->single_layer = o.build_single_layer != 0;
      g->fmm_order = o.fmm_order;
      BPQN_REQUIRE(o.fmm_order == 0 || (o.fmm_order >= 3 && o.fmm_order <= 12), "fmm_order must be 0 or in [3, 12]");
      const char* ov = getenv("BPQN_OVERLAP_K2");
      g->overlap_k2 = ov && ov[0] == '1';
      build_grid(p, radius, g->grid);
      g->nq = g->grid.nq;
      g->n = g->np * g->nq;
      g->nb = sh_count(p);
      upload(g->xi_d, g->grid.xi, st);
      upload(g->w_d, g->grid.w, st);
      set_centers(*g, centers_host, st);
      size_t n3 = 3 * (size_t)g->n;
      g->far.alloc(n3);
      g->nearout.alloc(n3);
      g->rhs.alloc(n3);
      g->sol.alloc(n3);
      g->tmp.alloc(n3);
      g->tmp2.alloc(n3);
      g->ft.alloc(6 * (size_t)g->np);
      g->uo.alloc(6 * (size_t)g->np);
      gmres_reserve(*g, 100);
      BPQN_CUDA(cudaMallocHost(&g->host_scal, 64 * sizeof(double)));
      precompute(*g, st, true);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
    return BPQN_OK;
  });
}

int bpqn_geometry_destroy(bpqn_geom_t g) {
  return guarded([&]() -> int {
    delete g;
    return BPQN_OK;
  });
}

int bpqn_geometry_update(bpqn_geom_t g, const double* centers_host, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && centers_host, "null pointer");
    cudaStream_t st = S(stream);
    set_centers(*g, centers_host, st);
    precompute(*g, st, false);  // near rows only; grid, SH analysis, self operators and inverse kept
    g->nc = 0;
    g->rec_k = 0;
    return BPQN_OK;
  });
}

int bpqn_geometry_shard(bpqn_geom_t g, int rank, int world, double* send_dev, double* recv_dev,
                        int (*allgather)(void* user), void* user) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    BPQN_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
    // any (re)sharding drops a previous symmetric-K1 registration: its buffers were sized for
    // the old world (bpqn_geometry_shard_symmetric must be called again)
    g->sh_rs_fn = nullptr;
    g->sh_rs_send = g->sh_rs_recv = nullptr;
    g->sh_rs_user = nullptr;
    comm_destroy(*g);  // callback sharding replaces an NCCL sharding
    g->sh_sym_nccl = false;
    g->gm_cycle.clear();
    if (world == 1) {
      g->shard_world = 1;
      g->shard_rank = 0;
      return BPQN_OK;
    }
    BPQN_REQUIRE(world <= g->np, "more ranks than spheres");
    BPQN_REQUIRE(send_dev && recv_dev && allgather, "null buffer or callback");
    g->gm_cycle.clear();
    g->shard_rank = rank;
    g->shard_world = world;
    g->sh_send = send_dev;
    g->sh_recv = recv_dev;
    g->sh_fn = allgather;
    g->sh_user = user;
    shard_ranges(*g);
    return BPQN_OK;
  });
}

int bpqn_nccl_unique_id(void* uid128) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(uid128, "null pointer");
    comm_unique_id(uid128);
    return BPQN_OK;
  });
}

int bpqn_geometry_shard_nccl(bpqn_geom_t g, int rank, int world, const void* uid128, int symmetric) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && uid128, "null pointer");
    BPQN_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
    BPQN_REQUIRE(world <= g->np, "more ranks than spheres");
    g->sh_fn = nullptr;
    g->sh_send = g->sh_recv = nullptr;
    g->sh_user = nullptr;
    g->sh_rs_fn = nullptr;
    g->sh_rs_send = g->sh_rs_recv = nullptr;
    g->sh_rs_user = nullptr;
    g->gm_cycle.clear();
    g->shard_world = 1;
    g->shard_rank = 0;
    comm_init(*g, rank, world, uid128);  // collective over the world ranks
    g->shard_rank = rank;
    g->shard_world = world;
    g->sh_sym_nccl = symmetric != 0 && g->nq >= 32 && g->np <= 4096;
    shard_ranges(*g);
    return BPQN_OK;
  });
}

int bpqn_geometry_shard_symmetric(bpqn_geom_t g, double* rs_send_dev, double* rs_recv_dev,
                                  int (*reduce_scatter)(void* user), void* user) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    g->gm_cycle.clear();
    if (!reduce_scatter) {  // back to the one-directional K1 over the owned target rows
      g->sh_rs_fn = nullptr;
      g->sh_rs_send = g->sh_rs_recv = nullptr;
      g->sh_rs_user = nullptr;
      return BPQN_OK;
    }
    BPQN_REQUIRE(g->shard_world > 1, "handle is not sharded (call bpqn_geometry_shard first)");
    BPQN_REQUIRE(rs_send_dev && rs_recv_dev, "null buffer");
    BPQN_REQUIRE(g->nq >= 32 && g->np <= 4096, "symmetric K1 needs Nq >= 32 (p >= 4) and Np <= 4096");
    g->sh_rs_send = rs_send_dev;
    g->sh_rs_recv = rs_recv_dev;
    g->sh_rs_fn = reduce_scatter;
    g->sh_rs_user = user;
    return BPQN_OK;
  });
}

int bpqn_geometry_info(bpqn_geom_t g, int* n_nodes, int* nq, long long* n_incidences, long long* device_bytes) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    if (n_nodes) *n_nodes = g->n;
    if (nq) *nq = g->nq;
    if (n_incidences) *n_incidences = g->n_inc;
    if (device_bytes) {
      long long b = 0;
      b += g->X.bytes() + g->src.bytes() + g->analysis.bytes() + g->E_S.bytes() + g->E_L.bytes() + g->E_A.bytes();
      b += g->T_S.bytes() + g->T_D.bytes() + g->V.bytes() + g->far.bytes() * 6;
      *device_bytes = b;
    }
    return BPQN_OK;
  });
}

int bpqn_contacts(bpqn_geom_t g, double thr, int max_contacts, int* n_contacts_host, int* pairs_dev,
                  double* normals_dev, double* gaps_dev, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && n_contacts_host, "null pointer");
    BPQN_REQUIRE(max_contacts >= 0, "max_contacts < 0");
    cudaStream_t st = S(stream);
    int cap = (int)std::min<long long>((long long)g->np * (g->np - 1) / 2, 1 << 26);
    g->pairs.ensure(2 * (size_t)std::max(cap, 1));
    g->normals.ensure(3 * (size_t)std::max(cap, 1));
    g->gaps.ensure((size_t)std::max(cap, 1));
    int nc = detect_contacts(*g, thr, cap, g->pairs.p, g->normals.p, g->gaps.p, st);
    g->nc = nc;
    *n_contacts_host = nc;
    int ncopy = std::min(nc, max_contacts);
    if (ncopy > 0) {
      BPQN_REQUIRE(pairs_dev && normals_dev && gaps_dev, "null output pointer");
      BPQN_CUDA(cudaMemcpyAsync(pairs_dev, g->pairs.p, 2 * sizeof(int) * ncopy, cudaMemcpyDeviceToDevice, st));
      BPQN_CUDA(cudaMemcpyAsync(normals_dev, g->normals.p, 3 * sizeof(double) * ncopy, cudaMemcpyDeviceToDevice, st));
      BPQN_CUDA(cudaMemcpyAsync(gaps_dev, g->gaps.p, sizeof(double) * ncopy, cudaMemcpyDeviceToDevice, st));
    }
    BPQN_CUDA(cudaStreamSynchronize(st));
    if (nc > max_contacts) {
      set_error("more contacts than max_contacts");
      return BPQN_ERR_CAPACITY;
    }
    return BPQN_OK;
  });
}

int bpqn_set_contacts(bpqn_geom_t g, int n_contacts, const int* pairs_dev, const double* normals_dev,
                      const double* gaps_dev, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    BPQN_REQUIRE(n_contacts >= 0, "n_contacts < 0");
    cudaStream_t st = S(stream);
    g->pairs.ensure(2 * (size_t)std::max(n_contacts, 1));
    g->normals.ensure(3 * (size_t)std::max(n_contacts, 1));
    g->gaps.ensure((size_t)std::max(n_contacts, 1));
    if (n_contacts > 0) {
      BPQN_REQUIRE(pairs_dev && normals_dev && gaps_dev, "null pointer");
      BPQN_CUDA(cudaMemcpyAsync(g->pairs.p, pairs_dev, 2 * sizeof(int) * n_contacts, cudaMemcpyDeviceToDevice, st));
      BPQN_CUDA(cudaMemcpyAsync(g->normals.p, normals_dev, 3 * sizeof(double) * n_contacts, cudaMemcpyDeviceToDevice, st));
      BPQN_CUDA(cudaMemcpyAsync(g->gaps.p, gaps_dev, sizeof(double) * n_contacts, cudaMemcpyDeviceToDevice, st));
    }
    g->nc = n_contacts;
    return BPQN_OK;
  });
}

int bpqn_layer_apply(bpqn_geom_t g, const double* f_dev, const double* q_dev, double* u_dev, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && u_dev, "null pointer");
    cudaStream_t st = S(stream);
    if (!f_dev && !q_dev) {
      BPQN_CUDA(cudaMemsetAsync(u_dev, 0, 3 * sizeof(double) * (size_t)g->n, st));
      return BPQN_OK;
    }
    BPQN_REQUIRE(!f_dev || g->E_S.p, "geometry built without single-layer data");
    apply_operator(*g, f_dev, q_dev, g->E_S.p, g->E_L.p, u_dev, st);
    return BPQN_OK;
  });
}

int bpqn_janus_slip(bpqn_geom_t g, const double* axes_host, double B, double* slip_dev, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && axes_host && slip_dev, "null pointer");
    cudaStream_t st = S(stream);
    DBuf<double> ax;
    ax.alloc(3 * (size_t)g->np);
    BPQN_CUDA(cudaMemcpyAsync(ax.p, axes_host, 3 * sizeof(double) * g->np, cudaMemcpyHostToDevice, st));
    launch_slip(*g, ax.p, B, slip_dev, st);
    BPQN_CUDA(cudaStreamSynchronize(st));
    return BPQN_OK;
  });
}

int bpqn_mobility_apply(bpqn_geom_t g, const double* ft_dev, const double* slip_dev, double* uo_dev,
                        const bpqn_gmres_opts* gm, bpqn_gmres_stats* st, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && ft_dev && uo_dev, "null pointer");
    bpqn_gmres_stats tmp{};
    int rc = mobility(*g, ft_dev, slip_dev, uo_dev, gm_or_default(gm), tmp, S(stream));
    BPQN_CUDA(cudaStreamSynchronize(S(stream)));
    if (st) *st = tmp;
    if (rc) set_error("GMRES did not converge / NaN");
    return rc;
  });
}

int bpqn_lcp_mvp(bpqn_geom_t g, const double* lambda_dev, double* w_dev, const bpqn_gmres_opts* gm,
                 bpqn_gmres_stats* st, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && lambda_dev && w_dev, "null pointer");
    bpqn_gmres_stats tmp{};
    int rc = lcp_mvp(*g, lambda_dev, w_dev, gm_or_default(gm), tmp, S(stream));
    BPQN_CUDA(cudaStreamSynchronize(S(stream)));
    if (st) *st = tmp;
    if (rc) set_error("GMRES did not converge / NaN");
    return rc;
  });
}

int bpqn_lcp_b(bpqn_geom_t g, const double* fnc_dev, const double* slip_dev, double dt, double* b_dev,
               const bpqn_gmres_opts* gm, bpqn_gmres_stats* st, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && fnc_dev && b_dev, "null pointer");
    BPQN_REQUIRE(dt > 0, "dt must be > 0");
    BPQN_REQUIRE(g->nc > 0, "no contacts installed");
    cudaStream_t s = S(stream);
    BPQN_CUDA(cudaMemsetAsync(g->ft.p, 0, 6 * sizeof(double) * g->np, s));
    BPQN_CUDA(cudaMemcpy2DAsync(g->ft.p, 6 * sizeof(double), fnc_dev, 3 * sizeof(double), 3 * sizeof(double),
                                g->np, cudaMemcpyDeviceToDevice, s));
    bpqn_gmres_stats tmp{};
    int rc = mobility(*g, g->ft.p, slip_dev, g->uo.p, gm_or_default(gm), tmp, s);
    launch_dt_gather(*g, g->uo.p, b_dev, 1.0, nullptr, s);
    launch_axpby(b_dev, 1.0 / dt, g->gaps.p, 1.0, g->nc, s);
    BPQN_CUDA(cudaStreamSynchronize(s));
    if (st) *st = tmp;
    if (rc) set_error("GMRES did not converge / NaN");
    return rc;
  });
}

static PqnOpts to_pqn(const bpqn_solve_opts& o) {
  PqnOpts q;
  q.k_max = o.k_max;
  q.eps_abs = o.eps_kkt_abs;
  q.eps_rel = o.eps_kkt_rel;
  q.tau = o.tau;
  q.refresh = o.refresh_period;
  q.sub_eps_factor = o.sub_eps_factor;
  q.sub_k_max = o.sub_k_max;
  q.prox_tol = o.prox_tol;
  q.prox_jmax = o.prox_jmax;
  q.curv = o.curv_skip;
  q.sub_forcing = o.sub_forcing;
  q.verify_secants = o.verify_secants != 0;
  return q;
}

int bpqn_solve_lcp(bpqn_geom_t hi, bpqn_geom_t lo, const double* b_dev, double* lambda_dev,
                   const bpqn_solve_opts* opts, bpqn_report* rep, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(hi && b_dev && lambda_dev, "null pointer");
    bpqn_solve_opts o;
    bpqn_default_solve_opts(&o);
    if (opts) o = *opts;
    const bool bi = lo && o.method == 1;
    if (bi) BPQN_REQUIRE(lo->nc == hi->nc, "Bi-PQN needs the same contact set on both fidelities");
    cudaStream_t s = S(stream);
    const int nc = hi->nc;
    BPQN_REQUIRE(nc > 0, "no contacts installed");
    std::vector<double> b(nc), x0(nc);
    BPQN_CUDA(cudaMemcpyAsync(b.data(), b_dev, 8 * nc, cudaMemcpyDeviceToHost, s));
    BPQN_CUDA(cudaMemcpyAsync(x0.data(), lambda_dev, 8 * nc, cudaMemcpyDeviceToHost, s));
    BPQN_CUDA(cudaStreamSynchronize(s));
    for (double v : x0) BPQN_REQUIRE(v >= 0, "x_init must be >= 0");
    if (o.gm_hi.recycle) {  // reserved here, outside the MVPs (no allocation in the hot calls)
      gmres_recycle_reserve(*hi);
      hi->rec_k = 0;
    }
    if (bi && o.gm_lo.recycle) {
      gmres_recycle_reserve(*lo);
      lo->rec_k = 0;
    }
    DBuf<double> dv, dw;
    dv.alloc(nc);
    dw.alloc(nc);
    bpqn_gmres_opts ghi = gm_or_default(&o.gm_hi), glo = gm_or_default(&o.gm_lo);
    double ms_hi = 0, ms_lo = 0;
    int it_hi = 0, it_lo = 0, n_hi = 0, n_lo = 0;
    int gm_fail = 0;
    auto make = [&](Geom* g, const bpqn_gmres_opts& gm, double& ms, int& its, int& cnt) -> MvpFn {
      return [&, g, gm](const std::vector<double>& v, std::vector<double>& out, std::vector<double>* aux) {
        BPQN_CUDA(cudaMemcpyAsync(dv.p, v.data(), 8 * nc, cudaMemcpyHostToDevice, s));
        bpqn_gmres_stats st{};
        auto t0 = std::chrono::steady_clock::now();
        int rc = lcp_mvp(*g, dv.p, dw.p, gm, st, s);
        out.resize(nc);
        BPQN_CUDA(cudaMemcpyAsync(out.data(), dw.p, 8 * nc, cudaMemcpyDeviceToHost, s));
        BPQN_CUDA(cudaStreamSynchronize(s));
        auto t1 = std::chrono::steady_clock::now();
        ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
        its += st.iters;
        cnt++;
        if (rc) gm_fail = rc;
        static const bool log_mvp = getenv("BPQN_LOG_MVP") != nullptr;
        if (log_mvp)
          fprintf(stderr, "mvp %s #%d: rc %d its %d resid %.2e applies %d ms %.1f\n", g == hi ? "hi" : "lo", cnt, rc,
                  st.iters, st.rel_resid, st.applies, st.ms);
        (void)aux;
      };
    };
    MvpFn fhi = make(hi, ghi, ms_hi, it_hi, n_hi);
    auto t0 = std::chrono::steady_clock::now();
    PqnOpts q = to_pqn(o);
    std::vector<double> x;
    int iters = 0, term = 2, hi_mvps = 0, lo_mvps = 0;
    double kkt = 0, kkt_rel = 0, secant_res = 0;
    int lo_init = 0;
    DenseLoStats dls;
    std::vector<double> Ahat;
    bool dense_lo = false;
    // lo_dense = 2 (auto): form A^ when the LCP looks hard -- at least a quarter of the contacts start
    // approaching (b_l < 0), where Bi-PQN needs hundreds of lo MVPs (c4: 41 % negative, 386 lo MVPs);
    // warm online steps with a few approaching contacts need tens and stay matrix-free
    // In a time-stepping loop the same handles solve one LCP per step: the auto mode also forms A^ when the
    // previous Bi-PQN solve on this lo handle needed >= Nc / 4 lo MVPs (forming costs about that many
    // matrix-free lo MVPs: c4 lo 9.9 s ~ 116 x 85 ms; p_lo = 4 1.2 s ~ 170 x 7 ms).
    int n_neg = 0;
    for (double v : b) n_neg += v < 0.0;
    const bool busy_before = bi && lo->last_lo_mvps >= 0 && 4 * lo->last_lo_mvps >= nc;
    const bool want_dense = o.lo_dense == 1 || (o.lo_dense == 2 && (4 * n_neg >= nc || busy_before));
    if (bi && want_dense) {
      try {
        densify_lcp(*lo, glo, Ahat, dls, s);
        dense_lo = true;
        ms_lo += dls.ms_total;
      } catch (const Error& e) {
        if (e.code != BPQN_ERR_OOM) throw;
        cudaGetLastError();  // does not fit: matrix-free low fidelity
      }
    }
    if (bi) {
      MvpFn flo = make(lo, glo, ms_lo, it_lo, n_lo);
      if (dense_lo)  // every low-fidelity MVP is the Nc x Nc product with the formed A^
        flo = [&](const std::vector<double>& v, std::vector<double>& out, std::vector<double>*) {
          auto ta = std::chrono::steady_clock::now();
          out.assign(nc, 0.0);
          for (int i = 0; i < nc; ++i) {
            double acc = 0.0;
            const double* row = Ahat.data() + (size_t)i * nc;
            for (int j = 0; j < nc; ++j) acc += row[j] * v[j];
            out[i] = acc;
          }
          n_lo++;
          ms_lo += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count();
        };
      BiResult r = bi_pqn(fhi, flo, b, x0, q);
      prox_profile_flush();
      x = r.x;
      iters = r.iterations;
      term = r.termination;
      hi_mvps = r.hi_mvps;
      lo_mvps = r.lo_mvps;
      lo->last_lo_mvps = r.lo_mvps;
      kkt = r.kkt;
      kkt_rel = r.kkt_rel;
      secant_res = r.secant_residual;
      lo_init = r.init_lo_mvps;
    } else {
      MonoResult r = o.method == 2 ? bb_pgd(fhi, b, x0, q) : mono_pqn(fhi, b, x0, q, nullptr, nullptr, nullptr);
      prox_profile_flush();
      x = r.x;
      iters = r.iterations;
      term = r.termination;
      hi_mvps = r.mvps;
      kkt = r.kkt;
      kkt_rel = r.kkt_rel;
    }
    auto t1 = std::chrono::steady_clock::now();
    BPQN_CUDA(cudaMemcpyAsync(lambda_dev, x.data(), 8 * nc, cudaMemcpyHostToDevice, s));
    BPQN_CUDA(cudaStreamSynchronize(s));
    if (rep) {
      rep->iterations = iters;
      rep->hi_mvps = hi_mvps;
      rep->lo_mvps = lo_mvps;
      rep->gmres_iters_hi = it_hi;
      rep->gmres_iters_lo = it_lo;
      double t_hi = n_hi ? ms_hi / n_hi : 0, t_lo = n_lo ? ms_lo / n_lo : 0;
      double ratio = o.cost_ratio > 0 ? o.cost_ratio : (t_hi > 0 ? t_lo / t_hi : 0);
      rep->cost_ratio = ratio;
      rep->e_mvps = hi_mvps + lo_mvps * ratio;
      rep->kkt_abs = kkt;
      rep->kkt_rel = kkt_rel;
      rep->objective = 0;
      rep->ms_total = std::chrono::duration<double, std::milli>(t1 - t0).count();
      rep->ms_hi = ms_hi;
      rep->ms_lo = ms_lo;
      rep->termination = term;
      rep->secant_residual = secant_res;
      rep->lo_mvps_init = lo_init;
      rep->lo_dense_columns = dense_lo ? dls.columns : 0;
      rep->lo_dense_gmres_iters = dense_lo ? dls.iters : 0;
      rep->ms_lo_dense = dense_lo ? dls.ms_total : 0.0;
      if (dense_lo) {  // E-MVPs from measured time: the forming of A^ dominates the low-fidelity cost
        const double t_hi = n_hi ? ms_hi / n_hi : 0;
        rep->cost_ratio = o.cost_ratio > 0 ? o.cost_ratio : (t_hi > 0 && n_lo ? (ms_lo / n_lo) / t_hi : 0);
        rep->e_mvps = hi_mvps + (t_hi > 0 ? ms_lo / t_hi : 0);
      }
    }
    if (gm_fail) {
      set_error("an inner GMRES solve did not converge");
      return gm_fail;
    }
    if (term == 3) {
      set_error("PQN stalled");
      return BPQN_ERR_STALLED;
    }
    if (term == 2) {
      set_error("PQN reached k_max");
      return BPQN_ERR_NOCONV;
    }
    return BPQN_OK;
  });
}

static double min_gap(const std::vector<double>& c, int np, double a) {
  double m = std::numeric_limits<double>::infinity();
  for (int i = 0; i < np; ++i)
    for (int j = i + 1; j < np; ++j) {
      const double dx = c[3 * j] - c[3 * i], dy = c[3 * j + 1] - c[3 * i + 1], dz = c[3 * j + 2] - c[3 * i + 2];
      m = std::min(m, std::sqrt(dx * dx + dy * dy + dz * dz) - 2 * a);
    }
  return m;
}

int bpqn_dvi_step(bpqn_geom_t hi, bpqn_geom_t lo, double* centers_host, double* axes_host, const double* fnc_host,
                  double slip_B, double dt, double delta, const bpqn_solve_opts* opts, double* uo_host,
                  bpqn_step_report* rep, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(hi && centers_host && axes_host && fnc_host, "null pointer");
    BPQN_REQUIRE(dt > 0, "dt must be > 0");
    BPQN_REQUIRE(!lo || (lo->np == hi->np && lo->a == hi->a), "lo must cover the same spheres");
    auto t0 = std::chrono::steady_clock::now();
    cudaStream_t s = S(stream);
    Geom& g = *hi;
    const int np = g.np;
    bpqn_step_report R{};
    R.min_gap_before = min_gap(g.centers, np, g.a);
    bpqn_solve_opts o;
    bpqn_default_solve_opts(&o);
    if (opts) o = *opts;
    // contacts at the current configuration (K5), shared with the low fidelity
    const int cap = std::max(1, np * (np - 1) / 2);
    g.pairs.ensure(2 * (size_t)cap);
    g.normals.ensure(3 * (size_t)cap);
    g.gaps.ensure((size_t)cap);
    g.nc = detect_contacts(g, delta, cap, g.pairs.p, g.normals.p, g.gaps.p, s);
    const int nc = g.nc;
    R.n_contacts = nc;
    if (lo) {
      lo->pairs.ensure(2 * (size_t)cap);
      lo->normals.ensure(3 * (size_t)cap);
      lo->gaps.ensure((size_t)cap);
      if (nc > 0) {
        BPQN_CUDA(cudaMemcpyAsync(lo->pairs.p, g.pairs.p, 2 * sizeof(int) * nc, cudaMemcpyDeviceToDevice, s));
        BPQN_CUDA(cudaMemcpyAsync(lo->normals.p, g.normals.p, 3 * sizeof(double) * nc, cudaMemcpyDeviceToDevice, s));
        BPQN_CUDA(cudaMemcpyAsync(lo->gaps.p, g.gaps.p, sizeof(double) * nc, cudaMemcpyDeviceToDevice, s));
      }
      lo->nc = nc;
    }
    // non-collisional mobility with the Janus slip of the current axes
    DBuf<double> ax, slip, ft, uo_nc, uo_c, bvec, lam;
    ax.alloc(3 * (size_t)np);
    slip.alloc(3 * (size_t)g.n);
    ft.alloc(6 * (size_t)np);
    uo_nc.alloc(6 * (size_t)np);
    uo_c.alloc(6 * (size_t)np);
    BPQN_CUDA(cudaMemcpyAsync(ax.p, axes_host, 3 * sizeof(double) * np, cudaMemcpyHostToDevice, s));
    launch_slip(g, ax.p, slip_B, slip.p, s);
    std::vector<double> fth(6 * (size_t)np, 0.0);
    for (int m = 0; m < np; ++m)
      for (int c = 0; c < 3; ++c) fth[6 * m + c] = fnc_host[3 * m + c];
    BPQN_CUDA(cudaMemcpyAsync(ft.p, fth.data(), 6 * sizeof(double) * np, cudaMemcpyHostToDevice, s));
    bpqn_gmres_opts gm = gm_or_default(&o.gm_hi);
    int rc = mobility(g, ft.p, slip.p, uo_nc.p, gm, R.gm_nc, s);
    if (rc) return rc;
    std::vector<double> U(6 * (size_t)np);
    BPQN_CUDA(cudaMemcpyAsync(U.data(), uo_nc.p, 6 * sizeof(double) * np, cudaMemcpyDeviceToHost, s));
    BPQN_CUDA(cudaStreamSynchronize(s));
    if (nc > 0) {
      // b = Phi/dt + D^T U_nc ; LCP ; U_c = M D lambda
      bvec.alloc(nc);
      lam.alloc(nc);
      launch_dt_gather(g, uo_nc.p, bvec.p, 1.0, nullptr, s);
      launch_axpby(bvec.p, 1.0 / dt, g.gaps.p, 1.0, nc, s);
      // x^(-1): the previous step's lambda of the same sphere pairs (warm start), 0 for new pairs
      std::vector<int> ph(2 * (size_t)nc);
      BPQN_CUDA(cudaMemcpyAsync(ph.data(), g.pairs.p, 2 * sizeof(int) * nc, cudaMemcpyDeviceToHost, s));
      BPQN_CUDA(cudaStreamSynchronize(s));
      std::vector<long long> keys(nc);
      for (int l = 0; l < nc; ++l) keys[l] = (long long)ph[2 * l] * np + ph[2 * l + 1];
      std::vector<double> x0(nc, 0.0);
      if (o.warm_start && !g.dvi_keys.empty())
        for (int l = 0; l < nc; ++l) {
          auto it = std::lower_bound(g.dvi_keys.begin(), g.dvi_keys.end(), keys[l]);
          if (it != g.dvi_keys.end() && *it == keys[l]) x0[l] = g.dvi_lam[it - g.dvi_keys.begin()];
        }
      BPQN_CUDA(cudaMemcpyAsync(lam.p, x0.data(), sizeof(double) * nc, cudaMemcpyHostToDevice, s));
      R.solve_rc = bpqn_solve_lcp(hi, lo, bvec.p, lam.p, &o, &R.lcp, stream);
      if (R.solve_rc != BPQN_OK && R.solve_rc != BPQN_ERR_NOCONV && R.solve_rc != BPQN_ERR_STALLED)
        return R.solve_rc;
      launch_d_scatter(g, lam.p, ft.p, s);
      rc = mobility(g, ft.p, nullptr, uo_c.p, gm, R.gm_c, s);
      if (rc) return rc;
      std::vector<double> Uc(6 * (size_t)np), lh(nc);
      BPQN_CUDA(cudaMemcpyAsync(Uc.data(), uo_c.p, 6 * sizeof(double) * np, cudaMemcpyDeviceToHost, s));
      BPQN_CUDA(cudaMemcpyAsync(lh.data(), lam.p, sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
      BPQN_CUDA(cudaStreamSynchronize(s));
      for (size_t i = 0; i < U.size(); ++i) U[i] += Uc[i];
      for (double v : lh) R.active_contacts += v > 0.0;
      // keep (pair, lambda) sorted by pair for the next step's warm start (contact lists are lexicographic)
      std::vector<int> ord(nc);
      for (int l = 0; l < nc; ++l) ord[l] = l;
      std::sort(ord.begin(), ord.end(), [&](int a2, int b2) { return keys[a2] < keys[b2]; });
      g.dvi_keys.resize(nc);
      g.dvi_lam.resize(nc);
      for (int l = 0; l < nc; ++l) {
        g.dvi_keys[l] = keys[ord[l]];
        g.dvi_lam[l] = lh[ord[l]];
      }
    } else {
      g.dvi_keys.clear();
      g.dvi_lam.clear();
    }
    // forward Euler on centres and Janus axes
    std::vector<double> cn(3 * (size_t)np), an(3 * (size_t)np);
    for (int m = 0; m < np; ++m) {
      const double* u = &U[6 * m];
      const double* a = &axes_host[3 * m];
      double w[3] = {u[4] * a[2] - u[5] * a[1], u[5] * a[0] - u[3] * a[2], u[3] * a[1] - u[4] * a[0]};
      double nrm = 0;
      for (int c = 0; c < 3; ++c) {
        cn[3 * m + c] = centers_host[3 * m + c] + dt * u[c];
        an[3 * m + c] = a[c] + dt * w[c];
        nrm += an[3 * m + c] * an[3 * m + c];
      }
      nrm = std::sqrt(nrm);
      for (int c = 0; c < 3; ++c) an[3 * m + c] /= nrm;
    }
    R.min_gap_after = min_gap(cn, np, g.a);
    if (!(R.min_gap_after > 0)) {
      if (rep) *rep = R;
      throw Error{BPQN_ERR_INVALID, "the step makes spheres overlap (min gap " + std::to_string(R.min_gap_after) +
                                        "); reduce dt"};
    }
    set_centers(g, cn.data(), s);
    precompute(g, s, false);
    g.nc = 0;
    g.rec_k = 0;
    if (lo) {
      set_centers(*lo, cn.data(), s);
      precompute(*lo, s, false);
      lo->nc = 0;
      lo->rec_k = 0;
    }
    std::copy(cn.begin(), cn.end(), centers_host);
    std::copy(an.begin(), an.end(), axes_host);
    if (uo_host) std::copy(U.begin(), U.end(), uo_host);
    R.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (rep) *rep = R;
    return R.solve_rc;
  });
}

int bpqn_solve_lcp_dense(const double* A, const double* Ahat, int n, const double* b_host, double* x_host,
                         const bpqn_solve_opts* opts, bpqn_report* rep) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(A && b_host && x_host && n > 0, "null pointer / bad size");
    bpqn_solve_opts o;
    bpqn_default_solve_opts(&o);
    if (opts) o = *opts;
    auto dense = [n](const double* M) -> MvpFn {
      return [M, n](const std::vector<double>& v, std::vector<double>& out, std::vector<double>*) {
        out.assign(n, 0.0);
        for (int i = 0; i < n; ++i) {
          double s = 0;
          for (int j = 0; j < n; ++j) s += M[(size_t)i * n + j] * v[j];
          out[i] = s;
        }
      };
    };
    std::vector<double> b(b_host, b_host + n), x0(x_host, x_host + n);
    PqnOpts q = to_pqn(o);
    int term;
    if (Ahat && o.method == 1) {
      BiResult r = bi_pqn(dense(A), dense(Ahat), b, x0, q);
      std::copy(r.x.begin(), r.x.end(), x_host);
      term = r.termination;
      if (rep) {
        *rep = bpqn_report{};
        rep->iterations = r.iterations;
        rep->hi_mvps = r.hi_mvps;
        rep->lo_mvps = r.lo_mvps;
        rep->kkt_abs = r.kkt;
        rep->termination = term;
        rep->secant_residual = r.secant_residual;
        rep->lo_mvps_init = r.init_lo_mvps;
      }
    } else {
      MonoResult r = o.method == 2 ? bb_pgd(dense(A), b, x0, q) : mono_pqn(dense(A), b, x0, q, nullptr, nullptr, nullptr);
      std::copy(r.x.begin(), r.x.end(), x_host);
      term = r.termination;
      if (rep) {
        *rep = bpqn_report{};
        rep->iterations = r.iterations;
        rep->hi_mvps = r.mvps;
        rep->kkt_abs = r.kkt;
        rep->termination = term;
      }
    }
    if (term == 3) return BPQN_ERR_STALLED;
    if (term == 2) return BPQN_ERR_NOCONV;
    return BPQN_OK;
  });
}

int bpqn_solve_lcp_dense_dev(const double* A_dev, const double* Ahat_dev, int n, const double* b_dev, double* x_dev,
                             const bpqn_solve_opts* opts, bpqn_report* rep, void* stream) {
  try {
    BPQN_REQUIRE(A_dev && b_dev && x_dev && n > 0, "null pointer / bad size");
    cudaStream_t st = S(stream);
    std::vector<double> A((size_t)n * n), Ah, b(n), x(n);
    BPQN_CUDA(cudaMemcpyAsync(A.data(), A_dev, 8 * A.size(), cudaMemcpyDeviceToHost, st));
    if (Ahat_dev) {
      Ah.resize((size_t)n * n);
      BPQN_CUDA(cudaMemcpyAsync(Ah.data(), Ahat_dev, 8 * Ah.size(), cudaMemcpyDeviceToHost, st));
    }
    BPQN_CUDA(cudaMemcpyAsync(b.data(), b_dev, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
    BPQN_CUDA(cudaMemcpyAsync(x.data(), x_dev, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
    BPQN_CUDA(cudaStreamSynchronize(st));
    const int rc = bpqn_solve_lcp_dense(A.data(), Ahat_dev ? Ah.data() : nullptr, n, b.data(), x.data(), opts, rep);
    BPQN_CUDA(cudaMemcpyAsync(x_dev, x.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    BPQN_CUDA(cudaStreamSynchronize(st));
    return rc;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  }
}

int bpqn_lcp_matrix_dense(bpqn_geom_t g, const bpqn_gmres_opts* gm, double* A_host, bpqn_gmres_stats* st,
                          void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && A_host, "null pointer");
    BPQN_REQUIRE(g->nc > 0, "no contacts installed");
    DenseLoStats d;
    std::vector<double> A;
    densify_lcp(*g, gm_or_default(gm), A, d, S(stream));
    std::copy(A.begin(), A.end(), A_host);
    if (st) {
      st->iters = d.iters;
      st->restarts = 0;
      st->rel_resid = 0.0;
      st->ms = d.ms_total;
      st->applies = d.iters;
    }
    return BPQN_OK;
  });
}

int bpqn_operator_dense(bpqn_geom_t g, double* A_dev, void* stream) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g && A_dev, "null pointer");
    assemble_dense_operator(*g, A_dev, S(stream));
    return BPQN_OK;
  });
}

int bpqn_gmres_recycle_reset(bpqn_geom_t g) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    gmres_recycle_reserve(*g);
    g->rec_k = 0;
    return BPQN_OK;
  });
}

int bpqn_profile_get(bpqn_geom_t g, double* ms_allpairs, double* ms_near, double* ms_self,
                     double* allpairs_gflop, long long* allpairs_launches, long long* kernel_launches) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    profile_collect(*g);
    if (allpairs_gflop) *allpairs_gflop = g->prof.allpairs_flop * 1e-9;
    if (ms_allpairs) *ms_allpairs = g->prof.ms_allpairs;
    if (ms_near) *ms_near = g->prof.ms_near;
    if (ms_self) *ms_self = g->prof.ms_self;
    if (allpairs_launches) *allpairs_launches = g->prof.allpairs_launches;
    if (kernel_launches) *kernel_launches = g->prof.launches;
    return BPQN_OK;
  });
}

int bpqn_profile_reset(bpqn_geom_t g, int enable_events) {
  return guarded([&]() -> int {
    BPQN_REQUIRE(g, "null handle");
    profile_collect(*g);
    g->prof.ms_allpairs = g->prof.ms_near = g->prof.ms_self = 0;
    g->prof.allpairs_flop = 0;
    g->prof.allpairs_launches = g->prof.launches = 0;
    g->prof.events = enable_events != 0;
    return BPQN_OK;
  });
}

}  // extern "C"
