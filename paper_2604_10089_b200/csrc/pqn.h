// Host PQN solvers of libbpqn (see pqn.cpp).
#pragma once
#include <functional>
#include <utility>
#include <vector>

namespace bpqn {

using MvpFn = std::function<void(const std::vector<double>& v, std::vector<double>& out, std::vector<double>* aux)>;

struct PqnOpts {
  int k_max = 200;
  double eps_abs = 1e-10, eps_rel = 0.0, tau = 1.0;
  int refresh = 20;
  double sub_eps_factor = 1e-2;
  int sub_k_max = 50;
  double prox_tol = 0.0;
  int prox_jmax = 100;
  double curv = 1e-12;
  double sub_forcing = 0.0;
  bool verify_secants = false;  // Bi-PQN: measure max |B^(k) s - y| of the re-used pairs (tests)
};

// C^-1 U and C^-1 V (C = I + U U^T) for the prox's Woodbury step, kept across prox calls
// on the same memory and extended by Sherman-Morrison as pairs are appended (O(r n) per
// pair instead of O(r^2 n) per call); rebuilt after a clear or every 64 appends.
struct WoodburyCache {
  int r = 0, n = 0, appends = 0;
  std::vector<double> Um, Vm, CU, CV;  // [r][n] row-major
  // dual root [alpha; alpha~] of the last prox call and its rank: the next call on the same
  // (appended) memory starts its semi-smooth Newton from it, padded with zeros
  std::vector<double> alpha;
  int alpha_r = 0;
};

struct Bfgs {
  std::vector<std::vector<double>> U, V, S, Y;
  mutable WoodburyCache wc;
  void clear();
  std::vector<double> B(const std::vector<double>& x) const;
  std::vector<double> H(const std::vector<double>& g) const;
  bool update(const std::vector<double>& s, const std::vector<double>& y, const std::vector<double>* Bs,
              double curv);
};

struct MonoResult {
  std::vector<double> x, g, aux;
  std::vector<std::pair<std::vector<double>, std::vector<double>>> pairs;
  int iterations = 0, mvps = 0, termination = 2;
  double kkt = 0, kkt_rel = 0;
};

struct BiResult {
  std::vector<double> x, g;
  int iterations = 0, hi_mvps = 0, lo_mvps = 0, termination = 2, init_iterations = 0, init_lo_mvps = 0;
  std::vector<int> sub_iterations;
  double kkt = 0, kkt_rel = 0;
  double secant_residual = 0;  // with verify_secants: max over subproblems and seeded pairs
};

double kkt_abs(const std::vector<double>& x, const std::vector<double>& g);
void prox_profile_flush();
std::vector<double> weighted_prox(const Bfgs& q, const std::vector<double>& xt, double tol, int jmax, int* iters);
double optimal_eta(const std::vector<double>& x, const std::vector<double>& p, const std::vector<double>& g,
                   const std::vector<double>& Ap, std::vector<char>& bind);
MonoResult mono_pqn(const MvpFn& mvp, const std::vector<double>& b, const std::vector<double>& x0, const PqnOpts& o,
                    const std::vector<double>* g0, const std::vector<double>* aux0,
                    const std::vector<std::pair<std::vector<double>, std::vector<double>>>* seed);
MonoResult bb_pgd(const MvpFn& mvp, const std::vector<double>& b, const std::vector<double>& x0, const PqnOpts& o);
BiResult bi_pqn(const MvpFn& hi, const MvpFn& lo, const std::vector<double>& b, const std::vector<double>& x_init,
                const PqnOpts& o);

}  // namespace bpqn
