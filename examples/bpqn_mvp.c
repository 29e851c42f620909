/* Plain-C client of libbpqn (include/bpqn.h): one LCP MVP w = D^T M D lambda on a
 * 2x2x2 lattice of unit spheres, then a Mono-PQN solve -- no Python, no PyTorch.
 *
 *   ./bpqn_mvp [p]      prints one JSON line
 *
 * Device buffers come from the CUDA runtime; everything else is the C ABI.  Exit code:
 * 0 ok, 1 library error (message from bpqn_last_error), 2 CUDA runtime error. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "../include/bpqn.h"

#define CHECK(call)                                                                \
  do {                                                                             \
    int rc_ = (call);                                                              \
    if (rc_ != BPQN_OK && rc_ != BPQN_ERR_NOCONV) {                                \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, bpqn_last_error());      \
      return 1;                                                                    \
    }                                                                              \
  } while (0)
#define CUDA(call)                                                                 \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                  \
      return 2;                                                                    \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const int p = argc > 1 ? atoi(argv[1]) : 8;
  double centers[8 * 3];
  int k = 0;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int l = 0; l < 2; ++l) {
        centers[3 * k] = 2.05 * i + 0.01 * l;
        centers[3 * k + 1] = 2.05 * j - 0.01 * i;
        centers[3 * k + 2] = 2.05 * l + 0.005 * j;
        ++k;
      }
  bpqn_geom_t g;
  CHECK(bpqn_geometry_init(&g, 8, centers, 1.0, 1.0, p, NULL, NULL));
  const int cap = 28;
  int *pairs;
  double *normals, *gaps, *lam, *w, *b;
  CUDA(cudaMalloc((void**)&pairs, 2 * cap * sizeof(int)));
  CUDA(cudaMalloc((void**)&normals, 3 * cap * sizeof(double)));
  CUDA(cudaMalloc((void**)&gaps, cap * sizeof(double)));
  int nc = 0;
  CHECK(bpqn_contacts(g, 0.1, cap, &nc, pairs, normals, gaps, NULL));
  CUDA(cudaMalloc((void**)&lam, nc * sizeof(double)));
  CUDA(cudaMalloc((void**)&w, nc * sizeof(double)));
  CUDA(cudaMalloc((void**)&b, nc * sizeof(double)));
  double hl[64], hw[64], hb[64];
  for (int i = 0; i < nc; ++i) {
    hl[i] = 1.0 / (1 + i);
    hb[i] = (i % 2 ? 0.02 : -0.05);
  }
  CUDA(cudaMemcpy(lam, hl, nc * sizeof(double), cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(b, hb, nc * sizeof(double), cudaMemcpyHostToDevice));
  bpqn_gmres_opts gm;
  bpqn_default_gmres_opts(&gm);
  bpqn_gmres_stats st;
  CHECK(bpqn_lcp_mvp(g, lam, w, &gm, &st, NULL));
  CUDA(cudaMemcpy(hw, w, nc * sizeof(double), cudaMemcpyDeviceToHost));
  double nw = 0;
  for (int i = 0; i < nc; ++i) nw += hw[i] * hw[i];
  /* Mono-PQN from lambda = 0 */
  CUDA(cudaMemset(lam, 0, nc * sizeof(double)));
  bpqn_solve_opts so;
  bpqn_default_solve_opts(&so);
  bpqn_report rep;
  CHECK(bpqn_solve_lcp(g, NULL, b, lam, &so, &rep, NULL));
  printf("{\"p\": %d, \"n_contacts\": %d, \"w_norm\": %.17g, \"w0\": %.17g, \"gmres_iters\": %d, "
         "\"lcp_iterations\": %d, \"hi_mvps\": %d, \"kkt_abs\": %.3e}\n",
         p, nc, sqrt(nw), hw[0], st.iters, rep.iterations, rep.hi_mvps, rep.kkt_abs);
  bpqn_geometry_destroy(g);
  cudaFree(pairs);
  cudaFree(normals);
  cudaFree(gaps);
  cudaFree(lam);
  cudaFree(w);
  cudaFree(b);
  return 0;
}
