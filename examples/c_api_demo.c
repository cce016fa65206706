/*
 * c_api_demo.c -- the drop-in boundary used from plain C (no Python, no torch):
 * SparseEmbedding(n, t, seed).apply(A) through include/sketch_b200.h.
 *
 * Build:  gcc -O2 -I include examples/c_api_demo.c -o examples/c_api_demo \
 *           -L paper_1207_6365_b200 -lsketch_b200 -L /usr/local/cuda/lib64 -lcudart \
 *           -Wl,-rpath,$PWD/paper_1207_6365_b200
 * Run:    ./examples/c_api_demo   (prints SA[0][0..3] and the first buckets)
 *
 * Mirrors sketch.py:143-165: seed both PCG64 streams (sketch.py:51-53), draw
 * h/s (K1), build the plan (K2), S.A for a dense fp64 A (K3).  All device
 * buffers belong to the caller; workspaces are sized by the *_workspace calls.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "sketch_b200.h"

#define CK(x)                                                                     \
  do {                                                                            \
    if ((x) != SKT_OK) {                                                          \
      fprintf(stderr, "%s failed: %s\n", #x, skt_last_error());                   \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CU(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));             \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(void) {
  const int64_t n = 1000, d = 4;
  const uint64_t t = 64;
  const uint32_t seed_words[1] = {1u};  /* seed = 1 */
  const uint32_t key_h[2] = {0u, 0u}, key_s[2] = {0u, 1u};
  skt_pcg64 hs, ss;
  CK(skt_pcg64_seed(seed_words, 1, key_h, 2, &hs));
  CK(skt_pcg64_seed(seed_words, 1, key_s, 2, &ss));

  uint32_t *h, *rows;
  int8_t *s;
  int64_t *indptr;
  double *a, *sa;
  void *ws = NULL;
  size_t wsb = 0, wsb2 = 0;
  CU(cudaMalloc((void **)&h, n * sizeof(uint32_t)));
  CU(cudaMalloc((void **)&s, n));
  CU(cudaMalloc((void **)&rows, n * sizeof(uint32_t)));
  CU(cudaMalloc((void **)&indptr, (t + 1) * sizeof(int64_t)));
  CU(cudaMalloc((void **)&a, n * d * sizeof(double)));
  CU(cudaMalloc((void **)&sa, t * d * sizeof(double)));
  CK(skt_hash_signs_workspace(n, t, &wsb));
  CK(skt_plan_workspace(n, t, 0, &wsb2));
  if (wsb2 > wsb) wsb = wsb2;
  if (wsb) CU(cudaMalloc(&ws, wsb));

  double *ha = (double *)malloc(n * d * sizeof(double));
  for (int64_t i = 0; i < n * d; ++i) ha[i] = (double)(i % 7) - 3.0;
  CU(cudaMemcpy(a, ha, n * d * sizeof(double), cudaMemcpyHostToDevice));

  CK(skt_hash_signs(&hs, &ss, 0, n, t, h, s, ws, wsb, NULL));
  CK(skt_plan_build(h, s, n, t, 0, indptr, rows, NULL, ws, wsb, NULL));
  CK(skt_apply_dense(indptr, rows, t, n, a, SKT_F64, d, d, sa, SKT_F64, d, NULL, NULL));

  double hsa[4];
  uint32_t hh[4];
  CU(cudaMemcpy(hsa, sa, 4 * sizeof(double), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hh, h, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  printf("bucket[0..3] = %u %u %u %u\n", hh[0], hh[1], hh[2], hh[3]);
  printf("SA[0][0..3]  = %.17g %.17g %.17g %.17g\n", hsa[0], hsa[1], hsa[2], hsa[3]);
  printf("kernel launches: %llu\n", (unsigned long long)skt_launch_count());
  free(ha);
  return 0;
}
