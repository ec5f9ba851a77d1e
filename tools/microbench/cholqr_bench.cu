// Phase cycles of the CholeskyQR basis kernel (cholqr.cu) on one sketch, CTA 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLMRA_CHOLQR_CLOCKS \
//        -I../../paper_2303_11612_b200/csrc/kernels -o cholqr_bench cholqr_bench.cu
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>
#include "../../paper_2303_11612_b200/csrc/kernels/cholqr.cu"

int main(int argc, char** argv) {
  const long long I = argc > 1 ? atoll(argv[1]) : 1000;
  const int s = argc > 2 ? atoi(argv[2]) : 60;
  std::vector<double> h(I * s);
  unsigned long long x = 88172645463325252ull;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = (double)(x >> 11) * 0x1.0p-53 - 0.5;
  }
  double *c, *qc, *r;
  int* fail;
  cudaMalloc(&c, I * s * 8); cudaMalloc(&qc, I * s * 8); cudaMalloc(&r, s * s * 8); cudaMalloc(&fail, 4);
  cudaMemcpy(c, h.data(), I * s * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) lmra_dev::launch_cholqr(c, I, s, qc, r, fail, 0);
  unsigned long long z[10] = {0};
  cudaMemcpyToSymbol(lmra_dev::g_cqclk, z, sizeof(z));
  const int reps = 20;
  cudaEventRecord(a);
  for (int it = 0; it < reps; ++it) lmra_dev::launch_cholqr(c, I, s, qc, r, fail, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaMemcpyFromSymbol(z, lmra_dev::g_cqclk, sizeof(z));
  int f = -1;
  cudaMemcpy(&f, fail, 4, cudaMemcpyDeviceToHost);
  printf("I %lld s %d P %d: %.1f us per launch, fail %d, err %s\n", I, s, lmra_dev::cholqr_cluster_size(I),
         ms * 1e3 / reps, f, cudaGetErrorString(cudaGetLastError()));
  const char* names[] = {"load", "gram", "reduce", "chol+inv", " (loop)", "qupd", "rt"};
  printf("  (chol: U+A+bar %.0f, C+bar %.0f cycles per launch)\n", (double)z[8] / reps, (double)z[9] / reps);
  for (int i = 0; i < 7; ++i) if (names[i][0] != '-') printf("  %-7s %10.0f cycles per launch\n", names[i], (double)z[i] / reps);
  // check: orthogonality of Q and the residual C - Q R (host, plain loops)
  std::vector<double> q(I * s), rr(s * s);
  cudaMemcpy(q.data(), qc, I * s * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(rr.data(), r, s * s * 8, cudaMemcpyDeviceToHost);
  double orth = 0, res = 0, cn = 0;
  for (int a = 0; a < s; ++a)
    for (int b2 = 0; b2 < s; ++b2) {
      double acc = 0;
      for (long long i = 0; i < I; ++i) acc += q[i + I * a] * q[i + I * b2];
      orth = fmax(orth, fabs(acc - (a == b2)));
    }
  for (long long i = 0; i < I; ++i)
    for (int j = 0; j < s; ++j) {
      double acc = 0;
      for (int k = 0; k <= j; ++k) acc += q[i + I * k] * rr[k + s * j];
      res = fmax(res, fabs(acc - h[i + I * j]));
      cn = fmax(cn, fabs(h[i + I * j]));
    }
  printf("  max|Q^T Q - I| %.3g, max|C - Q R| / max|C| %.3g\n", orth, res / cn);
  return 0;
}
