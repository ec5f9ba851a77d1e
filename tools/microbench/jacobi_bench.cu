// Isolated timing of the orth Jacobi stage (cycles per round) on a random s x s matrix.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2303_11612_b200/csrc/kernels
//        -o jacobi_bench jacobi_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#define LMRA_JACOBI_CLOCKS 1

#include "../../paper_2303_11612_b200/csrc/kernels/orth.cu"

using namespace lmra_dev;

__global__ void __launch_bounds__(1024) jbench(const double* R, int s, int lpp, long long* out) {
  extern __shared__ double sm[];
  const int n = s + (s & 1);
  double* G = sm;
  double* J = G + s * n;
  int* flag = reinterpret_cast<int*>(J + n * n);
  for (int e = threadIdx.x; e < s * n; e += blockDim.x) G[e] = (e / s) < s ? R[e] : 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) J[e] = (e % n == e / n) ? 1.0 : 0.0;
  __syncthreads();
  long long t0 = clock64();
  bool ok = one_sided_jacobi(G, s, n, J, flag, 8.0 * s * 0x1.0p-53, reinterpret_cast<unsigned char*>(flag + 1));
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = ok;
  }
}

__global__ void __launch_bounds__(1024) qrbench(const double* C, int m, int s, int piv, long long* out) {
  extern __shared__ double sm[];
  double* A = sm;
  double* tau = A + m * s;
  double* cn = tau + s;
  int* pv = reinterpret_cast<int*>(cn + s);
  for (int e = threadIdx.x; e < m * s; e += blockDim.x) A[e] = C[e];
  __syncthreads();
  long long t0 = clock64();
  block_householder_qr(A, m, s, m, tau, piv ? pv : nullptr, cn);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 16);
  for (int s : {16, 30, 50, 60}) {
    std::vector<double> h(s * s);
    srand(1);
    for (auto& v : h) v = (rand() / (double)RAND_MAX) - 0.5;
    for (int j = 0; j < s; ++j)
      for (int i = j + 1; i < s; ++i) h[i + s * j] = 0.0;  // upper triangular like R
    // use R^T (lower) as G
    std::vector<double> g(s * s);
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) g[i + s * j] = h[j + s * i];
    double* d;
    cudaMalloc(&d, s * s * 8);
    cudaMemcpy(d, g.data(), s * s * 8, cudaMemcpyHostToDevice);
    int n = s + (s & 1);
    size_t smem = (s * n + n * n) * 8 + 64 + n * n;
    cudaFuncSetAttribute(jbench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int lpp : {0}) {
      jbench<<<1, 1024, smem>>>(d, s, lpp, out);
      cudaDeviceSynchronize();
      jbench<<<1, 1024, smem>>>(d, s, lpp, out);
      cudaDeviceSynchronize();
      unsigned long long clk[8];
      cudaMemcpyFromSymbol(clk, g_jclk, sizeof(clk));
      printf("{\"s\": %d, \"lpp\": %d, \"jacobi_cycles\": %lld, \"converged\": %lld, \"sweeps\": %d, "
             "\"dots_shfl\": %.0f, \"math\": %.0f, \"update\": %.0f, \"rot_rounds\": %llu}\n", s, lpp,
             out[0], out[1], last_jacobi_sweeps(), clk[0] / (double)clk[3], clk[1] / (double)clk[3],
             clk[2] / (double)clk[3], clk[3]);
      unsigned long long z[8] = {0};
      cudaMemcpyToSymbol(g_jclk, z, sizeof(z));
    }
    cudaFree(d);
  }
  for (int m : {180, 334, 400}) {
    int s = 60;
    std::vector<double> h(m * s);
    for (auto& v : h) v = (rand() / (double)RAND_MAX) - 0.5;
    double* d;
    cudaMalloc(&d, m * s * 8);
    cudaMemcpy(d, h.data(), m * s * 8, cudaMemcpyHostToDevice);
    size_t smem = (m * s + 2 * s) * 8 + s * 4 + 64;
    cudaFuncSetAttribute(qrbench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int piv : {0, 1}) {
      qrbench<<<1, 1024, smem>>>(d, m, s, piv, out);
      cudaDeviceSynchronize();
      qrbench<<<1, 1024, smem>>>(d, m, s, piv, out);
      cudaDeviceSynchronize();
      printf("{\"qr_m\": %d, \"s\": %d, \"pivot\": %d, \"cycles\": %lld}\n", m, s, piv, out[0]);
    }
    cudaFree(d);
  }
  return 0;
}
