// fp64 peak microbenchmarks for B200 (sm_100a): DFMA loop, DMMA (mma.sync f64)
// loops in every legal shape, and streaming read/copy bandwidth with fp64 loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C 2 regs. 8*8*4 = 256 FMA per warp instruction.
template <int CHAINS>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k4: A 2 regs, B 1 reg, C 4 regs. 16*8*4 = 512 FMA.
template <int CHAINS>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-6, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-6;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int j = 0; j < 4; ++j) c[k][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k16: A 8 regs, B 4 regs, C 4 regs. 16*8*16 = 2048 FMA.
template <int CHAINS>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + (threadIdx.x + j) * 1e-6;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - (threadIdx.x + j) * 1e-6;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int j = 0; j < 4; ++j) c[k][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void read_sum(const double2* __restrict__ x, size_t n2, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldg(x + i);
    s += v.x * v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_k(const double2* __restrict__ x, double2* __restrict__ y, size_t n2) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) y[i] = x[i];
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, l2 = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d}\n", sms, l2, clk);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int iters = 4096;
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, blocks = sms * bpsm;
    float ms = time_it([&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3); }, 5);
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf("{\"kernel\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, blocks = sms * bpsm;
    float ms = time_it([&] { dmma_m8n8k4<8><<<blocks, threads>>>(out, iters); }, 5);
    double fl = 2.0 * 256 * 8 * iters * (double)(threads / 32) * blocks;
    printf("{\"kernel\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, blocks = sms * bpsm;
    float ms = time_it([&] { dmma_m16n8k4<8><<<blocks, threads>>>(out, iters); }, 5);
    double fl = 2.0 * 512 * 8 * iters * (double)(threads / 32) * blocks;
    printf("{\"kernel\": \"dmma_m16n8k4\", \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) {
    int threads = 256, blocks = sms * bpsm;
    float ms = time_it([&] { dmma_m16n8k16<4><<<blocks, threads>>>(out, iters / 4); }, 5);
    double fl = 2.0 * 2048 * 4 * (iters / 4) * (double)(threads / 32) * blocks;
    printf("{\"kernel\": \"dmma_m16n8k16\", \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", bpsm, fl / ms / 1e9);
  }
  // streaming bandwidth (2 GiB buffers, far above L2)
  size_t n = (size_t)1 << 28;  // doubles = 2 GiB
  double *x, *y;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8));
  CK(cudaMemset(x, 0, n * 8));
  for (int bpsm : {2, 4, 8, 16}) {
    int blocks = sms * bpsm;
    float ms = time_it([&] { read_sum<<<blocks, 256>>>((const double2*)x, n / 2, out); }, 10);
    printf("{\"kernel\": \"read\", \"blocks_per_sm\": %d, \"gbs\": %.1f}\n", bpsm, n * 8.0 / ms / 1e6);
  }
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm;
    float ms = time_it([&] { copy_k<<<blocks, 256>>>((const double2*)x, (double2*)y, n / 2); }, 10);
    printf("{\"kernel\": \"copy\", \"blocks_per_sm\": %d, \"gbs\": %.1f}\n", bpsm, 2 * n * 8.0 / ms / 1e6);
  }
  return 0;
}
