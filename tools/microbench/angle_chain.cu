// Dependent-chain latency (cycles) of Jacobi angle formulations (orth.cu jacobi_angle) on sm_100a,
// plus the per-round partial combine (24 shared loads + tree sums) that precedes it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o angle_chain angle_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rsqrt_nr1(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  return y * fma(-h * y, y, 1.5);
}
__device__ __forceinline__ double rsqrt_raw(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

template <int V>
__device__ __forceinline__ void angle(double a, double b, double c, double tol2, double& cs, double& sn) {
  cs = 1.0; sn = 0.0;
  if (!(c != 0.0 && c * c > tol2 * (a * b))) return;
  const double d = b - a;
  const double q = fma(d, d, 4.0 * c * c);
  double r;
  if (V == 0) r = q * rsqrt_nr(q);
  if (V == 1) r = q * rsqrt_nr1(q);
  if (V == 2) {  // fp32 seed on the scaled q
    const int e = (__double2hiint(q) >> 20) - 1023;
    const double qs = __hiloint2double(__double2hiint(q) - (e & ~1) * (1 << 20), __double2loint(q));
    const float rf = sqrtf((float)qs);
    r = __hiloint2double(__double2hiint((double)rf) + ((e & ~1) >> 1) * (1 << 20), 0);
  }
  const double u = fabs(d) + r;
  const double qn = rsqrt_nr(2.0 * r * u);
  cs = u * qn;
  sn = (d >= 0.0 ? 2.0 * c : -2.0 * c) * qn;
}

template <int V>
__global__ void chain(const double* in, double* out, long long* cyc, int iters) {
  __shared__ double part[3 * 8 * 32];
  const int l = threadIdx.x;
  for (int i = l; i < 3 * 8 * 32; i += 32) part[i] = in[i];
  __syncwarp();
  double cs = 1.0, sn = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double pa[8], pb[8], pc[8];
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) {
      pa[w2] = part[(0 * 8 + w2) * 32 + l];
      pb[w2] = part[(1 * 8 + w2) * 32 + l];
      pc[w2] = part[(2 * 8 + w2) * 32 + l];
    }
    const double sa = ((pa[0] + pa[1]) + (pa[2] + pa[3])) + ((pa[4] + pa[5]) + (pa[6] + pa[7]));
    const double sb = ((pb[0] + pb[1]) + (pb[2] + pb[3])) + ((pb[4] + pb[5]) + (pb[6] + pb[7]));
    const double sc = ((pc[0] + pc[1]) + (pc[2] + pc[3])) + ((pc[4] + pc[5]) + (pc[6] + pc[7]));
    if (V == 9) { cs = sa + sb + sc; sn = cs; }
    else angle<V>(sa, sb, sc, 1e-26, cs, sn);
    // feed back (dependency): next round's partials change
    part[l] = cs * 0.5 + 0.25;
    part[32 * 8 + l] = sn * 0.5 + 0.75;
    __syncwarp();
  }
  long long t1 = clock64();
  if (l == 0) cyc[0] = t1 - t0;
  out[l] = cs + sn;
}

int main() {
  double *in, *out; long long* cyc;
  cudaMalloc(&in, 8 * 768); cudaMalloc(&out, 8 * 32); cudaMallocManaged(&cyc, 8);
  double h[768];
  for (int i = 0; i < 768; ++i) h[i] = 0.1 + 0.001 * i;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  const int iters = 2000;
#define RUN(V, name) chain<V><<<1, 32>>>(in, out, cyc, iters); cudaDeviceSynchronize(); \
  chain<V><<<1, 32>>>(in, out, cyc, iters); cudaDeviceSynchronize(); \
  printf("{\"variant\": \"%s\", \"cycles\": %.1f}\n", name, (double)cyc[0] / iters);
  RUN(9, "loads+sums only")
  RUN(0, "current (2x rsqrt_nr)")
  RUN(1, "r with 1 NR")
  RUN(2, "r from fp32 sqrt")
  return 0;
}
