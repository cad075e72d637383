// Accuracy of the MUFU FP64 seeds and of the refined rcp/sqrt used by the GPP
// kernel, plus an FP64 DFMA throughput sweep.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2008_11326_b200/csrc \
//        tools/mufu_accuracy.cu -o /tmp/mufu && /tmp/mufu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "gpp_kernels.cuh"

__global__ void acc_kernel(const double* x, int n, double* err) {
  // err[0..6]: max rel err of rcp.approx, rcp_refined, rsqrt.approx, sqrt_nr<1>, sqrt_nr<3>,
  // and the production step's 1/d and sqrt(d)
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i];
  double e[6];
  double r0 = gpp::rcp_approx(v), r1 = gpp::rcp_refined(v);
  double exact_r = 1.0 / v;
  e[0] = fabs(r0 - exact_r) / exact_r;
  e[1] = fabs(r1 - exact_r) / exact_r;
  double s_exact = sqrt(v);
  double rs = gpp::rsqrt_approx(v);
  e[2] = fabs(rs - 1.0 / s_exact) * s_exact;
  e[3] = fabs(gpp::sqrt_nr<1>(v) - s_exact) / s_exact;
  e[4] = fabs(gpp::sqrt_nr<3>(v) - s_exact) / s_exact;
  // The production kernel's step (gpp_kernels.cuh sacc_band): MUFU.RSQ64H
  // high word paired with an arbitrary (dead) low word, one cubic step, then
  // 1/d = rr^2 and sqrt(d) = t (1 + q).  The low word here is the element
  // index, scrambled: any value must do.
  double r;
  const double junk = __longlong_as_double(0x3ff0000000000000ull ^ (i * 0x9E3779B97F4A7C15ull));
  asm("{\n\t.reg .b32 wl, wh, rl, rh;\n\t.reg .f64 s;\n\t"
      "mov.b64 {wl, wh}, %1;\n\t"
      "rsqrt.approx.ftz.f64 s, %2;\n\t"
      "mov.b64 {rl, rh}, s;\n\t"
      "mov.b64 %0, {wl, rh};\n\t}"
      : "=d"(r) : "d"(junk), "d"(v));
  const double t = v * r;
  const double ee = fma(-t, r, 1.0);
  const double pe = fma(ee, 0.375, 0.5);
  const double q = ee * pe;
  const double rr = fma(r, q, r);
  const double sq = fma(t, q, t);
  const double inv = rr * rr;
  e[5] = fabs(inv - exact_r) / exact_r;
  double e6 = fabs(sq - s_exact) / s_exact;
  for (int k = 0; k < 6; ++k) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(err + k);
    atomicMax(p, __double_as_longlong(e[k]));
  }
  atomicMax(reinterpret_cast<unsigned long long*>(err + 6), __double_as_longlong(e6));
}

template <int CH>
__global__ void peak_kernel(double* sink, int iters, double b, double c) {
  double a[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += a[k];
  if (s == 1.2345e300) sink[0] = s;
}

template <int CH>
void peak(int blocks_per_sm, int threads) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  int iters = 400000 / CH * 8;
  int grid = sms * blocks_per_sm;
  peak_kernel<CH><<<grid, threads>>>(sink, iters / 10, 0.999999, 1e-7);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  peak_kernel<CH><<<grid, threads>>>(sink, iters, 0.999999, 1e-7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double tf = 2.0 * CH * (double)iters * grid * threads / (ms * 1e-3) / 1e12;
  printf("peak chains=%2d blocks/SM=%d threads=%d: %.2f TFLOP/s (%.1f ms)\n", CH, blocks_per_sm, threads, tf, ms);
  cudaFree(sink);
}

int main() {
  const int n = 1 << 22;
  double* h = new double[n];
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    double u = (s >> 11) * (1.0 / 9007199254740992.0);
    h[i] = std::pow(10.0, -8.0 + 16.0 * u);  // 1e-8 .. 1e8, log-uniform
  }
  double *x, *err;
  cudaMalloc(&x, n * 8); cudaMalloc(&err, 8 * 8);
  cudaMemcpy(x, h, n * 8, cudaMemcpyHostToDevice);
  cudaMemset(err, 0, 8 * 8);
  acc_kernel<<<(n + 255) / 256, 256>>>(x, n, err);
  double e[8]; cudaMemcpy(e, err, 8 * 8, cudaMemcpyDeviceToHost);
  printf("max rel err: rcp.approx %.3e (2^%.1f)  rcp_refined %.3e  rsqrt.approx %.3e (2^%.1f)  sqrt_nr1 %.3e  sqrt_nr3(cubic) %.3e\n",
         e[0], std::log2(e[0]), e[1], e[2], std::log2(e[2]), e[3], e[4]);
  printf("production step (seed high word + arbitrary low word, one cubic step): 1/d %.3e (%.2f ulp)  sqrt(d) %.3e (%.2f ulp)\n",
         e[5], e[5] / 1.1102230246251565e-16, e[6], e[6] / 1.1102230246251565e-16);
  peak<4>(8, 256); peak<8>(8, 256); peak<16>(8, 256); peak<8>(4, 256); peak<8>(16, 128); peak<32>(4, 256);
  return 0;
}
