// FP64 issue-model probe: DFMA throughput vs operand pattern and mixed ALU work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_issue_probe.cu -o /tmp/p && /tmp/p
#include <cstdio>
#include <cuda_runtime.h>

// mode 0: a_k = fma(a_k, b, c)               (2 distinct regs + acc; b,c shared)
// mode 1: a_k = fma(x_k, y_k, a_k)           (3 distinct per instr; x,y rotate)
// mode 2: a_k = a_k * b_k                    (DMUL, 2 distinct)
// mode 3: mode 1 + one 64-bit integer compare+select per DFMA
// mode 4: a_k = fma(a_k, a_k, c)             (1 distinct + c)
template <int MODE>
__global__ void k(double* sink, int iters, double b, double c) {
  constexpr int CH = 8;
  double a[CH], x[CH], y[CH];
  long long cnt = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = threadIdx.x * 1e-3 + i;
    x[i] = 1.0 + i * 1e-7 + threadIdx.x * 1e-9;
    y[i] = 0.999999 - i * 1e-8 - threadIdx.x * 1e-10;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) a[i] = fma(a[i], b, c);
      if (MODE == 1 || MODE == 3) a[i] = fma(x[i], y[(i + 3) % CH], a[i]);
      if (MODE == 2) a[i] = a[i] * x[i];
      if (MODE == 4) a[i] = fma(a[i], a[i], c);
      if (MODE == 3) {
        long long ab = __double_as_longlong(a[i]);
        cnt += (ab > 0x3ff0000000000000ll) ? 1 : 0;
      }
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) { x[i] = x[(i + 1) % CH]; }
  }
  double s = cnt;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i] + x[i];
  if (s == 1.2345e300) sink[0] = s;
}

template <int MODE>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  int iters = 200000, grid = sms * 4, threads = 256;
  k<MODE><<<grid, threads>>>(sink, 1000, 0.999999, 1e-7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<grid, threads>>>(sink, iters, 0.999999, 1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 8.0 * iters * (double)grid * threads;
  printf("%-40s %.3f Tinstr/s (x2 = %.2f TFLOP/s-equiv)  %.2f ms\n", name, ops / (ms * 1e-3) / 1e12,
         2 * ops / (ms * 1e-3) / 1e12, ms);
  cudaFree(sink);
}

int main() {
  run<0>("dfma a=fma(a,b,c)");
  run<4>("dfma a=fma(a,a,c)");
  run<1>("dfma a=fma(x,y,a) 3 distinct");
  run<2>("dmul a=a*x");
  run<3>("dfma 3-distinct + int64 cmp/add");
  return 0;
}
